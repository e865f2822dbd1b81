"""Per-phase cycle breakdown of k_mcmc (debug build with -DPS_PHASES)."""
import ctypes, math, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PARASIM_B200_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                     "paper_1807_05358_b200", "_lib", "dbg", "libparasim_cuda.so"))
import paper_1807_05358_b200 as ps
from paper_1807_05358_b200 import _native as nat
from paper_1807_05358_b200.lowering import lower
mode = sys.argv[1] if len(sys.argv) > 1 else "full-iteration"
C = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
g, topo = ps.inception_v3(), ps.multi_node_topology(4, 4)
init = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, 4, c) for c in range(1, C)]
low = lower(g, topo, ps.CostProfile(), mode, max_degree=4, strategies=init)
L = nat.lib()
L.ps_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_int]
maps = np.zeros((C, low.n_ops), np.int32); asg = np.zeros((C, low.n_slots), np.uint8)
for i, s in enumerate(init):
    low.encode(s, maps[i], asg[i])
seeds = np.array([1000003 * i for i in range(C)], np.uint64)
mp = nat.PsMcmcParams(nat.PS_RNG_PHILOX, 0, 0.0, math.log(10.0), 0, 0)
h = ctypes.c_void_p()
nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), C, nat.ptr(maps), nat.ptr(asg), nat.ptr(seeds), None, ctypes.byref(h)), "create")
nat.check(L.ps_mcmc_run_budget(h, 1 << 30, 50_000_000, None), "run")
ph = np.zeros(16, np.uint64)
nat.check(L.ps_debug_phases(nat.ptr(ph), 1), "phases")
nat.check(L.ps_mcmc_run_budget(h, 1 << 30, 100_000_000, None), "run")
nat.check(L.ps_debug_phases(nat.ptr(ph), 1), "phases")
info = low.info()
names = ["setup", "init", "select", "succ-setup", "succ-iters", "sel:LB(fast)", "mcmc-loop", "proposals", "sims", "rows-staged",
         "state-in-smem", "rounds", "sum-n", "winners", "iters"]
sims = ph[8]; rounds = ph[11]
print(f"mode={mode} chains={C} SC={info.shared_counters} warps/SM={info.resident_warps_per_sm} wpb={info.warps_per_block}")
print(f"sims={sims} proposals={ph[7]} rounds/sim={rounds/max(sims,1):.1f} avg n={ph[12]/max(rounds,1):.1f} "
      f"winners/round={ph[13]/max(rounds,1):.2f} iters/round={ph[14]/max(rounds,1):.2f} rows staged={ph[9]/max(sims,1):.2f} "
      f"state in smem={ph[10]/max(sims,1):.2f}")
tot = ph[6]
names.append("sel:claim+compact(fast)")
for i in (0, 1, 2, 5, 15, 3, 4):
    print(f"{names[i]:12s} {ph[i]/max(sims,1):12.0f} cycles/sim  {100*ph[i]/max(tot,1):5.1f}% of loop   "
          f"{ph[i]/max(rounds,1):8.0f} cycles/round")
print(f"loop total {tot/max(sims,1):.0f} cycles/sim")
