"""Per-phase cycle breakdown of k_mcmc (debug build with -DPS_PHASES):
python scripts/phases.py [mode] [chains] [config] [budget_ms]"""
import ctypes, math, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PARASIM_B200_LIB", os.path.join(ROOT, "paper_1807_05358_b200", "_lib", "dbg", "libparasim_cuda.so"))
import paper_1807_05358_b200 as ps
from paper_1807_05358_b200 import _native as nat
from bench import Chains
mode = sys.argv[1] if len(sys.argv) > 1 else "full-iteration"
C = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
cfg = sys.argv[3] if len(sys.argv) > 3 else "inception"
bms = float(sys.argv[4]) if len(sys.argv) > 4 else 100.0
distinct = None if cfg in ("inception", "alexnet", "resnet") else 16
ch = Chains(cfg, mode, C, 0, True, 0, distinct=distinct)
L = nat.lib()
L.ps_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_int]
N = 40
ph = np.zeros(N, np.uint64)
nat.check(L.ps_mcmc_run_budget(ch.h, 1 << 30, int(bms * 0.5e6), None), "run")
nat.check(L.ps_debug_phases(nat.ptr(ph), 1), "phases")
nat.check(L.ps_mcmc_run_budget(ch.h, 1 << 30, int(bms * 1e6), None), "run")
nat.check(L.ps_debug_phases(nat.ptr(ph), 1), "phases")
info = ch.low.info()
names = ["setup", "init", "select", "succ-setup", "succ-iters", "sel:LB(fast)", "mcmc-loop", "proposals", "sims",
         "rows-staged", "state-in-smem", "rounds", "sum-n", "winners", "iters", "sel:claim+compact(fast)",
         "slow rounds", "slow sum-n", "slow winners", "slow cycles"]
sims = ph[8]; rounds = ph[11]
print(f"{cfg} mode={mode} chains={C} SC={info.shared_counters} cap={info.ready_capacity} "
      f"warps/SM={info.resident_warps_per_sm} wpb={info.warps_per_block} slots={ch.low.n_slots} queues={info.n_queues}")
print(f"sims={sims} proposals={ph[7]} rounds/sim={rounds/max(sims,1):.1f} avg n={ph[12]/max(rounds,1):.1f} "
      f"winners/round={ph[13]/max(rounds,1):.2f} iters/round={ph[14]/max(rounds,1):.2f} rows staged={ph[9]/max(sims,1):.2f} "
      f"state in smem={ph[10]/max(sims,1):.2f}")
print(f"slow rounds {100*ph[16]/max(rounds,1):.1f}% avg n(slow)={ph[17]/max(ph[16],1):.1f} "
      f"winners(slow)={ph[18]/max(ph[16],1):.2f} cycles/slow round={ph[19]/max(ph[16],1):.0f}")
print(f"run-winners {ph[20]/max(rounds,1):.0f} cycles/round; refill restarts {100*ph[21]/max(rounds,1):.1f}% of rounds; "
      f"medium-path rounds {100*ph[22]/max(rounds,1):.1f}%")
print(f"snapshots {ph[23]/max(sims,1):.1f}/sim, unusable: back set {100*ph[24]/max(ph[23],1):.1f}% "
      f"ready set over capacity {100*ph[25]/max(ph[23],1):.1f}%")
print(f"init: in-degrees {ph[26]/max(sims,1):.0f} cycles/sim, restore or seed {ph[27]/max(sims,1):.0f} cycles/sim")
print(f"snapshot writes {ph[28]/max(sims,1):.0f} cycles/sim, delta_prepare {ph[29]/max(sims,1):.0f} cycles/sim")
print(f"front trims {100*ph[31]/max(rounds,1):.1f}% of rounds, {ph[30]/max(ph[31],1):.0f} cycles each, "
      f"{ph[30]/max(rounds,1):.0f} cycles/round")
print(f"restarted selections (refill from BACK_CHECK) {ph[32]/max(rounds,1):.0f} cycles/round; "
      f"round-start refills / combined slow set-up {ph[33]/max(rounds,1):.0f} cycles/round")
tot = ph[6]
for i in (0, 1, 2, 5, 15, 19, 3, 4):
    print(f"{names[i]:12s} {ph[i]/max(sims,1):12.0f} cycles/sim  {100*ph[i]/max(tot,1):5.1f}% of loop   "
          f"{ph[i]/max(rounds,1):8.0f} cycles/round")
print(f"loop total {tot/max(sims,1):.0f} cycles/sim")
