"""Debug: per-chain delta bookkeeping after each launch (GPU box)."""
import ctypes, math, sys, os, random
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1807_05358_b200 as ps
from paper_1807_05358_b200 import _native as nat
from paper_1807_05358_b200.lowering import lower

if "--pre" in sys.argv:
    from helpers import random_graph, random_topology
    for seed in range(10):
        rng = random.Random(3000 + seed)
        g = random_graph(rng, 4, 14); topo = random_topology(rng, rng.choice((2, 4, 8, 16)))
        mode = ps.MODE_FULL if seed % 2 else ps.MODE_FORWARD; md = rng.choice((2, 3, 4))
        init = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, md, seed + i) for i in range(3)]
        ps.mcmc_search(g, topo, ps.CostProfile(), ps.SearchParams(max_proposals=120, seed=seed, max_degree=md, mode=mode,
                                                                  initial=init, polish=False, rng="philox"))
g, topo, md = ps.inception_v3(), ps.multi_node_topology(4, 4), 4
C = 96
init = [ps.data_parallel_strategy(g, topo)] + ps.random_strategies(g, topo, md, list(range(1, C)))
low = lower(g, topo, ps.CostProfile(), ps.MODE_FULL, max_degree=md, strategies=init)
maps = np.zeros((C, low.n_ops), dtype=np.int32); asg = np.zeros((C, low.n_slots), dtype=np.uint8)
for i, s in enumerate(init):
    low.encode(s, maps[i], asg[i])
L = nat.lib()
L.ps_debug_delta_state.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
mp = nat.PsMcmcParams(nat.PS_RNG_PHILOX, 0, 0.0, math.log(10.0), 0, 0, 1)
h = ctypes.c_void_p()
sd = np.array([1000003 * c for c in range(C)], dtype=np.uint64)
nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), C, nat.ptr(maps), nat.ptr(asg), nat.ptr(sd), None, ctypes.byref(h)), "create")
dt = np.dtype([("stride", np.int32), ("nvalid", np.int32), ("cur", np.uint32), ("bad", np.uint32), ("fsel", np.int32),
               ("pad", np.int32), ("run", np.int64), ("reused", np.int64)])
for launch in range(4):
    nat.check(L.ps_mcmc_run(h, 0 if launch == 0 else 50, None), "run")
    out = np.zeros(C, dtype=dt)
    nat.check(L.ps_debug_delta_state(h, out.ctypes.data), "dbg")
    print("launch", launch, "stride", np.unique(out["stride"])[:10], "nvalid", np.unique(out["nvalid"])[:10],
          "bad", [hex(x) for x in np.unique(out["bad"])[:6]], "run", out["run"][:6], "reused", out["reused"][:6])
summ = (nat.PsChainSummary * C)()
nat.check(L.ps_mcmc_read(h, summ, None, None, None, None), "read")
print("summary rounds", [(s.rounds_run, s.rounds_reused) for s in summ[:6]])
tc = np.zeros((C, 1)); 
nat.check(L.ps_mcmc_read(h, summ, None, None, nat.ptr(tc), None), "read")
print("summary rounds (trace ptr)", [(s.rounds_run, s.rounds_reused) for s in summ[:6]])
