"""Debug: first divergent proposal between delta and from-scratch evaluation (GPU box)."""
import ctypes, math, sys, os, random
import numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
os.environ["PS_DELTA_TRACE"] = "200"
import paper_1807_05358_b200 as ps
from paper_1807_05358_b200 import _native as nat
from paper_1807_05358_b200.lowering import lower
from helpers import random_graph, random_topology
L = nat.lib()
L.ps_debug_delta_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
for seed in range(10):
    rng = random.Random(3000 + seed)
    g = random_graph(rng, 4, 14); topo = random_topology(rng, rng.choice((2, 4, 8, 16)))
    mode = ps.MODE_FULL if seed % 2 else ps.MODE_FORWARD; md = rng.choice((2, 3, 4))
    init = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, md, seed + i) for i in range(3)]
    low = lower(g, topo, ps.CostProfile(), mode, max_degree=md, strategies=init)
    C, P = len(init), 120
    res = {}
    for delta in (1, 0):
        maps = np.zeros((C, low.n_ops), dtype=np.int32); asg = np.zeros((C, low.n_slots), dtype=np.uint8)
        for i, s in enumerate(init):
            low.encode(s, maps[i], asg[i])
        mp = nat.PsMcmcParams(nat.PS_RNG_PHILOX, 0, 0.0, math.log(10.0), 1, P, delta)
        h = ctypes.c_void_p()
        sd = np.array([seed + 1000003 * c for c in range(C)], dtype=np.uint64)
        nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), C, nat.ptr(maps), nat.ptr(asg), nat.ptr(sd), None, ctypes.byref(h)), "c")
        nat.check(L.ps_mcmc_run(h, P, None), "r")
        summ = (nat.PsChainSummary * C)()
        tc = np.zeros((C, P))
        nat.check(L.ps_mcmc_read(h, summ, None, None, nat.ptr(tc), None), "read")
        dbg = np.zeros((C, 200, 8), dtype=np.int32)
        frb = np.zeros((C, 4, low.n_ops), dtype=np.int32)
        if delta:
            nat.check(L.ps_debug_delta_trace(h, nat.ptr(dbg), nat.ptr(frb)), "dbg")
        res[delta] = (tc, dbg, frb)
        L.ps_mcmc_destroy(h)
    a, b = res[1][0], res[0][0]
    for c in range(C):
        bad = np.nonzero(a[c] != b[c])[0]
        if bad.size:
            k = int(bad[0])
            print(f"seed {seed} mode {mode} chain {c} first diff at proposal {k}: delta {a[c,k]!r} scratch {b[c,k]!r}")
            print("  ops:", low.ops, "n_ops", low.n_ops)
            for q in range(max(0, k - 3), k + 1):
                print("  prop", q, "op,j,nvalid,rounds,stride,last,bad,fsel =", list(res[1][1][c, q]))
            print("  frb:", res[1][2][c].tolist())
            pairs = [(low.ops[s_], low.ops[d_]) for s_, d_ in low.pairs]
            print("  pairs:", pairs)
            break
