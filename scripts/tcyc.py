"""Cycle timeline of one simulation (warp 0, block 0) through the round's
checkpoints (debug build with -DPS_TCYC): mean cycles between checkpoints."""
import ctypes, math, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PARASIM_B200_LIB", os.path.join(ROOT, "paper_1807_05358_b200", "_lib", "tc", "libparasim_cuda.so"))
import paper_1807_05358_b200 as ps
from paper_1807_05358_b200 import _native as nat
from paper_1807_05358_b200.lowering import lower
C = 1024
g, topo = ps.inception_v3(), ps.multi_node_topology(4, 4)
print("lib", os.environ["PARASIM_B200_LIB"])
init = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, 4, c) for c in range(1, C)]
low = lower(g, topo, ps.CostProfile(), "full-iteration", max_degree=4, strategies=init)
L = nat.lib()
maps = np.zeros((C, low.n_ops), np.int32); asg = np.zeros((C, low.n_slots), np.uint8)
for i, s in enumerate(init):
    low.encode(s, maps[i], asg[i])
seeds = np.array([1000003 * i for i in range(C)], np.uint64)
mp = nat.PsMcmcParams(nat.PS_RNG_PHILOX, 0, 0.0, math.log(10.0), 0, 0)
h = ctypes.c_void_p()
nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), C, nat.ptr(maps), nat.ptr(asg), nat.ptr(seeds), None, ctypes.byref(h)), "create")
nat.check(L.ps_mcmc_run_budget(h, 1 << 30, 50_000_000, None), "run")
buf = np.zeros(4096 * 16, np.int64)
L.ps_debug_tcyc.argtypes = [ctypes.c_void_p]
nat.check(L.ps_debug_tcyc(nat.ptr(buf)), "tcyc")
raw = buf.reshape(4096, 16).astype(np.float64)
t = raw[:, :10]
names = ["top->el", "el->LB", "LB->any(member)", "->claim/lost", "->rank(match)", "->compact", "->run(+trace)",
         "->succ setup", "->iterations"]
fast = (t[:, :10] > 0).all(axis=1)
fast &= (np.diff(t, axis=1) >= 0).all(axis=1)
print(f"rounds traced: {(t[:, 0] > 0).sum()}, fast-path rounds: {fast.sum()}")
d = np.diff(t[fast], axis=1)
for i, n in enumerate(names):
    print(f"{n:18s} {d[:, i].mean():8.1f} cycles (median {np.median(d[:, i]):.0f})")
sub = raw[fast][:, [7, 10, 11, 8, 12, 13, 14, 9]]
for i, n in enumerate(["succ: shfl/decode", "succ: pair walk+fixed", "succ: entry load+max", "it0: entry->key/link",
                       "it0: atomicMax+sync", "it0: count/attrs", "it: err/push/rest"]):
    dd = sub[:, i + 1] - sub[:, i]
    print(f"  {n:24s} {dd.mean():8.1f} (median {np.median(dd):.0f})")
tot = t[fast][:, 9] - t[fast][:, 0]
nxt = t[1:, 0] - t[:-1, 9]
print(f"round (fast) {tot.mean():.0f} cycles; loop-back {np.median(nxt[nxt > 0]):.0f}")
ok = (raw[:, 0] > 0) & (raw[:, 9] > raw[:, 0])
slow = ok & ~fast
st = raw[slow][:, 9] - raw[slow][:, 0]
if slow.sum():
    print(f"slow-path rounds: {slow.sum()} of {ok.sum()}, mean {st.mean():.0f} cycles "
          f"({100 * st.sum() / (raw[ok][:, 9] - raw[ok][:, 0]).sum():.1f}% of round time)")
