"""Per-launch time and proposals of time-boxed k_mcmc segments (multiplexed vs waves)."""
import ctypes, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from bench import Chains
cfg = sys.argv[1]; C = int(sys.argv[2]); bms = float(sys.argv[3])
ch = Chains(cfg, "full-iteration", C, 0, True, 0, distinct=16)
s = torch.cuda.current_stream()
sh = ctypes.c_void_p(s.cuda_stream)
prev = 0
for i in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); ch.step(ch.h, sh, int(bms * 1e6), 0); b.record(s); torch.cuda.synchronize()
    summ = ch.summary()
    props = sum(x.proposals for x in summ)
    pc = np.array([x.proposals for x in summ])
    print(f"launch {i}: {a.elapsed_time(b):.0f} ms, proposals {props - prev}, per-chain min/max {pc.min()}/{pc.max()}")
    prev = props
