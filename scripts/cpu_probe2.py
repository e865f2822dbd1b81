"""Is the CPU baseline slower after the GPU part of the bench?"""
import os, subprocess, sys, json, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1807_05358_b200 as ps
from bench import cpu_baseline, initial_strategies, workload
g, topo, md, _ = workload("inception")
init = initial_strategies(g, topo, md, 0, 1024)
seeds = [1000003 * c for c in range(1024)]
prof = ps.CostProfile()
def run(tag):
    r = cpu_baseline(g, topo, prof, "full-iteration", md, init, seeds, 6, os.cpu_count(), proposals=815, first=0)
    print(tag, round(r["value"]), flush=True)
run("before-cuda")
import torch
x = torch.zeros(1, device="cuda"); torch.cuda.synchronize()
run("after-cuda-init")
from bench import Chains
import ctypes
ch = Chains("inception", "full-iteration", 1024, 0, True, 0)
s = torch.cuda.current_stream(); sh = ctypes.c_void_p(s.cuda_stream)
for _ in range(5): ch.step(ch.h, sh, 100_000_000, 0)
torch.cuda.synchronize()
run("after-gpu-work")
ch.destroy()
run("after-destroy")
