"""CPU baseline probe: rate vs starting chain and window."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1807_05358_b200 as ps
from bench import cpu_baseline, initial_strategies, workload
g, topo, md, _ = workload("inception")
init = initial_strategies(g, topo, md, 0, 1024)
seeds = [1000003 * c for c in range(1024)]
prof = ps.CostProfile()
for first, win, secs in [(0, 815, 6), (368, 1000, 6), (0, 1000, 6), (368, 815, 6), (16, 815, 6)]:
    r = cpu_baseline(g, topo, prof, "full-iteration", md, init, seeds, secs, os.cpu_count(), proposals=win, first=first)
    print(first, win, round(r["value"]), r["sample"])
