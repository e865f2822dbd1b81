#!/usr/bin/env python3
"""Microbench: a reference-style update_task_graph + delta_simulate loop through
the drop-in API (the loop the reference's mcmc_search runs per proposal,
search.py:230-241), ours vs the unmodified reference (baseline/_ref, the
`pip install --target` copy of /root/reference/pkg; skipped if absent).

Both sides replay the same sequence of single-op changes (Inception-v3 on 4x4
devices, full-iteration, max degree 4, from a random start) and must produce
identical makespans.  Prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def changes(g, topo, md, n, seed):
    import paper_1807_05358_b200 as ps
    rng = random.Random(seed)
    out = []
    ops = sorted(g.ops)
    for _ in range(n):
        op_id = rng.choice(ops)
        cfg = rng.choice(ps.enumerate_configs(g.ops[op_id], topo, md))
        asg = tuple(rng.choice(topo.device_ids()) for _ in range(cfg.size()))
        out.append((op_id, dict(cfg.degrees), asg))
    return out


def run_ours(g, topo, start, seq, mode):
    import paper_1807_05358_b200 as ps
    prof = ps.CostProfile()
    tg = ps.build_task_graph(g, topo, start, prof, mode)
    ps.full_simulate(tg)
    # warm the resident delta handle with one change (excluded from timing)
    op_id, deg, asg = seq[0]
    _, ch = ps.update_task_graph(tg, g, topo, op_id, ps.ParallelizationConfig(dict(deg), asg))
    ps.delta_simulate(tg, ch)
    out = []
    t0 = time.perf_counter()
    for op_id, deg, asg in seq[1:]:
        _, ch = ps.update_task_graph(tg, g, topo, op_id, ps.ParallelizationConfig(dict(deg), asg))
        out.append(ps.delta_simulate(tg, ch).makespan)
    return out, time.perf_counter() - t0


def run_reference(g_json, topo_json, start_json, seq, mode, limit):
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    import parasim as ref
    from parasim import formats as rf
    g = rf.graph_from_json(g_json)
    topo = rf.topology_from_json(topo_json)
    start = rf.strategy_from_json(start_json)
    prof = ref.CostProfile()
    tg = ref.build_task_graph(g, topo, start, prof, mode)
    ref.full_simulate(tg)
    op_id, deg, asg = seq[0]
    _, ch = ref.update_task_graph(tg, g, topo, op_id, ref.ParallelizationConfig(dict(deg), asg))
    ref.delta_simulate(tg, ch)
    out = []
    t0 = time.perf_counter()
    for op_id, deg, asg in seq[1:limit + 1]:
        _, ch = ref.update_task_graph(tg, g, topo, op_id, ref.ParallelizationConfig(dict(deg), asg))
        out.append(ref.delta_simulate(tg, ch).makespan)
    return out, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--changes", type=int, default=400)
    ap.add_argument("--ref-changes", type=int, default=40)
    ap.add_argument("--mode", default="full-iteration")
    args = ap.parse_args()
    import paper_1807_05358_b200 as ps
    from paper_1807_05358_b200 import formats
    g, topo, md = ps.inception_v3(), ps.multi_node_topology(4, 4), 4
    start = ps.random_strategy(g, topo, md, 1)
    seq = changes(g, topo, md, args.changes + 1, 5)
    ours, t_ours = run_ours(g, topo, start, seq, args.mode)
    line = {"what": "update_task_graph + delta_simulate per change, drop-in API",
            "workload": "Inception-v3 b64, 4x4 devices, " + args.mode + ", max degree 4, random start",
            "ours_changes": len(ours), "ours_ms_per_change": 1e3 * t_ours / len(ours)}
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "parasim")):
        ref, t_ref = run_reference(formats.graph_to_json(g), formats.topology_to_json(topo),
                                   formats.strategy_to_json(start), seq, args.mode, args.ref_changes)
        assert ref == ours[:len(ref)], "makespans differ from the reference"
        line.update({"reference_changes": len(ref), "reference_ms_per_change": 1e3 * t_ref / len(ref),
                     "speedup": (t_ref / len(ref)) / (t_ours / len(ours)), "identical_makespans": True})
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
