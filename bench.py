#!/usr/bin/env python3
"""Benchmark: simulated strategy evaluations/sec on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): Inception-v3 (125 ops, batch 64) on a
simulated 4-node x 4-GPU topology, full-iteration task graphs, max_degree 4,
1024 MCMC chains per GPU (weak scaling: each rank owns 1024 chains), initial
strategies [data-parallel] + random_strategy(seed=c), Philox stream.
A step = every chain makes ``--proposals`` Metropolis proposals, each scored
by a full GPU re-simulation of the changed strategy (one k_mcmc launch);
value = proposals (= strategy evaluations) of all ranks / max-over-ranks time.

``--impl reference`` times the CPU restatement of the reference path
(oracle/parasim_oracle.c: rebuild + full simulate per proposal) on all host
threads, on a bounded sample of the same chains, rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated strategy evals/sec (full+delta) at 1/2/4/8 B200 vs host-CPU ref"
UNIT = "evals/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--chains", type=int, default=1024, help="chains per GPU")
    ap.add_argument("--proposals", type=int, default=16, help="proposals per chain per step (--budget-ms 0)")
    ap.add_argument("--budget-ms", type=float, default=100.0,
                    help="time-boxed steps: each chain proposes until this much device time has passed")
    ap.add_argument("--mode", default="full-iteration", choices=("forward", "full-iteration"))
    ap.add_argument("--config", default="inception", choices=("inception", "alexnet", "resnet", "nmt", "random"))
    ap.add_argument("--ops", type=int, default=1000, help="operator count of the random-DAG config")
    ap.add_argument("--no-delta", action="store_true",
                    help="score every proposal from time zero instead of resuming from a snapshot")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def workload(name, ops=1000):
    import paper_1807_05358_b200 as ps
    if name == "inception":
        return ps.inception_v3(), ps.multi_node_topology(4, 4), 4, "Inception-v3 b64 on 4x4 GPUs (16 devices, 120 links)"
    if name == "alexnet":
        return ps.alexnet_like(), ps.single_node_topology(4), 4, "AlexNet-like on 1x4 GPUs"
    if name == "resnet":
        return ps.resnet101(), ps.multi_node_topology(16, 4), 8, "ResNet-101 b64 on 16x4 GPUs (64 devices)"
    if name == "nmt":
        return (ps.nmt_like(steps=40, layers=2, batch=64, hidden=1024, vocab=32768), ps.multi_node_topology(16, 4), 8,
                "NMT-40 on 16x4 GPUs")
    return ps.random_dag(ops, seed=1000), ps.multi_node_topology(4, 4), 4, f"random DAG {ops} ops on 4x4 GPUs"


def initial_strategies(g, topo, md, first, count):
    """[data_parallel] + [random_strategy(seed=c) for c in 1..]: chain c's start."""
    import paper_1807_05358_b200 as ps
    seeds = [c for c in range(first, first + count) if c != 0]
    rand = iter(ps.random_strategies(g, topo, md, seeds))
    return [ps.data_parallel_strategy(g, topo) if c == 0 else next(rand) for c in range(first, first + count)]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def profiled_traffic_per_eval():
    """DRAM bytes per evaluation of k_mcmc from the committed ncu capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh).get("k_mcmc_dram_bytes_per_eval")
    except Exception:
        return None


def cpu_baseline(g, topo, prof, mode, md, init, seeds, seconds, threads):
    """The oracle (CPU restatement of the reference path) on a bounded sample."""
    from oracle.oracle_io import Oracle
    orc = Oracle()
    n = min(len(init), threads)
    times = []
    for p in (1, 3):  # two calibration points: the slope is the per-proposal cost
        t0 = time.perf_counter()
        orc.mcmc(g, topo, prof, mode, init[:n], seeds[:n], p, md, rng_mode="philox", threads=threads)
        times.append(time.perf_counter() - t0)
    per_prop = max(1e-6, (times[1] - times[0]) / 2)
    props = max(2, int(seconds / per_prop))
    t0 = time.perf_counter()
    out = orc.mcmc(g, topo, prof, mode, init[:n], seeds[:n], props, md, rng_mode="philox", threads=threads)
    dt = time.perf_counter() - t0
    total = float(out["summary"][:, 2].sum())
    # the initial full evaluation of each chain is counted as an evaluation too
    evals = total + n
    return {"value": evals / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n} chains x {props} proposals ({mode}, rebuild+full simulate per proposal), {dt:.1f}s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_1807_05358_b200 as ps
    g, topo, md, desc = workload(args.config, args.ops)
    prof = ps.CostProfile()
    threads = os.cpu_count() or 1
    init = initial_strategies(g, topo, md, 0, threads)
    seeds = [1000003 * c for c in range(threads)]
    vals = []
    for i in range(args.warmup + args.steps):
        res = cpu_baseline(g, topo, prof, args.mode, md, init, seeds, max(2.0, args.cpu_seconds / 3), threads)
        if i >= args.warmup:
            vals.append(res["value"])
    v = statistics.mean(vals)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": desc, "mode": args.mode, "max_degree": md, "chains": len(init)},
            "cpu_baseline": {**res, "value": v},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1807_05358_b200 as ps
    from paper_1807_05358_b200 import _native as nat
    from paper_1807_05358_b200.lowering import lower
    from paper_1807_05358_b200.rng import mt_state_words  # noqa: F401

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PS_BENCH_BACKEND=gloo lets the N>1 path be exercised with ranks sharing one
    # GPU (a test hook; the driver's runs use NCCL, one rank per GPU)
    backend = os.environ.get("PS_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    g, topo, md, desc = workload(args.config, args.ops)
    prof = ps.CostProfile()
    C = args.chains
    first = rank * C
    init = initial_strategies(g, topo, md, first, C)
    from paper_1807_05358_b200.search import fit_capacity
    # every rank lowers the same map set (the data-parallel start's maps first), so
    # encoded strategies mean the same thing on every GPU for the final exchange
    low = lower(g, topo, prof, args.mode, max_degree=md, strategies=[ps.data_parallel_strategy(g, topo)] + init,
                device=local)
    L = nat.lib()
    maps = np.zeros((C, low.n_ops), dtype=np.int32)
    asg = np.zeros((C, low.n_slots), dtype=np.uint8)
    for i, s in enumerate(init):
        low.encode(s, maps[i], asg[i])
    low = fit_capacity(low, maps, asg)  # ready-set capacity from a pilot evaluation of the starts
    info = low.info()
    seeds = np.array([1000003 * (first + i) for i in range(C)], dtype=np.uint64)
    mp = nat.PsMcmcParams(nat.PS_RNG_PHILOX, 0, 0.0, math.log(10.0), 0, 0, 0 if args.no_delta else 1)
    h = ctypes.c_void_p()
    nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), C, nat.ptr(maps), nat.ptr(asg), nat.ptr(seeds), None,
                               ctypes.byref(h)), "ps_mcmc_create")
    stream = torch.cuda.current_stream(dev)
    sh = ctypes.c_void_p(stream.cuda_stream)
    P = args.proposals
    budget_ns = int(args.budget_ms * 1e6)

    def run_step(handle):
        if budget_ns:
            nat.check(L.ps_mcmc_run_budget(handle, 1 << 30, budget_ns, sh), "ps_mcmc_run_budget")
        else:
            nat.check(L.ps_mcmc_run(handle, P, sh), "ps_mcmc_run")

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    # first launch also scores the initial strategies (warm-up)
    for _ in range(args.warmup):
        run_step(h)
        flush.zero_()
    torch.cuda.synchronize(dev)
    # algorithmic bytes per evaluation: 32 B per task + 4 B per dependency, averaged
    # over a sample of the chains' live strategies (traced on the GPU)
    sm = np.zeros((C, low.n_ops), dtype=np.int32)
    sa = np.zeros((C, low.n_slots), dtype=np.uint8)
    nat.check(L.ps_mcmc_read_state(h, nat.ptr(sm), nat.ptr(sa)), "ps_mcmc_read_state")
    tasks_edges = []
    for i in range(0, C, max(1, C // 16)):
        tg = ps.TaskGraph(g, topo, low.decode(sm[i], sa[i]), prof, args.mode)
        from paper_1807_05358_b200.taskgraph import _bind
        _bind(tg, low)
        T = len(tg.tasks)
        E = sum(len(t.outputs) for t in tg.tasks.values())
        tasks_edges.append((T, E))
    T_avg = statistics.mean(t for t, _ in tasks_edges)
    E_avg = statistics.mean(e for _, e in tasks_edges)
    bytes_per_eval = 32.0 * T_avg + 4.0 * E_avg
    summ0 = (nat.PsChainSummary * C)()
    nat.check(L.ps_mcmc_read(h, summ0, None, None, None, None), "ps_mcmc_read")
    props0 = sum(s.proposals for s in summ0)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            starts[i].record(stream)
            run_step(h)
            ends[i].record(stream)
            flush.zero_()  # L2 flush between timed steps (outside the events)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    summ = (nat.PsChainSummary * C)()
    nat.check(L.ps_mcmc_read(h, summ, None, None, None, None), "ps_mcmc_read")
    evals = sum(s.proposals for s in summ) - props0
    rounds_run = sum(s.rounds_run for s in summ) - sum(s.rounds_run for s in summ0)
    rounds_reused = sum(s.rounds_reused for s in summ) - sum(s.rounds_reused for s in summ0)
    bad = sum(1 for s in summ if s.status != nat.PS_STATUS_OK)
    # best strategy across chains: device argmin, then the one cross-GPU exchange
    from paper_1807_05358_b200.parallel import global_best
    bc, bi = ctypes.c_double(), ctypes.c_int32()
    nat.check(L.ps_mcmc_best(h, ctypes.byref(bc), ctypes.byref(bi)), "ps_mcmc_best")
    bm_all = np.zeros((C, low.n_ops), dtype=np.int32)
    ba_all = np.zeros((C, low.n_slots), dtype=np.uint8)
    nat.check(L.ps_mcmc_read(h, None, nat.ptr(bm_all), nat.ptr(ba_all), None, None), "ps_mcmc_read")
    li = int(bi.value)
    win_cost, win_chain, win_map, win_asg = global_best(
        float(bc.value), first + li if li >= 0 else -1, bm_all[max(li, 0)], ba_all[max(li, 0)], device=dev)
    t_max = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    ev = torch.tensor([float(evals)], dtype=torch.float64, device=dev)
    best = torch.tensor([win_cost], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(ev, op=dist.ReduceOp.SUM)
    total_ms = float(t_max.item())
    all_evals = float(ev.item())
    value = all_evals / (total_ms / 1e3)

    # ---- e2e: the C-ABI with host buffers, H2D of the step's inputs and D2H of its results inside the timing
    e2e_times = []

    def pinned(a):  # page-locked host copy (numpy view of pinned memory)
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        out = t.numpy()
        out[...] = a
        return out, t

    (pmaps, _t1), (pasg, _t2), (pseeds, _t3) = pinned(maps), pinned(asg), pinned(seeds)
    h2d = pmaps.nbytes + pasg.nbytes + pseeds.nbytes
    best_maps, _t4 = pinned(np.zeros((C, low.n_ops), dtype=np.int32))
    best_asg, _t5 = pinned(np.zeros((C, low.n_slots), dtype=np.uint8))
    d2h = ctypes.sizeof(nat.PsChainSummary) * C + best_maps.nbytes + best_asg.nbytes
    e2e_evals = 0
    for i in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        h2 = ctypes.c_void_p()
        nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), C, nat.ptr(pmaps), nat.ptr(pasg), nat.ptr(pseeds),
                                   None, ctypes.byref(h2)), "ps_mcmc_create")
        t1 = time.perf_counter()
        run_step(h2)
        t2 = time.perf_counter()
        s2 = (nat.PsChainSummary * C)()
        nat.check(L.ps_mcmc_read(h2, s2, nat.ptr(best_maps), nat.ptr(best_asg), None, None), "ps_mcmc_read")
        dt = time.perf_counter() - t0
        if os.environ.get("PS_BENCH_VERBOSE"):
            print(f"e2e phases: create {1e3 * (t1 - t0):.2f} launch {1e3 * (t2 - t1):.2f} "
                  f"read {1e3 * (time.perf_counter() - t2):.2f} ms", file=sys.stderr)
        L.ps_mcmc_destroy(h2)
        if i >= args.warmup:
            e2e_times.append(dt)
            if os.environ.get("PS_BENCH_VERBOSE"):
                print(f"e2e step {i}: {dt * 1e3:.2f} ms", file=sys.stderr)
            # evaluations = the initial scoring of every chain + its proposals
            e2e_evals += sum(s.proposals for s in s2) + C
    e2e_t = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=dev)
    e2e_n = torch.tensor([float(e2e_evals)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(e2e_n, op=dist.ReduceOp.SUM)
    e2e_value = float(e2e_n.item()) / float(e2e_t.item())

    # ---- full evaluation (build + full simulate, no search): the chains' current
    # strategies scored in one k_simulate_batch launch per step, device-resident
    # (8 candidates per chain and launch, so the launch is not paced by its slowest candidate)
    FB = 8 * C
    fmaps = torch.from_numpy(np.repeat(sm, 8, axis=0)).to(dev)
    fasg = torch.from_numpy(np.repeat(sa, 8, axis=0)).to(dev)
    fmk = torch.empty(FB, dtype=torch.float64, device=dev)
    fst = torch.empty(FB, dtype=torch.int32, device=dev)

    def full_step():
        nat.check(L.ps_simulate_batch(low.handle(), ctypes.c_void_p(fmaps.data_ptr()), ctypes.c_void_p(fasg.data_ptr()),
                                      FB, ctypes.c_void_p(fmk.data_ptr()), ctypes.c_void_p(fst.data_ptr()),
                                      nat.PS_DEVICE_PTRS, sh), "ps_simulate_batch")

    for _ in range(args.warmup):
        full_step()
    torch.cuda.synchronize(dev)
    fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a_, b_ in fev:
        a_.record(stream)
        full_step()
        b_.record(stream)
        flush.zero_()  # L2 flush between timed steps (outside the events)
    torch.cuda.synchronize(dev)
    f_ms = torch.tensor([sum(a_.elapsed_time(b_) for a_, b_ in fev)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(f_ms, op=dist.ReduceOp.MAX)
    full_value = world * FB * args.steps / (float(f_ms.item()) / 1e3)
    bad_full = int((fst != nat.PS_STATUS_OK).sum().item())

    peak, peak_src = measured_peak()
    achieved = bytes_per_eval * (evals / (total_ms / 1e3)) / 1e9  # this rank's kernel, GB/s
    tpe = profiled_traffic_per_eval()
    traffic = tpe * evals / args.steps if tpe is not None else None  # DRAM bytes per k_mcmc launch
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "mode": args.mode, "max_degree": md, "chains_per_gpu": C,
                   "step": (f"time-boxed: every chain proposes for {args.budget_ms:g} ms of device time"
                            if budget_ns else f"{P} proposals per chain"),
                   "proposals_per_step": round(evals / args.steps, 1),
                   "rng": "philox", "l2": "flushed between steps (256 MB write)",
                   "tasks_per_eval": round(T_avg, 1), "deps_per_eval": round(E_avg, 1),
                   "ready_capacity": info.ready_capacity, "overlap_entries": info.n_entries,
                   "shared_counters": info.shared_counters, "resident_warps_per_sm": info.resident_warps_per_sm,
                   "warps_per_block": info.warps_per_block},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "note": (f"B_eval = 32*T + 4*E = {bytes_per_eval:.0f} B per evaluation (SURVEY 8d), "
                              f"{evals / args.steps:.0f} evaluations per launch; peak {peak_src}; "
                              "traffic from profiles/traffic.json (ncu)")},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": args.steps,
        "clocks": clocks.summary(),
        "delta": {"enabled": not args.no_delta, "rounds_run": int(rounds_run), "rounds_reused": int(rounds_reused),
                  "reused_fraction": rounds_reused / max(1, rounds_run + rounds_reused)},
        "chain_failures": bad, "best_makespan": float(best.item()), "best_chain": win_chain,
        "full_eval": {"value": full_value, "unit": UNIT, "candidates_per_launch": FB, "failures": bad_full,
                      "note": "full evaluations (no search) of the chains' current strategies (8 adjacent copies each), "
                              "one k_simulate_batch launch per step, device-resident inputs"},
    }
    L.ps_mcmc_destroy(h)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        line["cpu_baseline"] = cpu_baseline(g, topo, prof, args.mode, md, init, [1000003 * c for c in range(C)],
                                            args.cpu_seconds, threads)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
