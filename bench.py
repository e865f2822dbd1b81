#!/usr/bin/env python3
"""Benchmark: simulated strategy evaluations/sec on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): Inception-v3 (125 ops, batch 64) on a
simulated 4-node x 4-GPU topology, full-iteration task graphs, max_degree 4,
1024 MCMC chains per GPU (weak scaling: each rank owns 1024 chains), initial
strategies [data-parallel] + random_strategy(seed=c), Philox stream.
A step = every chain makes ``--proposals`` Metropolis proposals, each scored
by a full GPU re-simulation of the changed strategy (one k_mcmc launch);
value = proposals (= strategy evaluations) of all ranks / max-over-ranks time.

Proposals are scored by checkpointed delta evaluation (the B200 form of the
reference's update_task_graph + delta_simulate); ``full_eval`` reports full
evaluations (build + full simulate, ``k_simulate_batch``) of the chains'
strategies beside it, and ``configs`` the other BASELINE configs (AlexNet,
ResNet-101 on 64 devices, NMT-40 on 64 devices, random DAGs of 1k / 10k ops)
with their own rooflines.

``--impl reference`` times the CPU restatement of the reference path
(oracle/parasim_oracle.c: rebuild + full simulate per proposal) on all host
threads, on a wall-clock-bounded sample of the same chains, rank 0 only; the
unmodified Python reference (baseline/_ref, ``mcmc_search(polish=False)`` over
a process pool) is timed beside it as ``python_reference`` when installed.
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
    ap.add_argument("--config", default="inception", choices=("inception", "alexnet", "resnet", "nmt", "random", "random1k", "random10k"))
    ap.add_argument("--ops", type=int, default=1000, help="operator count of the random-DAG config")
    ap.add_argument("--no-delta", action="store_true",
                    help="score every proposal from time zero instead of resuming from a snapshot")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-proposals", type=int, default=1000,
                    help="CPU arm: proposals per chain, the window the GPU chains cover in the default bench")
    ap.add_argument("--py-ref-seconds", type=float, default=8.0,
                    help="wall time of the Python-reference leg (0: skip)")
    ap.add_argument("--extra", default="inception-forward,alexnet,resnet,nmt,random1k,random10k",
                    help="other BASELINE configs measured after the headline ('none': skip)")
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
    if name.startswith("random") and name[6:].rstrip("k").isdigit():
        ops = int(name[6:].rstrip("k")) * (1000 if name.endswith("k") else 1)
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


def cpu_baseline(g, topo, prof, mode, md, init, seeds, seconds, threads, proposals=1000, first=0):
    """The oracle (CPU restatement of the reference path) on a bounded sample of
    the GPU workload: the same chains (starts and seeds, from chain `first` on),
    each running the same window of `proposals` proposals from its start that the
    GPU chains run in the bench (chains slow down as their strategies evolve, so
    the window matters), `threads` chains at a time on all host threads, until
    `seconds` have passed (each chain also stops at that deadline)."""
    from oracle.oracle_io import Oracle
    try:  # (a process that initialised CUDA may have been pinned to the GPU's NUMA node)
        before = len(os.sched_getaffinity(0))
        os.sched_setaffinity(0, range(os.cpu_count() or 1))
        if os.environ.get("PS_BENCH_VERBOSE"):
            print(f"cpu_baseline: affinity {before} -> {len(os.sched_getaffinity(0))} cpus", file=sys.stderr)
    except (AttributeError, OSError):
        pass
    orc = Oracle()
    t0 = time.perf_counter()
    evals = props = done = 0
    c = first
    while done == 0 or time.perf_counter() - t0 < seconds:
        batch = [(c + j) % len(init) for j in range(threads)]
        left = seconds - (time.perf_counter() - t0)
        out = orc.mcmc(g, topo, prof, mode, [init[i] for i in batch], [seeds[i] for i in batch], proposals, md,
                       rng_mode="philox", threads=threads, deadline_s=max(0.05, left))
        p = float(out["summary"][:, 2].sum())
        props += p
        evals += p + len(batch)  # (the initial full evaluation of each chain counts too)
        done += len(batch)
        c += len(batch)
    dt = time.perf_counter() - t0
    return {"value": evals / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"{done} chains (from chain {first}) x up to {proposals} proposals each, the GPU chains' "
                       f"window ({props / done:.0f} on average; {mode}, rebuild + full simulate per proposal), "
                       f"{threads} at a time, {dt:.1f}s"),
            "next_chain": c}


def _py_ref_chain(job):
    """One chain of the unmodified reference (baseline/_ref): mcmc_search with
    a single initial strategy, seed 1000003*c (its chain-c seed), polish off."""
    ref_path, g_json, topo_json, s_json, seed, mode, md, seconds = job
    sys.path.insert(0, ref_path)
    import parasim
    from parasim import formats as rf
    g, topo = rf.graph_from_json(g_json), rf.topology_from_json(topo_json)
    params = parasim.SearchParams(budget_seconds=seconds, seed=seed, max_degree=md, mode=mode, polish=False,
                                  initial=[rf.strategy_from_json(s_json)], stagnation_floor=1e9)
    t0 = time.perf_counter()
    rep = parasim.mcmc_search(g, topo, parasim.CostProfile(), params)
    return rep.proposals + 1, time.perf_counter() - t0


def python_reference(g, topo, mode, md, init, seconds, procs):
    """The reference's own Python path: mcmc_search(polish=False),
    one chain per process over all host cores, wall-clock bounded by its own
    budget rule; evaluations = proposals + the initial full simulation."""
    ref_path = os.path.join(ROOT, "baseline", "_ref")
    if seconds <= 0 or not os.path.isdir(os.path.join(ref_path, "parasim")):
        return None
    import multiprocessing as mproc
    from paper_1807_05358_b200 import formats
    gj, tj = formats.graph_to_json(g), formats.topology_to_json(topo)
    n = min(len(init), procs)
    jobs = [(ref_path, gj, tj, formats.strategy_to_json(init[c]), 1000003 * c, mode, md, seconds) for c in range(n)]
    t0 = time.perf_counter()
    with mproc.get_context("spawn").Pool(n) as pool:
        res = pool.map(_py_ref_chain, jobs)
    wall = time.perf_counter() - t0
    evals = sum(e for e, _ in res)
    busy = max(t for _, t in res)
    return {"value": evals / busy, "unit": UNIT, "cores": n, "kind": "reference (unmodified Python, baseline/_ref)",
            "sample": (f"{n} chains, mcmc_search(polish=False, budget_seconds={seconds:g}) one per process, "
                       f"{evals} evaluations in {busy:.1f}s of search ({wall:.1f}s with process start-up)")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_1807_05358_b200 as ps
    g, topo, md, desc = workload(args.config, args.ops)
    prof = ps.CostProfile()
    threads = os.cpu_count() or 1
    C = args.chains
    init = initial_strategies(g, topo, md, 0, C)
    seeds = [1000003 * c for c in range(C)]
    vals = []
    nxt = 0
    for i in range(args.warmup + args.steps):
        # warm-up steps are short (1 s); timed steps are wall-clock-bounded samples
        # that continue through the chain list
        secs = 1.0 if i < args.warmup else max(2.0, args.cpu_seconds / 2)
        res = cpu_baseline(g, topo, prof, args.mode, md, init, seeds, secs, threads,
                           proposals=args.ref_proposals, first=nxt)
        nxt = res.pop("next_chain")
        if i >= args.warmup:
            vals.append(res["value"])
    v = statistics.mean(vals)
    py = python_reference(g, topo, args.mode, md, init, args.py_ref_seconds, threads)
    if py is not None:
        res = {**res, "python_reference": py}
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": desc, "mode": args.mode, "max_degree": md, "chains": len(init),
                       "proposals_per_chain": args.ref_proposals},
            "cpu_baseline": {**res, "value": v},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


class Chains:
    """One MCMC handle over C chains of a workload, set up through the C ABI."""

    def __init__(self, name, mode, C, first, delta, device, ops=1000, distinct=None):
        import paper_1807_05358_b200 as ps
        from paper_1807_05358_b200 import _native as nat
        from paper_1807_05358_b200.lowering import lower
        from paper_1807_05358_b200.search import fit_capacity
        self.ps, self.nat, self.L = ps, nat, nat.lib()
        g, topo, md, desc = workload(name, ops)
        self.g, self.topo, self.md, self.desc, self.mode, self.C = g, topo, md, desc, mode, C
        self.prof = ps.CostProfile()
        if distinct is None:
            init = initial_strategies(g, topo, md, first, C)
            starts = init
        else:
            # very large graphs: `distinct` starts (DP + random) tiled over the
            # chains; every chain still has its own Philox stream
            starts = initial_strategies(g, topo, md, 0, distinct)
            init = [starts[i % distinct] for i in range(C)]
        self.init = init
        # every rank lowers the same map set (the data-parallel start's maps first), so
        # encoded strategies mean the same thing on every GPU for the final exchange
        low = lower(g, topo, self.prof, mode, max_degree=md,
                    strategies=[ps.data_parallel_strategy(g, topo)] + list(starts), device=device)
        maps = np.zeros((C, low.n_ops), dtype=np.int32)
        asg = np.zeros((C, low.n_slots), dtype=np.uint8)
        enc = {}
        for i, s in enumerate(init):
            if id(s) not in enc:
                enc[id(s)] = low.encode(s)
            maps[i], asg[i] = enc[id(s)]
        n_fit = C if distinct is None else distinct
        low = fit_capacity(low, maps[:n_fit], asg[:n_fit])  # ready-set capacity from a pilot evaluation
        self.low, self.maps, self.asg = low, maps, asg
        self.seeds = np.array([1000003 * (first + i) for i in range(C)], dtype=np.uint64)
        self.mp = nat.PsMcmcParams(nat.PS_RNG_PHILOX, 0, 0.0, math.log(10.0), 0, 0, 1 if delta else 0)
        self.h = self.create(maps, asg, self.seeds)

    def create(self, maps, asg, seeds):
        nat = self.nat
        h = ctypes.c_void_p()
        nat.check(self.L.ps_mcmc_create(self.low.handle(), ctypes.byref(self.mp), self.C, nat.ptr(maps), nat.ptr(asg),
                                        nat.ptr(seeds), None, ctypes.byref(h)), "ps_mcmc_create")
        return h

    def step(self, h, stream_handle, budget_ns, proposals):
        nat = self.nat
        if budget_ns:
            nat.check(self.L.ps_mcmc_run_budget(h, 1 << 30, budget_ns, stream_handle), "ps_mcmc_run_budget")
        else:
            nat.check(self.L.ps_mcmc_run(h, proposals, stream_handle), "ps_mcmc_run")

    def summary(self, h=None):
        s = (self.nat.PsChainSummary * self.C)()
        self.nat.check(self.L.ps_mcmc_read(h or self.h, s, None, None, None, None), "ps_mcmc_read")
        return s

    def state(self):
        sm = np.zeros((self.C, self.low.n_ops), dtype=np.int32)
        sa = np.zeros((self.C, self.low.n_slots), dtype=np.uint8)
        self.nat.check(self.L.ps_mcmc_read_state(self.h, self.nat.ptr(sm), self.nat.ptr(sa)), "ps_mcmc_read_state")
        return sm, sa

    def bytes_per_eval(self, sm, sa, samples):
        """Algorithmic bytes per evaluation: 32 B per task + 4 B per dependency
        (SURVEY 8d), averaged over a sample of the chains' live strategies
        (traced on the GPU)."""
        from paper_1807_05358_b200.taskgraph import _bind
        te = []
        for i in range(0, self.C, max(1, self.C // samples)):
            tg = self.ps.TaskGraph(self.g, self.topo, self.low.decode(sm[i], sa[i]), self.prof, self.mode)
            _bind(tg, self.low)
            T = len(tg.tasks)
            E = sum(len(t.outputs) for t in tg.tasks.values())
            te.append((T, E))
        T_avg = statistics.mean(t for t, _ in te)
        E_avg = statistics.mean(e for _, e in te)
        return 32.0 * T_avg + 4.0 * E_avg, T_avg, E_avg

    def destroy(self):
        self.L.ps_mcmc_destroy(self.h)


def timed_steps(ch, h, stream, sh, steps, budget_ns, proposals, flush):
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a_, b_ in ev:
        a_.record(stream)
        ch.step(h, sh, budget_ns, proposals)
        b_.record(stream)
        flush.zero_()  # L2 flush between timed steps (outside the events)
    torch.cuda.synchronize()
    return [a_.elapsed_time(b_) for a_, b_ in ev]


EXTRA = {  # name: (chains, step budget ms, distinct starts or None, trace samples)
    "inception-forward": (1024, 100.0, None, 16),  # the headline workload in forward mode
    "alexnet": (1024, 100.0, None, 16),
    "resnet": (1024, 100.0, None, 8),
    "nmt": (4096, 300.0, 64, 4),
    "random1k": (4096, 300.0, 64, 4),
    "random10k": (4096, 2500.0, 16, 2),
}


def measure_extra(name, mode, device, stream, sh, flush, peak, steps=3, warmup=2):
    C, bms, distinct, samples = EXTRA[name]
    if name.endswith("-forward"):
        name, mode = name[:-len("-forward")], "forward"
    ch = Chains(name, mode, C, 0, True, device, distinct=distinct)
    budget_ns = int(bms * 1e6)
    for _ in range(warmup):
        ch.step(ch.h, sh, budget_ns, 0)
    import torch
    torch.cuda.synchronize()
    s0 = ch.summary()
    ms = timed_steps(ch, ch.h, stream, sh, steps, budget_ns, 0, flush)
    s1 = ch.summary()
    evals = sum(s.proposals for s in s1) - sum(s.proposals for s in s0)
    run = sum(s.rounds_run for s in s1) - sum(s.rounds_run for s in s0)
    reused = sum(s.rounds_reused for s in s1) - sum(s.rounds_reused for s in s0)
    sm, sa = ch.state()
    bpe, T, E = ch.bytes_per_eval(sm, sa, samples)
    info = ch.low.info()
    ch.destroy()
    v = evals / (sum(ms) / 1e3)
    achieved = bpe * v / 1e9
    return {"workload": ch.desc, "mode": mode, "max_degree": ch.md, "chains": C, "value": v, "unit": UNIT,
            "tasks_per_s": v * T, "ms_per_step": sum(ms) / steps, "steps": steps,
            "step": f"time-boxed {bms:g} ms", "tasks_per_eval": round(T, 1), "deps_per_eval": round(E, 1),
            "delta_reused_fraction": reused / max(1, run + reused),
            "failures": sum(1 for s in s1 if s.status != ch.nat.PS_STATUS_OK),
            "resident_warps_per_sm": info.resident_warps_per_sm, "ready_capacity": info.ready_capacity,
            "starts": "data-parallel + random" + (f" ({distinct} distinct, tiled)" if distinct else ""),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "note": f"B_eval = 32*T + 4*E = {bpe:.0f} B"}}


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1807_05358_b200 as ps
    from paper_1807_05358_b200 import _native as nat

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
    C = args.chains
    # weak scaling: C chains per rank, rank r owning the contiguous block
    # parallel.shard(r, world, world * C) = [r C, (r + 1) C) -- the same split the
    # API's SearchParams(devices=[...]) uses
    from paper_1807_05358_b200.parallel import shard
    blk = shard(rank, world, world * C)
    first = blk.start
    assert len(blk) == C
    ch = Chains(args.config, args.mode, C, first, not args.no_delta, local, ops=args.ops)
    L, low, g, topo, md, desc, prof = ch.L, ch.low, ch.g, ch.topo, ch.md, ch.desc, ch.prof
    info = low.info()
    stream = torch.cuda.current_stream(dev)
    sh = ctypes.c_void_p(stream.cuda_stream)
    P = args.proposals
    budget_ns = int(args.budget_ms * 1e6)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    # first launch also scores the initial strategies (warm-up)
    for _ in range(args.warmup):
        ch.step(ch.h, sh, budget_ns, P)
        flush.zero_()
    torch.cuda.synchronize(dev)
    sm, sa = ch.state()
    bytes_per_eval, T_avg, E_avg = ch.bytes_per_eval(sm, sa, 16)
    summ0 = ch.summary()
    props0 = sum(s.proposals for s in summ0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        step_ms = timed_steps(ch, ch.h, stream, sh, args.steps, budget_ns, P, flush)
    if world > 1:
        dist.barrier()
    total_ms = sum(step_ms)
    summ = ch.summary()
    evals = sum(s.proposals for s in summ) - props0
    rounds_run = sum(s.rounds_run for s in summ) - sum(s.rounds_run for s in summ0)
    rounds_reused = sum(s.rounds_reused for s in summ) - sum(s.rounds_reused for s in summ0)
    bad = sum(1 for s in summ if s.status != nat.PS_STATUS_OK)
    # best strategy across chains: device argmin, then the one cross-GPU exchange
    from paper_1807_05358_b200.parallel import global_best
    bc, bi = ctypes.c_double(), ctypes.c_int32()
    nat.check(L.ps_mcmc_best(ch.h, ctypes.byref(bc), ctypes.byref(bi)), "ps_mcmc_best")
    bm_all = np.zeros((C, low.n_ops), dtype=np.int32)
    ba_all = np.zeros((C, low.n_slots), dtype=np.uint8)
    nat.check(L.ps_mcmc_read(ch.h, None, nat.ptr(bm_all), nat.ptr(ba_all), None, None), "ps_mcmc_read")
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

    # ---- e2e: the C-ABI with host buffers, H2D of the step's inputs and D2H of
    # its results inside the timing.  Each step resumes the chains' warm live
    # strategies (read back after the timed region) on a fresh handle -- create
    # (H2D), one time-boxed segment, read summaries + best strategies (D2H) --
    # so it runs the same search phase as `value`, plus the handle set-up.
    e2e_times = []
    wm, wa = ch.state()

    def pinned(a):  # page-locked host copy (numpy view of pinned memory)
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        out = t.numpy()
        out[...] = a
        return out, t

    (pmaps, _t1), (pasg, _t2), (pseeds, _t3) = pinned(wm), pinned(wa), pinned(ch.seeds + np.uint64(7))
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
        h2 = ch.create(pmaps, pasg, pseeds)
        t1 = time.perf_counter()
        ch.step(h2, sh, budget_ns, P)
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
                   "evaluation": "delta (resume from a snapshot)" if not args.no_delta else "full re-simulation",
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
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "note": "per step: ps_mcmc_create from the warm chains' strategies (pinned host buffers), one "
                        "time-boxed segment, ps_mcmc_read of summaries + best strategies; the initial scoring "
                        "of each chain counts as an evaluation"},
        "gpu_launches": args.steps,
        "clocks": clocks.summary(),
        "delta": {"enabled": not args.no_delta, "rounds_run": int(rounds_run), "rounds_reused": int(rounds_reused),
                  "reused_fraction": rounds_reused / max(1, rounds_run + rounds_reused)},
        "evals_by_kind": {"delta_per_s": value if not args.no_delta else None, "full_per_s": full_value,
                          "note": "delta = MCMC proposals resumed from a snapshot (value); full = build + full "
                                  "simulation of given strategies (full_eval)"},
        "chain_failures": bad, "best_makespan": float(best.item()), "best_chain": win_chain,
        "full_eval": {"value": full_value, "unit": UNIT, "candidates_per_launch": FB, "failures": bad_full,
                      "note": "full evaluations (no search) of the chains' current strategies (8 adjacent copies each), "
                              "one k_simulate_batch launch per step, device-resident inputs"},
    }
    ch.destroy()
    extras = [x for x in args.extra.split(",") if x and x != "none"] if world == 1 else []
    if extras:
        line["configs"] = {}
        for name in extras:
            try:
                line["configs"][name] = measure_extra(name, args.mode, local, stream, sh, flush, peak)
            except Exception as exc:  # noqa: BLE001 - report, keep the headline
                line["configs"][name] = {"error": f"{type(exc).__name__}: {exc}"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        # the GPU chains' window: proposals per chain from their starts to the end of the timed steps
        window = max(1, round(sum(s.proposals for s in summ) / C))
        # (in a fresh process: this one holds a CUDA context and its runtime threads)
        import multiprocessing as mproc
        with mproc.get_context("spawn").Pool(1) as pool:
            # (a fresh profile: `prof` now caches every lowered map's analytic time, which
            # the oracle would take as explicit overrides and look up more slowly)
            line["cpu_baseline"] = pool.apply(cpu_baseline, (g, topo, ps.CostProfile(), args.mode, md, ch.init,
                                                             [1000003 * c for c in range(C)], args.cpu_seconds,
                                                             threads), {"proposals": window})
        line["cpu_baseline"].pop("next_chain", None)
        py = python_reference(g, topo, args.mode, md, ch.init, args.py_ref_seconds, threads)
        if py is not None:
            line["cpu_baseline"]["python_reference"] = py
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
