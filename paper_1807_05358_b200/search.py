"""Strategy search: the reference's ``parasim.search`` API on the GPU path.

``mcmc_search`` runs every chain at once, one warp per chain (``k_mcmc``),
instead of one after another (reference search.py:193): chain c keeps the
reference's own seed ``params.seed + 1000003*c`` and, by default, CPython's
MT19937 stream for it, so each chain replays the unmodified reference's
proposals, accept/reject decisions, trace and best strategy
(``rng="philox"`` selects the shared counter-based stream of :mod:`.rng`).
A rejected proposal costs nothing to roll back: the chain's fragment (one
degree-map index and that op's devices) is restored in place.

The polish step and the local-optimality probe scan single-op neighbours in
the reference's enumeration order, evaluated in GPU batches, and keep the
reference's first-improvement semantics exactly (search.py:130-167,408-438).
"""

from __future__ import annotations

import ctypes
import logging
import math
import random
import time
from dataclasses import dataclass, field
from itertools import islice, product

import numpy as np

from . import _native as nat
from .cost import CostProfile
from .graph import DeviceTopology, OperatorGraph
from .lowering import MODE_FORWARD, degree_tuple, lower
from .partition import (ParallelizationConfig, ParallelizationStrategy, data_parallel_strategy,
                        enumerate_configs, output_region, random_strategy)
from .parallel import shard
from .rng import RNG_MT19937, RNG_PHILOX, mt_state_words

__all__ = [
    "SearchParams", "SearchReport", "ChainSummary", "SearchError", "SearchSpaceTooLarge",
    "ExhaustiveResult", "accept_probability", "accept", "propose", "mcmc_search",
    "exhaustive_optimal", "local_optimality_check", "evaluate_strategies",
]

_logger = logging.getLogger(__name__)


class SearchError(RuntimeError):
    pass


class SearchSpaceTooLarge(RuntimeError):
    pass


@dataclass
class SearchParams:
    budget_seconds: float | None = None
    max_proposals: int | None = None
    beta: float | None = None
    max_degree: int = 4
    seed: int = 0
    initial: list | None = None
    mode: str = MODE_FORWARD
    stagnation_floor: float = 2.0
    check_interval: int = 0
    polish: bool = True
    polish_cap: float = 2e5
    # B200 path knobs (new, optional)
    rng: str = RNG_MT19937          # "mt19937" replays the reference; "philox" = shared Philox stream
    segment: int = 256              # proposals per kernel launch between host checks
    device: int = 0
    delta: bool = True              # checkpointed delta evaluation of proposals (same results; faster)
    devices: list | None = None     # GPUs to shard the chains over (contiguous blocks; None: [device])


@dataclass
class ChainSummary:
    index: int
    initial_cost: float
    best_cost: float
    proposals: int
    accepted: int
    beta: float
    termination: str


@dataclass
class SearchReport:
    best_strategy: ParallelizationStrategy
    best_cost: float
    trace: list = field(default_factory=list)
    proposals: int = 0
    termination: str = "budget"
    chains: list = field(default_factory=list)


def accept_probability(cost_s: float, cost_s_star: float, beta: float) -> float:
    """min(1, exp(beta * (cost_s - cost_s_star))) (reference search.py:89-93)."""
    return 1.0 if cost_s_star <= cost_s else math.exp(beta * (cost_s - cost_s_star))


def accept(cost_s: float, cost_s_star: float, beta: float, rng: random.Random) -> bool:
    """Draws rng.random() only when the move is uphill (search.py:96-98)."""
    p = accept_probability(cost_s, cost_s_star, beta)
    return p >= 1.0 or rng.random() < p


def _propose_change(strategy, g, topo, max_degree, rng, config_cache):
    """Uniform op, uniform degree map, uniform device per task (search.py:101-115)."""
    op_id = rng.choice(sorted(g.ops))
    choices = config_cache.get(op_id)
    if choices is None:
        choices = config_cache[op_id] = enumerate_configs(g.ops[op_id], topo, max_degree)
    picked = rng.choice(choices)
    devices = topo.device_ids()
    return op_id, ParallelizationConfig(dict(picked.degrees),
                                        tuple(rng.choice(devices) for _ in range(picked.size())))


def propose(strategy: ParallelizationStrategy, g: OperatorGraph, topo: DeviceTopology, max_degree: int,
            rng: random.Random) -> ParallelizationStrategy:
    op_id, cfg = _propose_change(strategy, g, topo, max_degree, rng, {})
    out = strategy.copy()
    out.configs[op_id] = cfg
    return out


# -----------------------------------------------------------------------------
# batched evaluation

def evaluate_strategies(g: OperatorGraph, topo: DeviceTopology, profile: CostProfile, strategies,
                        mode: str = MODE_FORWARD, max_degree: int | None = None, low=None,
                        devices: list | None = None) -> np.ndarray:
    """Makespans of many strategies in one GPU launch (ps_simulate_batch), or
    one launch per GPU of ``devices`` over contiguous blocks of the list.
    Raises like build_task_graph for the first failing strategy."""
    from .taskgraph import TaskGraph, _bind, _check_config, _raise_status
    strategies = list(strategies)
    for s in strategies:
        for oid in sorted(g.ops):
            _check_config(g, topo, oid, s.configs[oid])
    if devices and len(devices) > 1 and len(strategies) > 1:
        from concurrent.futures import ThreadPoolExecutor
        parts = [list(shard(r, len(devices), len(strategies))) for r in range(len(devices))]
        jobs = [(d, p) for d, p in zip(devices, parts) if p]

        def one(job):
            d, part = job
            sub = [strategies[i] for i in part]
            lw = lower(g, topo, profile, mode, max_degree=max_degree, strategies=sub, device=d)
            return evaluate_strategies(g, topo, profile, sub, mode=mode, max_degree=max_degree, low=lw)

        with ThreadPoolExecutor(max_workers=len(jobs)) as pool:
            return np.concatenate(list(pool.map(one, jobs)))
    if devices and low is None:
        low = lower(g, topo, profile, mode, max_degree=max_degree, strategies=strategies, device=devices[0])
    if low is None or not all(low.has_maps_for(s) for s in strategies):
        low = lower(g, topo, profile, mode, max_degree=max_degree, strategies=strategies)
    n = len(strategies)
    maps = np.zeros((n, low.n_ops), dtype=np.int32)
    asg = np.zeros((n, low.n_slots), dtype=np.uint8)
    for i, s in enumerate(strategies):
        low.encode(s, maps[i], asg[i])
    return _eval_encoded(low, maps, asg, strategies)


def _eval_encoded(low, maps, asg, strategies=None, with_status=False):
    """Makespans of encoded strategies.  Raises like build_task_graph for the
    first failing one, or (``with_status``) returns (makespans, status, low)."""
    n = maps.shape[0]
    mk = np.zeros(n, dtype=np.float64)
    st = np.zeros(n, dtype=np.int32)
    while True:
        nat.check(nat.lib().ps_simulate_batch(low.handle(), nat.ptr(maps), nat.ptr(asg), n, nat.ptr(mk),
                                              nat.ptr(st), nat.PS_HOST_PTRS, None), "ps_simulate_batch")
        if not np.any(st == nat.PS_STATUS_CAPACITY):
            break
        low = _regrow(low)  # a ready set outgrew its shared-memory capacity: 4x capacity
    if with_status:
        return mk, st, low
    bad = np.nonzero(st)[0]
    if bad.size:
        i = int(bad[0])
        _raise_for(low, maps[i], asg[i], int(st[i]), strategies[i] if strategies is not None else None)
    return mk


def _raise_for(low, map_local, assign, status, strategy=None):
    from .taskgraph import TaskGraph, _bind, _raise_status
    strat = strategy if strategy is not None else low.decode(map_local, assign)
    tg = TaskGraph(low.graph, low.topology, strat, low.profile, low.mode)
    _bind(tg, low)
    _raise_status(tg, status)


def fit_capacity(low, maps, asg, headroom: int = 1):
    """A problem whose ready-set capacity fits the given candidates with
    ``headroom``x margin (chains wander; the data-parallel start is usually the
    widest): evaluates them, regrowing 4x on overflow."""
    cur = low
    n = maps.shape[0]
    mk = np.zeros(n, dtype=np.float64)
    st = np.zeros(n, dtype=np.int32)
    while True:
        nat.check(nat.lib().ps_simulate_batch(cur.handle(), nat.ptr(maps), nat.ptr(asg), n, nat.ptr(mk),
                                              nat.ptr(st), nat.PS_HOST_PTRS, None), "ps_simulate_batch")
        if not np.any(st == nat.PS_STATUS_CAPACITY):
            break
        cur = _regrow(cur)
    if headroom > 1:
        import copy
        cur = copy.copy(cur)
        cur._handle = None
        cur.ready_capacity = cur.ready_capacity * headroom
    return cur


def _regrow(low):
    """The same lowered problem with a 4x larger ready-set capacity (identical
    map tables, so encoded strategies stay valid)."""
    import copy
    new = copy.copy(low)
    new._handle = None
    new.ready_capacity = low.ready_capacity * 4
    return new


# -----------------------------------------------------------------------------
# MCMC

def _chain_error_text(exc: Exception) -> str:
    return f"error: {exc}"


def mcmc_search(g: OperatorGraph, topo: DeviceTopology, profile: CostProfile,
                params: SearchParams) -> SearchReport:
    """Metropolis-Hastings over single-op config changes, one GPU warp per
    chain (reference search.py:170-271)."""
    from .taskgraph import NoRouteError, TaskGraph, _bind, _check_config, _first_missing_route
    if params.budget_seconds is None and params.max_proposals is None:
        raise ValueError("SearchParams needs budget_seconds or max_proposals")
    initial = params.initial
    if initial is None:
        initial = [data_parallel_strategy(g, topo), random_strategy(g, topo, params.max_degree, params.seed)]
    g.topological_order()
    n = len(initial)
    start_err: dict[int, str] = {}
    live = []
    for ci, s0 in enumerate(initial):
        try:
            for oid in sorted(g.ops):
                if oid not in s0.configs:
                    raise KeyError(oid)
                _check_config(g, topo, oid, s0.configs[oid])
            live.append(ci)
        except Exception as exc:  # noqa: BLE001 - same isolation as the reference
            start_err[ci] = _chain_error_text(exc)
    summaries: list[ChainSummary | None] = [None] * n
    traces: list[list] = [[] for _ in range(n)]
    best: dict[int, tuple[float, ParallelizationStrategy]] = {}
    if live:
        devices = list(params.devices) if params.devices else [params.device]
        shards = [[live[i] for i in shard(r, len(devices), len(live))] for r in range(len(devices))]
        jobs = [(d, part) for d, part in zip(devices, shards) if part]

        def run_shard(device, part):
            # every shard lowers the same map set (all live starts), so an
            # encoded strategy means the same thing on every GPU
            low = lower(g, topo, profile, params.mode, max_degree=params.max_degree,
                        strategies=[initial[c] for c in live], device=device)
            while True:
                summ_d: list = [None] * n
                tr_d: list = [[] for _ in range(n)]
                best_d: dict = {}
                err_d: dict = {}
                if _run_chains(low, params, initial, part, summ_d, tr_d, best_d, err_d):
                    return summ_d, tr_d, best_d, err_d
                low = _regrow(low)  # some chain's ready set outgrew shared memory: rerun, same streams

        if len(jobs) == 1:
            results = [run_shard(*jobs[0])]
        else:
            # one host thread per GPU (ctypes drops the GIL inside every call);
            # the shards share nothing until the merge below
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(max_workers=len(jobs)) as pool:
                results = list(pool.map(lambda j: run_shard(*j), jobs))
        summaries = [None] * n
        traces = [[] for _ in range(n)]
        best = {}
        for (_, part), (summ_d, tr_d, best_d, err_d) in zip(jobs, results):
            for ci in part:
                summaries[ci], traces[ci] = summ_d[ci], tr_d[ci]
                if ci in best_d:
                    best[ci] = best_d[ci]
            start_err.update(err_d)
    for ci, msg in start_err.items():
        if summaries[ci] is None:
            _logger.warning("chain %d failed to start: %s", ci, msg[len("error: "):])
            summaries[ci] = ChainSummary(ci, math.inf, math.inf, 0, 0, 0.0, msg)
    trace: list = []
    iteration = 0
    best_overall = None
    for ci in range(n):
        for cand, ok in traces[ci]:
            iteration += 1
            trace.append((iteration, cand, ok))
        if ci in best and (best_overall is None or best[ci][0] < best_overall[0]):
            best_overall = (best[ci][0], best[ci][1], ci, summaries[ci].termination)
    if best_overall is None:
        raise SearchError("every chain failed")
    best_cost, best_strategy, _, termination = best_overall
    if params.polish:
        best_cost, best_strategy = _greedy_descend(g, topo, profile, best_strategy, best_cost, params)
    return SearchReport(best_strategy=best_strategy, best_cost=best_cost, trace=trace,
                        proposals=sum(c.proposals for c in summaries), termination=termination,
                        chains=list(summaries))


def _run_chains(low, params, initial, live, summaries, traces, best, start_err) -> bool:
    """Runs the chains; False if a chain hit the ready-set capacity (caller regrows)."""
    from .taskgraph import NoRouteError, TaskGraph, _bind, _first_missing_route
    L = nat.lib()
    n = len(live)
    maps = np.zeros((n, low.n_ops), dtype=np.int32)
    asg = np.zeros((n, low.n_slots), dtype=np.uint8)
    for i, ci in enumerate(live):
        low.encode(initial[ci], maps[i], asg[i])
    seeds = np.array([(params.seed + 1000003 * ci) for ci in live], dtype=object)
    seeds_u64 = np.array([int(s) % (1 << 64) for s in seeds], dtype=np.uint64)
    rng_mode = nat.PS_RNG_PHILOX if params.rng == RNG_PHILOX else nat.PS_RNG_MT19937
    mt = None
    if rng_mode == nat.PS_RNG_MT19937:
        mt = np.zeros((n, 625), dtype=np.uint32)
        for i, s in enumerate(seeds):
            words, pos = mt_state_words(int(s))
            mt[i, :624] = words
            mt[i, 624] = pos
    deterministic = params.budget_seconds is None
    cap = int(params.max_proposals) if params.max_proposals is not None else 0
    seg = max(1, int(params.segment))
    if params.check_interval:
        seg = min(seg, int(params.check_interval)) if not deterministic else int(params.check_interval)
    # the device keeps a ring of `record` proposals per chain: every proposal of a
    # fixed-length search, or one segment of a time-boxed one (read after each)
    record = cap if deterministic else seg
    mp = nat.PsMcmcParams(rng_mode, params.beta is not None, float(params.beta or 0.0), math.log(10.0),
                          1 if record else 0, record, 1 if params.delta else 0)
    h = ctypes.c_void_p()
    nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), n, nat.ptr(maps), nat.ptr(asg), nat.ptr(seeds_u64),
                               nat.ptr(mt) if mt is not None else None, ctypes.byref(h)), "ps_mcmc_create")
    summ = (nat.PsChainSummary * n)()
    term = ["budget"] * n
    seg_trace: list[list] = [[] for _ in range(n)]
    try:
        if deterministic:
            done = 0
            while True:
                step = min(cap - done, seg) if cap else 0
                nat.check(L.ps_mcmc_run(h, step, None), "ps_mcmc_run")
                done += step
                if params.check_interval and step == seg:
                    _verify_chains(low, h, n, live, summ)
                if done >= cap:
                    break
            term = ["proposal-limit"] * n
        else:
            t0 = time.monotonic()
            last_best = np.full(n, np.inf)
            last_improve = np.full(n, t0)
            stopped = np.zeros(n, dtype=bool)
            copied = np.zeros(n, dtype=np.int64)
            tc = np.zeros((n, record), dtype=np.float64)
            tok = np.zeros((n, record), dtype=np.uint8)
            while True:
                step = seg
                if cap:
                    live_props = [summ[i].proposals for i in range(n) if not stopped[i]]
                    step = min(step, cap - int(max(live_props, default=0)))
                remaining = params.budget_seconds - (time.monotonic() - t0)
                if step > 0 and remaining > 0:
                    # a time-boxed segment: chains stop between proposals once the
                    # remaining budget is spent (device clock), so a short budget
                    # does not overrun by a whole segment
                    nat.check(L.ps_mcmc_run_budget(h, step, max(1, int(remaining * 1e9)), None),
                              "ps_mcmc_run_budget")
                nat.check(L.ps_mcmc_read(h, summ, None, None, nat.ptr(tc), nat.ptr(tok)), "ps_mcmc_read")
                for i in range(n):
                    p = int(summ[i].proposals)
                    seg_trace[i].extend((float(tc[i, j % record]), bool(tok[i, j % record]))
                                        for j in range(int(copied[i]), p))
                    copied[i] = p
                if params.check_interval:
                    _verify_chains(low, h, n, live, summ)
                now = time.monotonic()
                halt = np.zeros(n, dtype=np.uint8)
                for i in range(n):
                    s = summ[i]
                    if s.best_cost < last_best[i]:
                        last_best[i] = s.best_cost
                        last_improve[i] = now
                    if stopped[i] or s.status != nat.PS_STATUS_OK:
                        continue
                    if cap and s.proposals >= cap:
                        term[i] = "proposal-limit"
                    elif now - t0 >= params.budget_seconds:
                        term[i] = "budget"
                    elif now - last_improve[i] > max((now - t0) / 2, params.stagnation_floor):
                        term[i] = "stagnation"
                    else:
                        continue
                    halt[i] = 1
                    stopped[i] = True
                if halt.any():
                    nat.check(L.ps_mcmc_stop(h, nat.ptr(halt)), "ps_mcmc_stop")
                if all(stopped[i] or summ[i].status != nat.PS_STATUS_OK for i in range(n)):
                    break
        bmaps = np.zeros((n, low.n_ops), dtype=np.int32)
        basg = np.zeros((n, low.n_slots), dtype=np.uint8)
        det_trace = deterministic and record
        tc = np.zeros((n, max(record, 1)), dtype=np.float64)
        tok = np.zeros((n, max(record, 1)), dtype=np.uint8)
        nat.check(L.ps_mcmc_read(h, summ, nat.ptr(bmaps), nat.ptr(basg), nat.ptr(tc) if det_trace else None,
                                 nat.ptr(tok) if det_trace else None), "ps_mcmc_read")
        if any(summ[i].status == nat.PS_STATUS_CAPACITY for i in range(n)):
            return False
        for i, ci in enumerate(live):
            s = summ[i]
            termination = term[i]
            if s.status == nat.PS_STATUS_NO_ROUTE:
                if s.proposals == 0 and not math.isfinite(s.initial_cost):
                    tg = TaskGraph(low.graph, low.topology, initial[ci].copy(), low.profile, low.mode)
                    _bind(tg, low)
                    a, b = _first_missing_route(tg) or ("?", "?")
                    start_err[ci] = f"error: {NoRouteError(f'no route between device {a} and device {b}')}"
                    continue
                # a proposal needed a missing link: the chain's live state holds it
                a, b = _proposal_route_error(low, h, i, int(s.last_op))
                termination = f"error: no route between device {a} and device {b}"
                _logger.warning("chain %d aborted after %d proposals: %s", ci, s.proposals, termination[7:])
            summaries[ci] = ChainSummary(ci, s.initial_cost, s.best_cost, int(s.proposals), int(s.accepted),
                                         s.beta, termination)
            if det_trace:
                k = min(int(s.proposals), record)
                traces[ci] = [(float(tc[i, j]), bool(tok[i, j])) for j in range(k)]
            elif not deterministic:
                traces[ci] = seg_trace[i]
            best[ci] = (s.best_cost, low.decode(bmaps[i], basg[i], template=initial[ci]))
    finally:
        L.ps_mcmc_destroy(h)
    return True


def _verify_chains(low, h, n, live, summ):
    """check_interval (search.py:242-249): every live chain's cached cost must
    equal a fresh evaluation of its current strategy."""
    L = nat.lib()
    nat.check(L.ps_mcmc_read(h, summ, None, None, None, None), "ps_mcmc_read")
    maps = np.zeros((n, low.n_ops), dtype=np.int32)
    asg = np.zeros((n, low.n_slots), dtype=np.uint8)
    nat.check(L.ps_mcmc_read_state(h, nat.ptr(maps), nat.ptr(asg)), "ps_mcmc_read_state")
    ok = [i for i in range(n) if summ[i].status == nat.PS_STATUS_OK]
    if not ok:
        return
    fresh = _eval_encoded(low, maps[ok], asg[ok])
    for j, i in enumerate(ok):
        if float(fresh[j]) != summ[i].cost:
            raise SearchError(f"chain {live[i]}: cached cost {summ[i].cost!r} diverged from fresh "
                              f"simulation {float(fresh[j])!r}")


def _proposal_route_error(low, h, i, op_rank):
    """Device pair the reference's update_task_graph would report for the
    failing proposal of chain i: predecessor pairs, successor pairs, then the
    op's rings (taskgraph.py:377-386).  The chain state still holds it."""
    from .taskgraph import TaskGraph, _bind, _first_missing_route
    L = nat.lib()
    n = h_chains = None
    maps = np.zeros((_mcmc_n(h), low.n_ops), dtype=np.int32)
    asg = np.zeros((_mcmc_n(h), low.n_slots), dtype=np.uint8)
    nat.check(L.ps_mcmc_read_state(h, nat.ptr(maps), nat.ptr(asg)), "ps_mcmc_read_state")
    strat = low.decode(maps[i], asg[i])
    tg = TaskGraph(low.graph, low.topology, strat, low.profile, low.mode)
    _bind(tg, low)
    op_id = low.ops[op_rank]
    g = low.graph
    order = [(p, op_id) for p in g.predecessors(op_id)] + [(op_id, s) for s in g.successors(op_id)]
    return _first_missing_route(tg, pair_order=order, sync_ops=[op_id]) or ("?", "?")


def _mcmc_n(h):
    return int(nat.lib().ps_mcmc_chains(h))


def _neighbours(g, topo, maps, devices, op_id, current):
    for m in maps[op_id]:
        for assignment in product(devices, repeat=m.size()):
            if m.degrees == current.degrees and assignment == current.assignment:
                continue
            yield ParallelizationConfig(dict(m.degrees), assignment)


def _neighbour_batch(low, op_id, base_m, base_a, cfgs, best):
    """Scores single-op neighbours in one GPU batch.  Returns the index of the
    first neighbour (in scan order) that improves on ``best`` -- with its cost
    -- or (None, None); a neighbour the reference's update_task_graph would fail
    on (a missing link) raises, but only when no improving neighbour precedes it
    (the reference scans sequentially and stops at whichever comes first)."""
    r = low.rank[op_id]
    off = int(low.slot_off[r])
    mm = np.repeat(base_m[None], len(cfgs), axis=0)
    aa = np.repeat(base_a[None], len(cfgs), axis=0)
    for j, (t, assignment) in enumerate(cfgs):
        mm[j, r] = low.map_index[r][t]
        for k, dev in enumerate(assignment):
            aa[j, off + k] = low.dev_index[dev]
    costs, st, low2 = _eval_encoded(low, mm, aa, with_status=True)
    hit = np.nonzero((st != nat.PS_STATUS_OK) | (costs < best))[0]
    if hit.size == 0:
        return None, None
    j = int(hit[0])
    if st[j] != nat.PS_STATUS_OK:
        _raise_for(low2, mm[j], aa[j], int(st[j]))
    return j, float(costs[j])


def _greedy_descend(g, topo, profile, strategy, cost, params, batch: int = 4096):
    """First-improvement hill climb (reference search.py:130-167) with each
    op's neighbour list evaluated in GPU batches.  A neighbour equal to the
    op's config at the time it is reached is skipped; after an improvement
    the scan resumes right after it against the updated strategy -- exactly
    the reference's sequential semantics."""
    maps = {oid: enumerate_configs(g.ops[oid], topo, params.max_degree) for oid in sorted(g.ops)}
    ndev = len(topo.devices)
    count = sum(ndev ** m.size() for oid in maps for m in maps[oid])
    if count > params.polish_cap:
        _logger.info("skipping final descent: %.3g neighbors exceed polish_cap %.3g", count, params.polish_cap)
        return cost, strategy
    devices = topo.device_ids()
    low = lower(g, topo, profile, params.mode, max_degree=params.max_degree, strategies=[strategy],
                device=params.device)
    current = strategy.copy()
    base_m, base_a = low.encode(current)
    best = float(_eval_encoded(low, base_m[None], base_a[None], [current])[0])
    improved = True
    while improved:
        improved = False
        for op_id in sorted(g.ops):
            op = g.ops[op_id]
            cur = current.configs[op_id]
            cur_key = (degree_tuple(op, cur.degrees), tuple(cur.assignment))
            full = [(degree_tuple(op, m.degrees), a, m) for m in maps[op_id]
                    for a in product(devices, repeat=m.size())]
            pos = 0
            while pos < len(full):
                stop = min(len(full), pos + batch)
                idx = [i for i in range(pos, stop) if (full[i][0], full[i][1]) != cur_key]
                if not idx:
                    pos = stop
                    continue
                base_m, base_a = low.encode(current)
                j, cost = _neighbour_batch(low, op_id, base_m, base_a, [(full[i][0], full[i][1]) for i in idx], best)
                if j is None:
                    pos = stop
                    continue
                i = idx[j]
                best = cost
                t, a, m = full[i]
                current.configs[op_id] = ParallelizationConfig(dict(m.degrees), a)
                cur_key = (t, a)
                improved = True
                pos = i + 1
    return best, ParallelizationStrategy(dict(current.configs))


# -----------------------------------------------------------------------------
# validation drivers

@dataclass
class ExhaustiveResult:
    strategy: ParallelizationStrategy
    cost: float
    visited: int
    space_estimate: float


def local_optimality_check(strategy: ParallelizationStrategy, g: OperatorGraph, topo: DeviceTopology,
                           profile: CostProfile, max_degree: int = 4, cap: float = 5e6, mode: str = MODE_FORWARD,
                           batch: int = 4096):
    """First strictly improving single-op neighbour, or None (search.py:408-438);
    neighbours are scored in GPU batches in the reference's scan order."""
    devices = topo.device_ids()
    ndev = len(devices)
    maps = {oid: enumerate_configs(g.ops[oid], topo, max_degree) for oid in sorted(g.ops)}
    count = sum(ndev ** m.size() for oid in maps for m in maps[oid])
    if count > cap:
        raise SearchSpaceTooLarge(f"{count:.3g} neighbors exceed cap {cap:.3g}")
    low = lower(g, topo, profile, mode, max_degree=max_degree, strategies=[strategy])
    base_m, base_a = low.encode(strategy)
    base = float(_eval_encoded(low, base_m[None], base_a[None], [strategy])[0])
    for op_id in sorted(g.ops):
        op = g.ops[op_id]
        cur = strategy.configs[op_id]
        gen = ((degree_tuple(op, m.degrees), a, m) for m in maps[op_id] for a in product(devices, repeat=m.size())
               if not (m.degrees == cur.degrees and a == cur.assignment))
        while True:
            chunk = list(islice(gen, batch))
            if not chunk:
                break
            j, cost = _neighbour_batch(low, op_id, base_m, base_a, [(t, a) for t, a, _ in chunk], base)
            if j is not None:
                t, a, m = chunk[j]
                return op_id, ParallelizationConfig(dict(m.degrees), a), cost
    return None


def _canonical_assignments(n: int, used: frozenset, devices_by_kind: dict):
    """Device tuples of length n up to renaming of still-unused same-kind devices:
    each slot takes an already-used device or the lowest-id unused device of
    some kind (reference search.py:285-306)."""
    def rec(i, used_now, prefix):
        if i == n:
            yield tuple(prefix)
            return
        options = sorted(used_now)
        for kind in sorted(devices_by_kind):
            fresh = next((d for d in devices_by_kind[kind] if d not in used_now), None)
            if fresh is not None:
                options.append(fresh)
        for d in options:
            prefix.append(d)
            yield from rec(i + 1, used_now | {d}, prefix)
            prefix.pop()

    yield from rec(0, used, [])


def _prefix_graph(g: OperatorGraph, ops: list) -> OperatorGraph:
    keep = set(ops)
    sub = OperatorGraph()
    for oid in ops:
        sub.ops[oid] = g.ops[oid]
    sub.tensors = [e for e in g.tensors if e.src in keep and e.dst in keep]
    return sub


def exhaustive_optimal(g: OperatorGraph, topo: DeviceTopology, profile: CostProfile, max_degree: int = 4,
                       cap: float = 1e9, mode: str = MODE_FORWARD) -> ExhaustiveResult:
    """Provably optimal strategy by depth-first branch and bound over canonical
    configs (reference search.py:321-405): ops in topological order; a node dies
    when its prefix makespan or the critical-path bound through the remaining
    ops reaches the incumbent.  The same nodes are visited in the same order;
    all children of a node are scored in one GPU batch (prefix makespan plus
    each op's earliest task end), then walked in order with the live incumbent."""
    from .taskgraph import TaskGraph, _bind, _raise_status
    order = g.topological_order()
    maps = {oid: enumerate_configs(g.ops[oid], topo, max_degree) for oid in order}
    ndev = len(topo.devices)
    estimate = 1.0
    for oid in order:
        estimate *= sum(ndev ** m.size() for m in maps[oid])
    if estimate > cap:
        raise SearchSpaceTooLarge(f"estimated search space of {estimate:.3g} strategies exceeds cap {cap:.3g}")
    devices_by_kind: dict = {}
    for dev_id in sorted(topo.devices):
        devices_by_kind.setdefault(topo.devices[dev_id].kind, []).append(dev_id)
    kind_devices = [topo.devices[ids[0]] for ids in devices_by_kind.values()]
    min_time = {}
    for oid in order:
        op = g.ops[oid]
        best_t = math.inf
        for m in maps[oid]:
            reg = output_region(op, ParallelizationConfig(m.degrees, None), 0)
            for dev in kind_devices:
                t = profile.task_exe_time(op, reg, dev)
                if t < best_t:
                    best_t = t
        min_time[oid] = best_t
    preds = {oid: g.predecessors(oid) for oid in order}
    lows: dict = {}

    def prefix_low(depth):
        low = lows.get(depth)
        if low is None:
            low = lows[depth] = lower(_prefix_graph(g, order[:depth]), topo, profile, mode, max_degree=max_degree)
        return low

    seed = data_parallel_strategy(g, topo)
    best_cost = float(evaluate_strategies(g, topo, profile, [seed], mode=mode)[0])
    best_strategy = seed
    configs: dict = {}
    visited = 0
    N = len(order)

    def score_children(depth, children):
        """(makespan, status, op min ends) of configs + each child, on the prefix of depth+1 ops."""
        low = prefix_low(depth + 1)
        k = len(children)
        mm = np.zeros((k, low.n_ops), dtype=np.int32)
        aa = np.zeros((k, low.n_slots), dtype=np.uint8)
        op_id = order[depth]
        for j, cfg in enumerate(children):
            configs[op_id] = cfg
            low.encode(ParallelizationStrategy(configs), mm[j], aa[j])
        mk = np.zeros(k, dtype=np.float64)
        st = np.zeros(k, dtype=np.int32)
        opmin = np.zeros((k, low.n_ops), dtype=np.float64)
        while True:
            nat.check(nat.lib().ps_simulate_batch_ex(low.handle(), nat.ptr(mm), nat.ptr(aa), k, nat.ptr(mk),
                                                     nat.ptr(st), nat.ptr(opmin), nat.PS_HOST_PTRS, None),
                      "ps_simulate_batch_ex")
            if not np.any(st == nat.PS_STATUS_CAPACITY):
                break
            low = lows[depth + 1] = _regrow(low)
        return low, mk, st, opmin

    def visit(depth, used, makespan, min_end_row, low):
        nonlocal best_cost, best_strategy, visited
        visited += 1
        if depth > 0:
            if makespan >= best_cost:
                return
            if depth == N:
                best_cost = makespan
                best_strategy = ParallelizationStrategy(dict(configs))
                return
            min_end = {oid: float(min_end_row[low.rank[oid]]) for oid in order[:depth]}
            bound = makespan
            ec: dict = {}
            for oid in order[depth:]:
                base = 0.0
                for p in preds[oid]:
                    c = min_end[p] if p in min_end else ec.get(p, 0.0)
                    if c > base:
                        base = c
                ec[oid] = base + min_time[oid]
                if ec[oid] > bound:
                    bound = ec[oid]
            if bound >= best_cost:
                return
        elif not order:
            return
        op_id = order[depth]
        children = [(ParallelizationConfig(dict(m.degrees), a), a) for m in maps[op_id]
                    for a in _canonical_assignments(m.size(), used, devices_by_kind)]
        clow, mk, st, opmin = score_children(depth, [c for c, _ in children])
        for j, (cfg, a) in enumerate(children):
            configs[op_id] = cfg
            if st[j] != nat.PS_STATUS_OK:  # raise where the reference's build would
                tg = TaskGraph(clow.graph, topo, ParallelizationStrategy(dict(configs)), profile, mode)
                _bind(tg, clow)
                _raise_status(tg, int(st[j]))
            visit(depth + 1, used | set(a), float(mk[j]), opmin[j], clow)
        configs.pop(op_id, None)

    visit(0, frozenset(), 0.0, None, None)
    return ExhaustiveResult(best_strategy, best_cost, visited, estimate)
