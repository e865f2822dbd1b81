"""Task graphs: the reference's ``parasim.taskgraph`` API over the GPU path.

A :class:`TaskGraph` built by :func:`build_task_graph` is *strategy-backed*: it
holds the lowered problem (:mod:`.lowering`) and the strategy encoded as one
degree-map index per op plus one device per task slot.  The GPU never
materialises it for simulation -- ``k_simulate_batch`` walks successors
straight out of the overlap tables.  When a caller looks at ``tg.tasks`` (or a
timeline), one traced GPU simulation (``ps_simulate_trace``) reports every
task and dependency edge, and the host assembles ``Task`` objects numbered in
the reference's creation order (ops in topological order with their backward
twins, then transfers per op pair in tensor order and sorted (k, l), then
ring all-reduce hops; reference taskgraph.py:276-292), so ids, ``op_tasks``,
``edge_comm`` and the running aggregates match a fresh reference build.

Hand-built graphs (``_new_task``/``_link``, as the reference's tests do) are
*explicit* and simulate through ``ps_simulate_explicit``.
"""

from __future__ import annotations

import ctypes
import math
import weakref
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .cost import CostProfile
from .graph import Connection, DeviceTopology, OperatorGraph, parallelizable_dims
from .lowering import MODE_FORWARD, MODE_FULL, Lowered, degree_tuple, lower, origin_of
from .partition import ParallelizationConfig, ParallelizationStrategy, block_coords, output_region

__all__ = [
    "MODE_FORWARD", "MODE_FULL", "Task", "TimelineEntry", "TaskGraph", "NoRouteError",
    "build_task_graph", "update_task_graph", "link_device_id", "timeline_table",
    "structure_table", "export_dot",
]

NOTREADY, READY, COMPLETE = "NOTREADY", "READY", "COMPLETE"


def link_device_id(conn: Connection) -> str:
    a, b = conn.key()
    return f"link:{a}|{b}"


class NoRouteError(RuntimeError):
    pass


@dataclass(slots=True)
class Task:
    id: int
    kind: str
    device: str
    exe_time: float
    origin: tuple
    op_id: str | None = None
    task_index: int = 0
    nbytes: float = 0.0
    inputs: set = field(default_factory=set)
    outputs: set = field(default_factory=set)


@dataclass(slots=True)
class TimelineEntry:
    ready: float = 0.0
    start: float = 0.0
    end: float = 0.0
    state: str = NOTREADY


class TaskGraph:
    """Task graph plus (after simulation) its timeline; see module docstring."""

    def __init__(self, graph: OperatorGraph, topology: DeviceTopology,
                 strategy: ParallelizationStrategy, profile: CostProfile, mode: str):
        self.graph = graph
        self.topology = topology
        self.strategy = strategy
        self.profile = profile
        self.mode = mode
        self._tasks: dict[int, Task] = {}
        self._timeline: dict[int, TimelineEntry] = {}
        self.device_order: dict[str, list[int]] = {}
        self.device_keys: dict[str, list] = {}
        self.simulated = False
        self._next_id = 0
        self._device_busy: dict[str, float] = {dev: 0.0 for dev in topology.devices}
        self._total_comm_bytes = 0.0
        self._op_tasks: dict = {}
        self._op_bwd: dict = {}
        self._edge_comm: dict = {}
        self._edge_comm_bwd: dict = {}
        self._sync_tasks: dict = {}
        # strategy-backed state
        self._low: Lowered | None = None
        self._map: np.ndarray | None = None
        self._asg: np.ndarray | None = None
        self._mat_valid = False
        self._makespan: float | None = None
        self._dh = None           # resident delta-evaluation handle (_DeltaHandle)
        self._dh_pending = None   # op ranks changed since the handle's strategy (None: out of sync)

    # -- explicit construction (reference taskgraph.py:114-125) ----------------
    def _new_task(self, kind, device, exe_time, origin, op_id=None, task_index=0, nbytes=0.0) -> Task:
        if self._low is not None:
            raise RuntimeError("strategy-backed task graphs are immutable; use update_task_graph")
        t = Task(self._next_id, kind, device, exe_time, origin, op_id, task_index, nbytes)
        self._next_id += 1
        self._tasks[t.id] = t
        self._device_busy[device] = self._device_busy.get(device, 0.0) + exe_time
        if kind == "comm":
            self._total_comm_bytes += nbytes
        return t

    def _link(self, a: int, b: int):
        self._tasks[a].outputs.add(b)
        self._tasks[b].inputs.add(a)

    # -- lazily materialised views ------------------------------------------------
    def _view(self):
        if self._low is not None and not self._mat_valid:
            _materialize(self)

    @property
    def tasks(self) -> dict:
        self._view()
        return self._tasks

    @tasks.setter
    def tasks(self, value):
        self._tasks = value

    @property
    def timeline(self) -> dict:
        self._view()
        return self._timeline

    @timeline.setter
    def timeline(self, value):
        self._timeline = value

    @property
    def device_busy(self) -> dict:
        self._view()
        return self._device_busy

    @device_busy.setter
    def device_busy(self, value):
        self._device_busy = value

    @property
    def total_comm_bytes(self) -> float:
        self._view()
        return self._total_comm_bytes

    @total_comm_bytes.setter
    def total_comm_bytes(self, value):
        self._total_comm_bytes = value

    for _name in ("op_tasks", "op_bwd", "edge_comm", "edge_comm_bwd", "sync_tasks"):
        def _get(self, _n="_" + _name):
            self._view()
            return getattr(self, _n)
        locals()[_name] = property(_get)
    del _name, _get

    def device_ids(self) -> list[str]:
        ids = set(self.topology.devices)
        ids.update(t.device for t in self.tasks.values())
        return sorted(ids)


# -----------------------------------------------------------------------------
# strategy-backed construction

# Lowered problems cached per profile object, outside the profile (so the profile
# still pickles and deep-copies).  An entry is reused only while its fingerprint
# -- the graph's ops and tensors, the topology's devices and connections, the
# profile's entries, fallback and backward multiplier, the mode -- is unchanged:
# an in-place edit of any of them lowers again, as the reference would pick the
# new values up on its next build.
_LOWER_CACHE: dict = {}


def _fingerprint(g, topo, profile, mode):
    return (id(g), tuple(map(id, g.ops.values())), tuple(map(id, g.tensors)), id(topo),
            tuple(map(id, topo.devices.values())), tuple(map(id, topo.connections)), mode,
            profile.backward_multiplier, repr(profile.fallback), len(profile.entries),
            hash(frozenset(profile.entries.items())))


def _cache_get(profile):
    hit = _LOWER_CACHE.get(id(profile))
    if hit is None or hit[0]() is not profile:
        return None
    return hit


def _cache_put(profile, fp, low, strategies):
    pid = id(profile)
    try:
        ref = weakref.ref(profile, lambda _r, pid=pid: _LOWER_CACHE.pop(pid, None))
    except TypeError:
        return
    _LOWER_CACHE[pid] = (ref, fp, low, strategies)


def _problem_for(g, topo, profile, mode, strategy, max_degree=None) -> Lowered:
    """Reuse a lowered problem for (g, topo, profile, mode) when it covers the
    strategy's degree maps; otherwise lower again (union of maps)."""
    hit = _cache_get(profile)
    fp = _fingerprint(g, topo, profile, mode)
    if hit is not None and hit[1] == fp:
        low = hit[2]
        if (max_degree is None or low.max_degree == max_degree) and low.has_maps_for(strategy):
            return low
        strategies = [strategy] + hit[3]
        if max_degree is None:
            max_degree = low.max_degree
    else:
        strategies = [strategy]
        if max_degree is None:
            # every degree map of the reference's default proposal space (SearchParams.max_degree
            # = 4): update_task_graph to any of them then rewrites the encoded fragment in place
            max_degree = min(4, len(topo.devices))
    low = lower(g, topo, profile, mode, max_degree=max_degree, strategies=strategies, quiet_extra=True)
    # lowering inserts the fallback's answers into profile.entries: fingerprint after
    _cache_put(profile, _fingerprint(g, topo, profile, mode), low, strategies[-8:])
    return low


def _check_config(g, topo, op_id, cfg):
    """The reference's build-time failures for one config (partition.py:117-127,
    taskgraph.py:131-134): ValueError, TypeError/IndexError, KeyError."""
    op = g.ops[op_id]
    t = degree_tuple(op, cfg.degrees)
    for n, d in zip(op.output_shape.names(), t):
        if op.output_shape.size(n) % d:
            raise ValueError(f"op {op_id}: degree {d} does not divide {n} size {op.output_shape.size(n)}")
    if cfg.assignment is None:
        raise TypeError("'NoneType' object is not subscriptable")
    size = math.prod(t)
    if len(cfg.assignment) < size:
        raise IndexError("tuple index out of range")
    for dev in cfg.assignment[:size]:
        if dev not in topo.devices:
            raise KeyError(dev)


def _first_missing_route(tg: TaskGraph, pair_order=None, sync_ops=None):
    """The device pair the reference's build would report first
    (taskgraph.py:148-152,199-213,247-256): transfers per pair in tensor order
    and sorted (k, l), then rings per op in topological order.  ``pair_order``
    / ``sync_ops`` restrict and order the scan (update_task_graph's order)."""
    low = tg._low
    L = nat.lib()
    g, topo = tg.graph, tg.topology
    pair_ids = {(low.ops[s], low.ops[d]): p for p, (s, d) in enumerate(low.pairs)}
    scan = range(len(low.pairs)) if pair_order is None else [pair_ids[x] for x in pair_order if x in pair_ids]
    for p in scan:
        s, d = low.pairs[p]
        cs, cd = tg.strategy.configs[low.ops[s]], tg.strategy.configs[low.ops[d]]
        ms, md = int(tg._map[s]), int(tg._map[d])
        cap = low.arrays["map_size"][low.arrays["op_map_off"][s] + ms] * \
            low.arrays["map_size"][low.arrays["op_map_off"][d] + md]
        kk = np.zeros(cap, dtype=np.int32)
        ll = np.zeros(cap, dtype=np.int32)
        bb = np.zeros(cap, dtype=np.int64)
        n = ctypes.c_int()
        nat.check(L.ps_combo_entries(low.handle(), p, ms, md, int(cap), nat.ptr(kk), nat.ptr(ll), nat.ptr(bb),
                                     ctypes.byref(n)), "ps_combo_entries")
        for i in range(n.value):
            a, b = cs.assignment[kk[i]], cd.assignment[ll[i]]
            if a != b and topo.connection_between(a, b) is None:
                return a, b
    if tg.mode == MODE_FULL:
        for oid in (g.topological_order() if sync_ops is None else sync_ops):
            op = g.ops[oid]
            if op.param_bytes <= 0:
                continue
            cfg = tg.strategy.configs[oid]
            names = op.output_shape.names()
            degs = list(degree_tuple(op, cfg.degrees))
            classes = parallelizable_dims(op)
            pp = [i for i, n in enumerate(names) if classes.get(n) == "parameter"]
            groups: dict = {}
            for k, dev in enumerate(cfg.assignment):
                coords = block_coords(degs, k)
                groups.setdefault(tuple(coords[i] for i in pp), set()).add(dev)
            for key in sorted(groups):
                ring = sorted(groups[key])
                r = len(ring)
                if r < 2:
                    continue
                for h in range(2 * (r - 1)):
                    if topo.connection_between(ring[h % r], ring[(h + 1) % r]) is None:
                        return ring[h % r], ring[(h + 1) % r]
    return None


def _simulate_strategy(tg: TaskGraph) -> float:
    """Makespan of the current strategy through k_simulate_batch (n=1)."""
    low = tg._low
    L = nat.lib()
    mk = np.zeros(1, dtype=np.float64)
    st = np.zeros(1, dtype=np.int32)
    nat.check(L.ps_simulate_batch(low.handle(), nat.ptr(tg._map), nat.ptr(tg._asg), 1, nat.ptr(mk), nat.ptr(st),
                                  nat.PS_HOST_PTRS, None), "ps_simulate_batch")
    _raise_status(tg, int(st[0]))
    return float(mk[0])


def _raise_status(tg: TaskGraph, status: int):
    if status == nat.PS_STATUS_OK:
        return
    if status == nat.PS_STATUS_NO_ROUTE:
        pair = _first_missing_route(tg)
        a, b = pair if pair is not None else ("?", "?")
        raise NoRouteError(f"no route between device {a} and device {b}")
    if status == nat.PS_STATUS_CAPACITY:
        # grow the ready set and retry once on a fresh problem
        raise _CapacityRetry()
    raise RuntimeError(f"GPU simulation failed with status {status}")


class _CapacityRetry(Exception):
    pass


def _bind(tg: TaskGraph, low: Lowered):
    tg._low = low
    tg._map, tg._asg = low.encode(tg.strategy)
    tg._mat_valid = False


def build_task_graph(g: OperatorGraph, topo: DeviceTopology, strategy: ParallelizationStrategy,
                     profile: CostProfile, mode: str = MODE_FORWARD) -> TaskGraph:
    """Materialise a strategy (reference taskgraph.py:276-292) on the GPU path.

    Same errors as the reference: ValueError for a non-dividing degree,
    KeyError for an unknown device, NoRouteError for a missing link."""
    if mode not in (MODE_FORWARD, MODE_FULL):
        raise ValueError(f"unknown mode {mode!r}")
    tg = TaskGraph(g, topo, strategy.copy(), profile, mode)
    g.topological_order()
    for oid in sorted(g.ops):
        if oid not in tg.strategy.configs:
            raise KeyError(oid)
        _check_config(g, topo, oid, tg.strategy.configs[oid])
    _bind(tg, _problem_for(g, topo, profile, mode, tg.strategy))
    for _ in range(4):
        try:
            tg._makespan = _simulate_strategy(tg)
            break
        except _CapacityRetry:
            _grow(tg)
    return tg


def _grow(tg: TaskGraph):
    from .search import _regrow
    new = _regrow(tg._low)
    hit = _cache_get(tg.profile)
    if hit is not None and hit[2] is tg._low:
        _LOWER_CACHE[id(tg.profile)] = (hit[0], hit[1], new, hit[3])
    _bind(tg, new)


def update_task_graph(tg: TaskGraph, g: OperatorGraph, topo: DeviceTopology, op_id: str,
                      new_config: ParallelizationConfig):
    """Swap one op's config (reference taskgraph.py:309-418).

    Returns (tg, changed).  ``changed`` is empty for a no-op swap (same degree
    dict and assignment), else the ids -- in the updated graph -- of the op's
    own tasks and of every task whose inputs, device or exe time changed with
    it.  Unlike the reference, ids are renumbered in fresh-build order.

    The update itself only rewrites the op's fragment of the encoded strategy
    (one map index and that op's device bytes); ``changed`` is computed, and
    the task objects are assembled, only when someone reads them.  On a
    topology that is not a full mesh the updated graph is materialised at once,
    so a missing link raises NoRouteError here, as in the reference."""
    cur = tg.strategy.configs[op_id]
    if cur.degrees == new_config.degrees and cur.assignment == new_config.assignment:
        return tg, []
    if tg._low is None:
        raise RuntimeError("update_task_graph needs a strategy-backed task graph")
    _check_config(g, topo, op_id, new_config)
    old_strategy = tg.strategy.copy()
    cfg = ParallelizationConfig(dict(new_config.degrees),
                                tuple(new_config.assignment) if new_config.assignment is not None else None)
    tg.strategy.configs[op_id] = cfg
    low = tg._low
    r = low.rank[op_id]
    t = degree_tuple(g.ops[op_id], cfg.degrees)
    mi = low.map_index[r].get(t)
    if mi is None:
        # a degree map the lowered problem lacks: lower again (union of maps)
        low = _problem_for(g, topo, tg.profile, tg.mode, tg.strategy, max_degree=low.max_degree)
        _bind(tg, low)
    else:
        # patch the encoded fragment in place
        tg._map[r] = mi
        base = int(low.slot_off[r])
        for k in range(math.prod(t)):
            tg._asg[base + k] = low.dev_index[cfg.assignment[k]]
        tg._mat_valid = False
        _touch_profile(tg, op_id, cfg)
    tg._makespan = None
    if tg._dh is not None and tg._dh_pending is not None and tg._dh.low is tg._low:
        tg._dh_pending.append(r)
    else:
        tg._dh_pending = None
    if not _full_mesh(low):
        was_simulated = tg.simulated
        _materialize(tg)  # raises NoRouteError for a missing link, like the reference's update
        tg.simulated = was_simulated
    return tg, ChangedTasks(tg, old_strategy, tg.strategy.copy(), op_id)


def _touch_profile(tg: TaskGraph, op_id: str, cfg: ParallelizationConfig):
    """The profile lookups the reference's update makes for the new fragment
    (cost.py:113-121): a map first used here inserts its entry.  The lowered
    tables already hold the same value, so the cached problem stays valid."""
    prof, op = tg.profile, tg.graph.ops[op_id]
    n0 = len(prof.entries)
    region0 = output_region(op, cfg, 0)
    kinds = {}
    for dev in cfg.assignment[:math.prod(degree_tuple(op, cfg.degrees))]:
        d = tg.topology.devices[dev]
        kinds.setdefault(d.kind, d)
    for d in kinds.values():
        prof.task_exe_time(op, region0, d)
    if len(prof.entries) != n0:
        hit = _cache_get(prof)
        if hit is not None and hit[2] is tg._low:
            _cache_put(prof, _fingerprint(tg.graph, tg.topology, prof, tg.mode), hit[2], hit[3])


def _full_mesh(low: Lowered) -> bool:
    """Every device pair connected: no strategy can need a missing link."""
    v = getattr(low, "_full_mesh", None)
    if v is None:
        topo = low.topology
        ids = topo.device_ids()
        v = all(topo.connection_between(a, b) is not None for i, a in enumerate(ids) for b in ids[i + 1:])
        low._full_mesh = v
    return v


class ChangedTasks(Sequence):
    """update_task_graph's ``changed`` list, computed on first access: the op's
    own tasks and transfers / ring hops, plus every task whose device, exe time
    or input origins differ between the graph before and after the change."""

    __slots__ = ("_args", "_ids")

    def __init__(self, tg, old_strategy, new_strategy, op_id):
        self._args = (tg.graph, tg.topology, tg.profile, tg.mode, old_strategy, new_strategy, op_id)
        self._ids = None

    def _get(self) -> list:
        if self._ids is None:
            g, topo, profile, mode, old_s, new_s, op_id = self._args
            graphs = []
            for strat in (old_s, new_s):
                x = TaskGraph(g, topo, strat, profile, mode)
                _bind(x, _problem_for(g, topo, profile, mode, strat))
                _materialize(x)
                graphs.append(x)
            old, new = graphs
            before = {t.origin: (t.exe_time, t.device, frozenset(old._tasks[p].origin for p in t.inputs))
                      for t in old._tasks.values()}
            out = []
            for tid, t in new._tasks.items():
                if t.op_id == op_id or (t.origin[0] in ("edge", "edge_bwd", "sync") and op_id in t.origin[1:3]):
                    out.append(tid)
                    continue
                prev = before.get(t.origin)
                if prev is None or prev != (t.exe_time, t.device, frozenset(new._tasks[p].origin for p in t.inputs)):
                    out.append(tid)
            self._ids = sorted(out)
            self._args = None
        return self._ids

    def __bool__(self):
        return True  # the changed op always has at least one task

    def __len__(self):
        return len(self._get())

    def __getitem__(self, i):
        return self._get()[i]

    def __iter__(self):
        return iter(self._get())

    def __eq__(self, other):
        return list(self) == list(other) if isinstance(other, (list, tuple, Sequence)) else NotImplemented

    def __repr__(self):
        return repr(self._get())


def _destroy_handle(h, _low):
    nat.lib().ps_mcmc_destroy(h)


class _DeltaHandle:
    """A one-chain ps_mcmc handle with delta evaluation on: it holds the
    strategy the task graph was last delta-simulated with, and that
    simulation's snapshots, so the next single-op change resumes mid-timeline
    (ps_delta_batch)."""

    def __init__(self, low: Lowered, m: np.ndarray, a: np.ndarray):
        L = nat.lib()
        self.low = low
        self.h = ctypes.c_void_p()
        mp = nat.PsMcmcParams(nat.PS_RNG_PHILOX, 0, 0.0, math.log(10.0), 0, 0, 1)
        seeds = np.zeros(1, dtype=np.uint64)
        nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), 1, nat.ptr(m), nat.ptr(a), nat.ptr(seeds), None,
                                   ctypes.byref(self.h)), "ps_mcmc_create")
        weakref.finalize(self, _destroy_handle, self.h, low)  # (low: keeps the problem alive until then)
        nat.check(L.ps_mcmc_run(self.h, 0, None), "ps_mcmc_run")  # scores (and snapshots) the strategy
        summ = (nat.PsChainSummary * 1)()
        nat.check(L.ps_mcmc_read(self.h, summ, None, None, None, None), "ps_mcmc_read")
        self.cost, self.status = float(summ[0].cost), int(summ[0].status)
        self._op = np.zeros(1, dtype=np.int32)
        self._mi = np.zeros(1, dtype=np.int32)
        self._mk = np.zeros(1, dtype=np.float64)
        self._st = np.zeros(1, dtype=np.int32)

    def change(self, r: int, mi: int, devices: np.ndarray):
        """Commit op rank r := (map mi, devices); returns (makespan, status)."""
        self._op[0], self._mi[0] = r, mi
        a = np.ascontiguousarray(devices, dtype=np.uint8)
        nat.check(nat.lib().ps_delta_batch(self.h, nat.ptr(self._op), nat.ptr(self._mi), nat.ptr(a), max(1, a.size),
                                           None, nat.ptr(self._mk), nat.ptr(self._st), nat.PS_HOST_PTRS, None),
                  "ps_delta_batch")
        self.cost, self.status = float(self._mk[0]), int(self._st[0])
        return self.cost, self.status


def _delta_makespan(tg: TaskGraph) -> float:
    """Makespan of the updated strategy by delta evaluation on the task graph's
    resident handle (created -- one from-scratch scoring -- on first use)."""
    for _ in range(4):
        low = tg._low
        dh, pend = tg._dh, tg._dh_pending
        if dh is not None and dh.low is low and pend is not None and dh.status == nat.PS_STATUS_OK \
                and len(set(pend)) <= 4:
            st = nat.PS_STATUS_OK
            mk = dh.cost
            for r in dict.fromkeys(pend):  # each changed op once, in update order
                size = int(low.arrays["map_size"][low.arrays["op_map_off"][r] + int(tg._map[r])])
                base = int(low.slot_off[r])
                mk, st = dh.change(r, int(tg._map[r]), tg._asg[base:base + size])
                if st != nat.PS_STATUS_OK:
                    break
        else:
            dh = _DeltaHandle(low, tg._map, tg._asg)
            mk, st = dh.cost, dh.status
        if st == nat.PS_STATUS_OK:
            tg._dh, tg._dh_pending = dh, []
            return mk
        tg._dh, tg._dh_pending = None, None
        if st == nat.PS_STATUS_CAPACITY:
            _grow(tg)  # a ready set outgrew shared memory: 4x capacity, new handle
            continue
        _raise_status(tg, st)
    raise RuntimeError("delta evaluation did not converge on a ready-set capacity")


def _creation_key(low: Lowered, topo_pos: dict, pair_pos: dict, origin: tuple):
    kind = origin[0]
    if kind in ("op", "op_bwd"):
        return (0, topo_pos[origin[1]], 0 if kind == "op" else 1, origin[2])
    if kind in ("edge", "edge_bwd"):
        return (1, pair_pos[(origin[1], origin[2])], origin[3], origin[4], 0 if kind == "edge" else 1)
    return (2, topo_pos[origin[1]], origin[2], origin[3])


def _materialize(tg: TaskGraph):
    """Traced GPU simulation -> Task objects, timeline and aggregates."""
    low = tg._low
    L = nat.lib()
    for _ in range(4):
        task_cap = max(1024, 4 * low.n_slots + 64)
        edge_cap = 4 * task_cap
        while True:
            tasks = np.zeros(task_cap, dtype=nat.TRACE_DTYPE)
            ep = np.zeros(edge_cap, dtype=np.int32)
            es = np.zeros(edge_cap, dtype=np.uint64)
            nt, ne = ctypes.c_int(), ctypes.c_int()
            mk = ctypes.c_double()
            st = ctypes.c_int32()
            err = np.zeros(2, dtype=np.int32)
            rc = L.ps_simulate_trace(low.handle(), nat.ptr(tg._map), nat.ptr(tg._asg), task_cap, nat.ptr(tasks),
                                     ctypes.byref(nt), edge_cap, nat.ptr(ep), nat.ptr(es), ctypes.byref(ne),
                                     ctypes.byref(mk), ctypes.byref(st), nat.ptr(err))
            if rc == nat.PS_ERR_CAPACITY and (nt.value > task_cap or ne.value > edge_cap):
                task_cap = max(task_cap, nt.value) * 2
                edge_cap = max(edge_cap, ne.value) * 2
                continue
            nat.check(rc, "ps_simulate_trace")
            break
        try:
            _raise_status(tg, int(st.value))
            break
        except _CapacityRetry:
            _grow(tg)
            low = tg._low
    n = nt.value
    tasks = tasks[:n]
    g = tg.graph
    topo_pos = {oid: i for i, oid in enumerate(g.topological_order())}
    pair_pos = {(low.ops[s], low.ops[d]): i for i, (s, d) in enumerate(low.pairs)}
    origins = [origin_of(low, int(k)) for k in tasks["key"]]
    order = sorted(range(n), key=lambda i: _creation_key(low, topo_pos, pair_pos, origins[i]))
    id_of_pop = [0] * n
    for new_id, i in enumerate(order):
        id_of_pop[i] = new_id
    key_to_id = {int(tasks["key"][i]): id_of_pop[i] for i in range(n)}
    objs: dict[int, Task] = {}
    timeline: dict[int, TimelineEntry] = {}
    busy = {dev: 0.0 for dev in tg.topology.devices}
    comm_total = 0.0
    op_tasks: dict = {}
    op_bwd: dict = {}
    edge_comm: dict = {}
    edge_comm_bwd: dict = {}
    sync_tasks: dict = {}
    for new_id, i in enumerate(order):
        o = origins[i]
        rec = tasks[i]
        dev = low.queue_name(int(rec["queue"]))
        exe = float(rec["exe"])
        kind = "normal" if o[0] in ("op", "op_bwd") else "comm"
        if kind == "comm":
            nb = float(rec["nbytes"])
            nbytes = int(nb) if o[0] in ("edge", "edge_bwd") else nb
            t = Task(new_id, kind, dev, exe, o, nbytes=nbytes)
            comm_total += nbytes
        else:
            t = Task(new_id, kind, dev, exe, o, o[1], o[2])
        objs[new_id] = t
        busy[dev] = busy.get(dev, 0.0) + exe
        timeline[new_id] = TimelineEntry(float(rec["ready"]), float(rec["start"]), float(rec["end"]), COMPLETE)
        if o[0] == "op":
            op_tasks.setdefault(o[1], []).append(new_id)
        elif o[0] == "op_bwd":
            op_bwd.setdefault(o[1], []).append(new_id)
        elif o[0] == "edge":
            edge_comm.setdefault((o[1], o[2]), []).append(new_id)
        elif o[0] == "edge_bwd":
            edge_comm_bwd.setdefault((o[1], o[2]), []).append(new_id)
        else:
            sync_tasks.setdefault(o[1], []).append(new_id)
    for j in range(ne.value):
        a = id_of_pop[int(ep[j])]
        b = key_to_id[int(es[j])]
        objs[a].outputs.add(b)
        objs[b].inputs.add(a)
    if tg.mode == MODE_FULL:
        for oid, op in g.ops.items():
            if op.param_bytes > 0:
                sync_tasks.setdefault(oid, [])
    order_by_queue: dict[str, list[int]] = {}
    keys_by_queue: dict[str, list] = {}
    for i in range(n):  # pop order == per-queue FIFO order
        tid = id_of_pop[i]
        t = objs[tid]
        order_by_queue.setdefault(t.device, []).append(tid)
        keys_by_queue.setdefault(t.device, []).append((timeline[tid].ready, t.origin))
    tg._tasks = objs
    tg._timeline = timeline
    tg._device_busy = busy
    tg._total_comm_bytes = comm_total
    tg._op_tasks, tg._op_bwd = op_tasks, op_bwd
    tg._edge_comm, tg._edge_comm_bwd, tg._sync_tasks = edge_comm, edge_comm_bwd, sync_tasks
    tg.device_order, tg.device_keys = order_by_queue, keys_by_queue
    tg._next_id = n
    tg._makespan = float(mk.value)
    tg._mat_valid = True


# -----------------------------------------------------------------------------
# canonical views (reference taskgraph.py:424-458)

def timeline_table(tg: TaskGraph) -> dict:
    tl = tg.timeline
    return {t.origin: (tl[tid].start, tl[tid].end, t.device) for tid, t in tg.tasks.items()}


def structure_table(tg: TaskGraph) -> list:
    tasks = tg.tasks
    origin = {tid: t.origin for tid, t in tasks.items()}
    rows = [(t.origin, t.device, t.exe_time, t.nbytes, tuple(sorted(origin[p] for p in t.inputs)))
            for _, t in sorted(tasks.items())]
    rows.sort(key=lambda r: repr(r[0]))
    return rows


def export_dot(tg: TaskGraph) -> str:
    out = ["digraph taskgraph {"]
    tasks = tg.tasks
    for tid in sorted(tasks):
        t = tasks[tid]
        label = ":".join(map(str, t.origin)) + f"\\n{t.device}\\n{t.exe_time:.3g}s"
        out.append(f'  t{tid} [label="{label}"{" shape=box" if t.kind == "comm" else ""}];')
    for tid in sorted(tasks):
        out.extend(f"  t{tid} -> t{s};" for s in sorted(tasks[tid].outputs))
    out.append("}")
    return "\n".join(out)
