"""Simulators: the reference's ``parasim.simulate`` API over the GPU kernels.

Scheduling contract (reference simulate.py:1-11): FIFO per device and per
link, a task is ready when its last predecessor ends, ties on ready time break
by origin tuple.  ``full_simulate`` and ``delta_simulate`` both run the
warp-per-candidate replay of the reference's heap order
(``k_simulate_batch`` / ``ps_simulate_trace``); for a strategy-backed graph
``delta_simulate`` re-simulates the updated strategy on the GPU resumed from a
snapshot of the previous simulation taken before the changed op's first
dependent round (``ps_delta_batch`` on a resident one-chain handle); the
reference's contract is that delta and full agree exactly (simulate.py:121),
and they do, bit for bit.
``oracle_simulate`` re-simulates the materialised task list through the
structurally separate explicit-CSR kernel (``ps_simulate_explicit``).
"""

from __future__ import annotations

import csv
import ctypes
import json

import numpy as np

from . import _native as nat
from .taskgraph import COMPLETE, TaskGraph, TimelineEntry, _materialize

__all__ = ["SimulationResult", "SimulationError", "full_simulate", "delta_simulate", "oracle_simulate",
           "chrome_trace", "write_chrome_trace", "write_timeline_csv"]


class SimulationError(RuntimeError):
    pass


class SimulationResult:
    """makespan, timeline, device_busy, total_comm_bytes (reference simulate.py:39-52).

    For strategy-backed graphs the makespan comes straight from the batch
    kernel; the per-task views are assembled on first access."""

    __slots__ = ("makespan", "_tg", "_timeline", "_busy", "_comm")

    def __init__(self, makespan, timeline=None, device_busy=None, total_comm_bytes=None, tg=None):
        self.makespan = makespan
        self._tg = tg
        self._timeline = timeline
        self._busy = device_busy
        self._comm = total_comm_bytes

    def _load(self):
        if self._timeline is None and self._tg is not None:
            tg = self._tg
            self._timeline = tg.timeline
            self._busy = dict(tg.device_busy)
            self._comm = tg.total_comm_bytes

    @property
    def timeline(self):
        self._load()
        return self._timeline

    @property
    def device_busy(self):
        self._load()
        return self._busy

    @property
    def total_comm_bytes(self):
        self._load()
        return self._comm

    def __eq__(self, other):
        if not isinstance(other, SimulationResult):
            return NotImplemented
        return (self.makespan == other.makespan and self.timeline == other.timeline
                and self.device_busy == other.device_busy and self.total_comm_bytes == other.total_comm_bytes)

    def __repr__(self):
        return f"SimulationResult(makespan={self.makespan!r})"


def _explicit_arrays(tg: TaskGraph):
    tasks = tg.tasks
    ids = sorted(tasks)
    pos = {tid: i for i, tid in enumerate(ids)}
    queues = sorted({tasks[t].device for t in ids})
    qidx = {q: i for i, q in enumerate(queues)}
    origin_rank = {o: r for r, o in enumerate(sorted({tasks[t].origin for t in ids}))}
    n = len(ids)
    queue = np.array([qidx[tasks[t].device] for t in ids] or [0], dtype=np.int32)
    exe = np.array([tasks[t].exe_time for t in ids] or [0.0], dtype=np.float64)
    rank = np.array([origin_rank[tasks[t].origin] for t in ids] or [0], dtype=np.uint64)
    succ_off = np.zeros(n + 1, dtype=np.int32)
    succ = []
    for i, t in enumerate(ids):
        outs = [pos[s] for s in tasks[t].outputs]
        succ.extend(outs)
        succ_off[i + 1] = succ_off[i] + len(outs)
    return ids, queues, queue, exe, rank, succ_off, np.array(succ or [0], dtype=np.int32)


def _run_explicit(tg: TaskGraph):
    ids, queues, queue, exe, rank, succ_off, succ = _explicit_arrays(tg)
    n = len(ids)
    ready = np.zeros(max(n, 1))
    start = np.zeros(max(n, 1))
    end = np.zeros(max(n, 1))
    order = np.zeros(max(n, 1), dtype=np.int32)
    mk = ctypes.c_double()
    st = ctypes.c_int32()
    L = nat.lib()
    L.ps_simulate_explicit.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 9 + \
        [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32), ctypes.c_int]
    dev = tg._low.device if tg._low is not None else 0
    nat.check(L.ps_simulate_explicit(n, len(queues), nat.ptr(queue), nat.ptr(exe), nat.ptr(rank), nat.ptr(succ_off),
                                     nat.ptr(succ), nat.ptr(ready), nat.ptr(start), nat.ptr(end), nat.ptr(order),
                                     ctypes.byref(mk), ctypes.byref(st), dev), "ps_simulate_explicit")
    return ids, ready, start, end, order, float(mk.value), int(st.value)


def full_simulate(tg: TaskGraph) -> SimulationResult:
    """Simulate from scratch (reference simulate.py:68-117)."""
    if tg._low is not None:
        from .taskgraph import _simulate_strategy
        if tg._mat_valid:
            mk = tg._makespan
        else:
            mk = _simulate_strategy(tg)
            tg._makespan = mk
        tg.simulated = True
        return SimulationResult(mk, tg=tg)
    ids, ready, start, end, order, mk, status = _run_explicit(tg)
    tasks = tg.tasks
    if status != nat.PS_STATUS_OK:
        done = set(ids[int(i)] for i in order[:0])
        raise SimulationError(f"task {tasks[_first_stuck(tg, ids, order)].origin} never became ready "
                              "(cycle or broken dependency)")
    tl = {}
    dev_order: dict = {}
    dev_keys: dict = {}
    for j in range(len(ids)):
        i = int(order[j])
        tid = ids[i]
        tl[tid] = TimelineEntry(float(ready[i]), float(start[i]), float(end[i]), COMPLETE)
        d = tasks[tid].device
        dev_order.setdefault(d, []).append(tid)
        dev_keys.setdefault(d, []).append((float(ready[i]), tasks[tid].origin))
    tg._timeline = tl
    tg.device_order = dev_order
    tg.device_keys = dev_keys
    tg.simulated = True
    return _result(tg)


def _first_stuck(tg, ids, order):
    # tasks reachable only through a cycle never pop; report the smallest id
    tasks = tg.tasks
    indeg = {t: len(tasks[t].inputs) for t in ids}
    ready = [t for t in ids if indeg[t] == 0]
    seen = set(ready)
    while ready:
        t = ready.pop()
        for s in tasks[t].outputs:
            indeg[s] -= 1
            if indeg[s] == 0:
                seen.add(s)
                ready.append(s)
    return next(t for t in ids if t not in seen)


def _result(tg: TaskGraph) -> SimulationResult:
    makespan = 0.0
    tl = tg.timeline
    for lst in tg.device_order.values():
        if lst and tl[lst[-1]].end > makespan:
            makespan = tl[lst[-1]].end
    return SimulationResult(makespan, tl, dict(tg.device_busy), tg.total_comm_bytes)


def delta_simulate(tg: TaskGraph, changed: list[int]) -> SimulationResult:
    """Re-simulate after update_task_graph; equals full_simulate exactly
    (reference simulate.py:120-210)."""
    if not tg.simulated:
        raise SimulationError("delta_simulate requires a prior full_simulate on this graph")
    if not changed:
        if tg._low is not None:
            if tg._makespan is None:
                return full_simulate(tg)
            return SimulationResult(tg._makespan, tg=tg)
        return _result(tg)
    if tg._low is not None:
        from .taskgraph import _delta_makespan
        if tg._mat_valid and tg._makespan is not None:
            mk = tg._makespan
        else:
            mk = _delta_makespan(tg)
            tg._makespan = mk
        tg.simulated = True
        return SimulationResult(mk, tg=tg)
    return full_simulate(tg)


def oracle_simulate(tg: TaskGraph) -> float:
    """Makespan via the explicit-CSR kernel over the materialised task list
    (independent of the implicit fragment walk; reference simulate.py:213-276)."""
    if not tg.tasks:
        return 0.0
    ids, ready, start, end, order, mk, status = _run_explicit(tg)
    if status != nat.PS_STATUS_OK:
        raise SimulationError(f"task {tg.tasks[_first_stuck(tg, ids, order)].origin} never became ready "
                              "(cycle or broken dependency)")
    return mk


# -- timeline exports (reference simulate.py:282-317) --------------------------

def chrome_trace(tg: TaskGraph) -> dict:
    lanes = {dev: i for i, dev in enumerate(tg.device_ids())}
    events = [{"name": "process_name", "ph": "M", "pid": i, "tid": 0, "args": {"name": dev}}
              for dev, i in lanes.items()]
    tl = tg.timeline
    for tid in sorted(tg.tasks):
        t = tg.tasks[tid]
        e = tl[tid]
        events.append({"name": ":".join(map(str, t.origin)), "cat": t.kind, "ph": "X",
                       "ts": e.start * 1e6, "dur": (e.end - e.start) * 1e6, "pid": lanes[t.device], "tid": 0})
    return {"traceEvents": events, "displayTimeUnit": "ms"}


def write_chrome_trace(tg: TaskGraph, path):
    with open(path, "w") as fh:
        json.dump(chrome_trace(tg), fh, indent=1)


def write_timeline_csv(tg: TaskGraph, path):
    tl = tg.timeline
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["task", "device", "start", "end"])
        for tid in sorted(tg.tasks, key=lambda i: (tl[i].start, i)):
            t = tg.tasks[tid]
            w.writerow([":".join(map(str, t.origin)), t.device, repr(tl[tid].start), repr(tl[tid].end)])
