"""Lowering: (OperatorGraph, DeviceTopology, CostProfile, mode) -> device tables.

Everything the kernels need is flattened here into the ``ps_problem_desc`` of
include/parasim.h and handed to ``ps_problem_create``, which uploads it and
builds the region-overlap tables on the GPU.  Layout:

* ops are indexed by their rank in ``sorted(g.ops)`` -- the order the
  reference's origin tuples compare op ids in (simulate.py:5-7,
  taskgraph.py:135,143,210,217,258), so packed origin keys sort like tuples;
* devices by rank in ``topo.device_ids()``; a queue is a device or a link
  (one per connected unordered pair, the first connection registered wins,
  graph.py:223-230);
* per op a list of degree maps (degree per output dim): the
  ``enumerate_configs`` list first, in its order (proposals index into it),
  then any extra maps the caller's strategies use;
* per (op, map, device kind) the fp64 task time from the profile (every block
  of a map has the same dims, so one lookup covers all its tasks,
  cost.py:105-121) and its backward twin ``exe * backward_multiplier``;
* per op pair (distinct (src, dst) in ``g.tensors`` order) and tensor edge,
  a per-source-dim "need" descriptor (partition.need_descriptors);
* a strategy is (local map index per op, one device per task slot); op o's
  tasks occupy slots ``slot_off[o] .. slot_off[o] + size``.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .cost import cost_key_for
from .graph import DeviceTopology, OperatorGraph, parallelizable_dims
from .partition import ParallelizationConfig, enumerate_configs, grid_of, need_descriptors, output_region

__all__ = ["Lowered", "lower", "MODE_FORWARD", "MODE_FULL"]

MODE_FORWARD = "forward"
MODE_FULL = "full-iteration"

KIND_NAMES = ("edge", "edge_bwd", "op", "op_bwd", "sync")


_DEGREE_TUPLES: dict = {}


def degree_tuple(op, degrees: dict) -> tuple[int, ...]:
    """Degrees in output-dim order (missing dims = 1); memoised on the (frozen)
    output shape and the degree items, since large searches look the same few
    maps up millions of times."""
    key = (op.output_shape.dims, tuple(degrees.items()))
    hit = _DEGREE_TUPLES.get(key)
    if hit is not None:
        return hit
    names = op.output_shape.names()
    for n in degrees:
        if n not in names:
            raise ValueError(f"op {op.id}: degree given for dimension {n} absent from its output")
    t = tuple(int(degrees.get(n, 1)) for n in names)
    if len(_DEGREE_TUPLES) < 1 << 16:
        _DEGREE_TUPLES[key] = t
    return t


@dataclass
class Lowered:
    graph: OperatorGraph
    topology: DeviceTopology
    profile: object
    mode: str
    max_degree: int | None
    ops: list[str]
    rank: dict
    devices: list[str]
    dev_index: dict
    kinds: list[str]
    link_pairs: list[tuple[str, str]]
    link_names: list[str]
    maps: list[list[tuple[int, ...]]]
    map_index: list[dict]
    n_enum: list[int]
    slot_off: np.ndarray
    pairs: list[tuple[int, int]]
    arrays: dict = field(default_factory=dict)
    ready_capacity: int = 128
    device: int = 0
    _handle: object = None
    fingerprint: tuple = ()

    # -- device handle ---------------------------------------------------------
    @property
    def n_ops(self) -> int:
        return len(self.ops)

    @property
    def n_slots(self) -> int:
        return int(self.slot_off[-1])

    def queue_name(self, q: int) -> str:
        return self.devices[q] if q < len(self.devices) else self.link_names[q - len(self.devices)]

    def handle(self):
        if self._handle is None:
            L = nat.lib()
            a = self.arrays

            def p(name, ct=ctypes.c_int32):
                return a[name].ctypes.data_as(ctypes.POINTER(ct))

            d = nat.PsProblemDesc()
            d.abi_version = nat.ABI_VERSION
            d.n_ops, d.n_devices, d.n_kinds = len(self.ops), len(self.devices), len(self.kinds)
            d.n_links, d.n_pairs, d.n_maps = len(self.link_pairs), len(self.pairs), int(a["map_size"].size)
            d.mode_full = 1 if self.mode == MODE_FULL else 0
            d.n_slots = self.n_slots
            d.ready_capacity = self.ready_capacity
            for name in ("dev_kind", "link_of", "op_ndim", "op_esize", "op_param_mask", "op_map_off",
                         "op_nmaps_enum", "op_slot_off", "slot_op", "op_in_off", "op_in_pairs", "op_out_off",
                         "op_out_pairs", "map_deg", "map_size", "map_ngroups", "pair_src", "pair_dst",
                         "pair_need_off", "need", "combo_off", "combo_row_off", "combo_col_off"):
                setattr(d, name, p(name))
            for name in ("link_bw", "link_lat", "exe_fwd", "exe_bwd", "map_shard"):
                setattr(d, name, p(name, ctypes.c_double))
            d.op_dim = p("op_dim", ctypes.c_int64)
            d.backward_multiplier = float(self.profile.backward_multiplier)
            h = ctypes.c_void_p()
            nat.check(L.ps_problem_create(ctypes.byref(d), self.device, ctypes.byref(h)), "ps_problem_create")
            self._handle = h
        return self._handle

    def close(self):
        if self._handle is not None:
            nat.lib().ps_problem_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> nat.PsProblemInfo:
        out = nat.PsProblemInfo()
        nat.check(nat.lib().ps_problem_info_get(self.handle(), ctypes.byref(out)), "ps_problem_info_get")
        return out

    # -- strategies --------------------------------------------------------------
    def has_maps_for(self, strategy) -> bool:
        for oid in self.ops:
            op = self.graph.ops[oid]
            if degree_tuple(op, strategy.configs[oid].degrees) not in self.map_index[self.rank[oid]]:
                return False
        return True

    def encode(self, strategy, out_map=None, out_asg=None):
        """(map_local int32[n_ops], assign uint8[n_slots]) for a strategy."""
        m = np.zeros(len(self.ops), dtype=np.int32) if out_map is None else out_map
        a = np.zeros(self.n_slots, dtype=np.uint8) if out_asg is None else out_asg
        for r, oid in enumerate(self.ops):
            cfg = strategy.configs.get(oid)
            if cfg is None:
                raise KeyError(oid)
            op = self.graph.ops[oid]
            t = degree_tuple(op, cfg.degrees)
            mi = self.map_index[r].get(t)
            if mi is None:
                raise KeyError(f"degree map {t} of op {oid} is not in the lowered problem")
            m[r] = mi
            size = math.prod(t)
            if cfg.assignment is None or len(cfg.assignment) < size:
                raise IndexError(f"op {oid}: assignment must list {size} devices")
            base = int(self.slot_off[r])
            for k in range(size):
                a[base + k] = self.dev_index[cfg.assignment[k]]
        return m, a

    def decode(self, map_local, assign, template=None):
        """ParallelizationStrategy from device-side arrays.  Degree dicts follow
        ``template``'s key sets where it has that map, else enumerate_configs'."""
        from .partition import ParallelizationStrategy
        configs = {}
        for r, oid in enumerate(self.ops):
            op = self.graph.ops[oid]
            t = self.maps[r][int(map_local[r])]
            names = op.output_shape.names()
            tmpl = template.configs.get(oid) if template is not None else None
            if tmpl is not None and degree_tuple(op, tmpl.degrees) == t:
                degrees = {n: t[names.index(n)] for n in tmpl.degrees}
            else:
                pd = parallelizable_dims(op)
                degrees = {n: t[i] for i, n in enumerate(names) if n in pd}
            base = int(self.slot_off[r])
            asg = tuple(self.devices[int(assign[base + k])] for k in range(math.prod(t)))
            configs[oid] = ParallelizationConfig(degrees, asg)
        return ParallelizationStrategy(configs)


def lower(g: OperatorGraph, topo: DeviceTopology, profile, mode: str, max_degree: int | None = None,
          strategies=(), ready_capacity: int = 128, device: int = 0, quiet_extra: bool = False) -> Lowered:
    """Flatten a problem.  ``max_degree`` adds every enumerate_configs map (the
    MCMC proposal space); ``strategies`` adds the maps those strategies use.
    ``quiet_extra``: maps no given strategy uses are priced without inserting
    into ``profile.entries`` (a build then leaves the profile as the reference's
    build of those strategies would; update_task_graph inserts a map's entry
    when a strategy first uses it)."""
    if mode not in (MODE_FORWARD, MODE_FULL):
        raise ValueError(f"unknown mode {mode!r}")
    ops = sorted(g.ops)
    rank = {oid: i for i, oid in enumerate(ops)}
    devices = topo.device_ids()
    dev_index = {d: i for i, d in enumerate(devices)}
    if len(devices) > 64:
        raise ValueError("the GPU path supports at most 64 devices per topology")
    if len(ops) >= 65535:
        raise ValueError("the GPU path supports at most 65534 operations")
    kinds = sorted({topo.devices[d].kind for d in devices})
    kind_index = {k: i for i, k in enumerate(kinds)}
    dev_of_kind = {}
    for d in devices:
        dev_of_kind.setdefault(topo.devices[d].kind, topo.devices[d])
    full = mode == MODE_FULL
    g.topological_order()  # ValueError on a cycle, before any device work

    # links: one queue per connected unordered device pair
    D = len(devices)
    link_of = np.full(D * D, -1, dtype=np.int32)
    link_pairs, link_names, bw, lat = [], [], [], []
    for i in range(D):
        for j in range(i + 1, D):
            c = topo.connection_between(devices[i], devices[j])
            if c is None:
                continue
            li = len(link_pairs)
            link_pairs.append((devices[i], devices[j]))
            a, b = c.key()
            link_names.append(f"link:{a}|{b}")
            bw.append(float(c.bandwidth))
            lat.append(float(c.latency))
            link_of[i * D + j] = link_of[j * D + i] = li

    # degree maps per op
    maps: list[list[tuple[int, ...]]] = []
    map_index: list[dict] = []
    n_enum: list[int] = []
    used: list[set] = []  # per op: the maps some given strategy uses
    for oid in ops:
        op = g.ops[oid]
        lst = []
        if max_degree is not None:
            lst = [degree_tuple(op, c.degrees) for c in enumerate_configs(op, topo, max_degree)]
        n_enum.append(len(lst))
        idx = {t: i for i, t in enumerate(lst)}
        seen = {}  # id(degrees dict) -> tuple: batched strategies share their dicts
        used_r = set()
        used.append(used_r)
        for s in strategies:
            cfg = s.configs.get(oid)
            if cfg is None:
                continue
            t = seen.get(id(cfg.degrees))
            if t is None:
                t = seen[id(cfg.degrees)] = degree_tuple(op, cfg.degrees)
                used_r.add(t)
            if t not in idx:
                grid_of(op, ParallelizationConfig(dict(zip(op.output_shape.names(), t))))  # divisibility
                idx[t] = len(lst)
                lst.append(t)
        if not lst:
            t = tuple(1 for _ in op.output_shape.dims)
            idx[t] = 0
            lst.append(t)
        maps.append(lst)
        map_index.append(idx)

    n_ops = len(ops)
    op_map_off = np.zeros(n_ops + 1, dtype=np.int32)
    op_map_off[1:] = np.cumsum([len(m) for m in maps])
    n_maps = int(op_map_off[-1])
    map_deg = np.ones((n_maps, 5), dtype=np.int32)
    map_size = np.zeros(n_maps, dtype=np.int32)
    exe_fwd = np.zeros((n_maps, len(kinds)), dtype=np.float64)
    exe_bwd = np.zeros((n_maps, len(kinds)), dtype=np.float64)
    map_shard = np.zeros(n_maps, dtype=np.float64)
    map_ngroups = np.ones(n_maps, dtype=np.int32)
    op_ndim = np.zeros(n_ops, dtype=np.int32)
    op_dim = np.ones((n_ops, 5), dtype=np.int64)
    op_esize = np.zeros(n_ops, dtype=np.int32)
    op_param_mask = np.full(n_ops, -1, dtype=np.int32)
    mult = profile.backward_multiplier
    max_size = np.zeros(n_ops, dtype=np.int64)
    for r, oid in enumerate(ops):
        op = g.ops[oid]
        names = op.output_shape.names()
        if len(names) > 5:
            raise ValueError(f"op {oid}: more than 5 output dims")
        op_ndim[r] = len(names)
        op_dim[r, :len(names)] = op.output_shape.sizes()
        op_esize[r] = op.output_shape.element_size
        classes = parallelizable_dims(op)
        pmask = 0
        for i, n in enumerate(names):
            if classes.get(n) == "parameter":
                pmask |= 1 << i
        if full and op.param_bytes > 0:
            op_param_mask[r] = pmask
        for mi, t in enumerate(maps[r]):
            gi = int(op_map_off[r]) + mi
            map_deg[gi, :len(t)] = t
            size = math.prod(t)
            map_size[gi] = size
            max_size[r] = max(max_size[r], size)
            cfg = ParallelizationConfig(dict(zip(names, t)))
            region0 = output_region(op, cfg, 0)
            quiet = quiet_extra and t not in used[r]
            for kname, ki in kind_index.items():
                if quiet:
                    key = cost_key_for(op, region0, kname)
                    e = profile.entries.get(key)
                    if e is None:
                        e = profile.fallback.time(op, key)
                else:
                    e = profile.task_exe_time(op, region0, dev_of_kind[kname])
                if not e >= 0.0:
                    # the reference would schedule a negative (or NaN) time; its heap order
                    # is then no longer monotone in ready time, which the GPU replay assumes
                    raise ValueError(f"op {oid}: task time {e!r} for {kname} is negative or NaN; "
                                     "the GPU path needs non-negative task times")
                exe_fwd[gi, ki] = e
                exe_bwd[gi, ki] = e * mult
            if op_param_mask[r] >= 0:
                groups = math.prod(t[i] for i in range(len(t)) if pmask >> i & 1)
                map_ngroups[gi] = groups
                map_shard[gi] = op.param_bytes / (groups or 1)
    if max_size.max(initial=0) > 255:
        raise ValueError("degree maps with more than 255 tasks are not supported")
    slot_off = np.zeros(n_ops + 1, dtype=np.int32)
    slot_off[1:] = np.cumsum(max_size)
    slot_op = np.repeat(np.arange(n_ops, dtype=np.int32), max_size)

    # op pairs in tensor order, with need descriptors per tensor edge
    pair_id: dict = {}
    pairs: list[tuple[int, int]] = []
    pair_edges: list[list] = []
    for e in g.tensors:
        if e.src not in rank or e.dst not in rank:
            raise KeyError(e.src if e.src not in rank else e.dst)
        key = (rank[e.src], rank[e.dst])
        if key not in pair_id:
            pair_id[key] = len(pairs)
            pairs.append(key)
            pair_edges.append([])
        pair_edges[pair_id[key]].append(e)
    need_rows = []
    pair_need_off = [0]
    for (s, d), edges in zip(pairs, pair_edges):
        src_op, dst_op = g.ops[ops[s]], g.ops[ops[d]]
        multi = dst_op.kind.tag in ("ElementWise", "Concat")
        for e in edges:
            if e.dst_slot < 0 or e.dst_slot >= (len(dst_op.input_shapes) if multi else 1):
                continue  # the reference's needs.get(slot) is None for these
            descs = {dn.name: dn for dn in need_descriptors(dst_op, e.dst_slot)}
            row = np.zeros((5, 8), dtype=np.int32)
            for j, (n, _) in enumerate(src_op.output_shape.dims):
                dn = descs[n]  # KeyError exactly where the reference's need[name] fails
                row[j] = (dn.mode, dn.out_dim, dn.extent, dn.kernel, dn.stride, dn.pad, dn.offset, 0)
            need_rows.append(row)
        pair_need_off.append(len(need_rows))
    need = np.stack(need_rows) if need_rows else np.zeros((0, 5, 8), dtype=np.int32)

    n_pairs = len(pairs)
    in_lists = [[] for _ in range(n_ops)]
    out_lists = [[] for _ in range(n_ops)]
    for p, (s, d) in enumerate(pairs):
        out_lists[s].append(p)
        in_lists[d].append(p)

    def csr(lists):
        off = np.zeros(n_ops + 1, dtype=np.int32)
        off[1:] = np.cumsum([len(x) for x in lists])
        flat = np.array([p for x in lists for p in x] or [0], dtype=np.int32)
        return off, flat

    op_in_off, op_in_pairs = csr(in_lists)
    op_out_off, op_out_pairs = csr(out_lists)

    combo_counts = np.array([len(maps[s]) * len(maps[d]) for s, d in pairs], dtype=np.int64)
    combo_off = np.zeros(n_pairs + 1, dtype=np.int64)
    combo_off[1:] = np.cumsum(combo_counts)
    rows, cols = [], []
    for s, d in pairs:
        ss = map_size[op_map_off[s]:op_map_off[s + 1]].astype(np.int64)
        ds = map_size[op_map_off[d]:op_map_off[d + 1]].astype(np.int64)
        rows.append(np.repeat(ss, len(ds)))
        cols.append(np.tile(ds, len(ss)))
    rows = np.concatenate(rows) if rows else np.zeros(0, dtype=np.int64)
    cols = np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)
    combo_row_off = np.zeros(rows.size + 1, dtype=np.int64)
    combo_row_off[1:] = np.cumsum(rows)
    combo_col_off = np.zeros(cols.size + 1, dtype=np.int64)
    combo_col_off[1:] = np.cumsum(cols)
    if combo_row_off[-1] >= 2 ** 31 - 1 or combo_col_off[-1] >= 2 ** 31 - 1 or combo_off[-1] >= 2 ** 31 - 1:
        raise ValueError("problem too large for 32-bit table offsets")

    arrays = {
        "dev_kind": np.array([kind_index[topo.devices[d].kind] for d in devices], dtype=np.int32),
        "link_of": link_of,
        "link_bw": np.array(bw or [1.0], dtype=np.float64),
        "link_lat": np.array(lat or [0.0], dtype=np.float64),
        "op_ndim": op_ndim, "op_dim": np.ascontiguousarray(op_dim.reshape(-1)), "op_esize": op_esize,
        "op_param_mask": op_param_mask, "op_map_off": op_map_off,
        "op_nmaps_enum": np.array(n_enum, dtype=np.int32), "op_slot_off": slot_off, "slot_op": slot_op,
        "op_in_off": op_in_off, "op_in_pairs": op_in_pairs, "op_out_off": op_out_off, "op_out_pairs": op_out_pairs,
        "map_deg": np.ascontiguousarray(map_deg.reshape(-1)), "map_size": map_size,
        "exe_fwd": np.ascontiguousarray(exe_fwd.reshape(-1)), "exe_bwd": np.ascontiguousarray(exe_bwd.reshape(-1)),
        "map_shard": map_shard, "map_ngroups": map_ngroups,
        "pair_src": np.array([s for s, _ in pairs] or [0], dtype=np.int32),
        "pair_dst": np.array([d for _, d in pairs] or [0], dtype=np.int32),
        "pair_need_off": np.array(pair_need_off, dtype=np.int32),
        "need": np.ascontiguousarray(need.reshape(-1)) if need.size else np.zeros(8, dtype=np.int32),
        "combo_off": combo_off.astype(np.int32), "combo_row_off": combo_row_off.astype(np.int32),
        "combo_col_off": combo_col_off.astype(np.int32),
    }
    return Lowered(graph=g, topology=topo, profile=profile, mode=mode, max_degree=max_degree, ops=ops, rank=rank,
                   devices=devices, dev_index=dev_index, kinds=kinds, link_pairs=link_pairs, link_names=link_names,
                   maps=maps, map_index=map_index, n_enum=n_enum, slot_off=slot_off, pairs=pairs, arrays=arrays,
                   ready_capacity=ready_capacity, device=device)


def origin_of(low: Lowered, key: int) -> tuple:
    """Packed origin key -> the reference's origin tuple."""
    kind = key >> 61
    a, b, c, d = (key >> 45) & 0xFFFF, (key >> 29) & 0xFFFF, (key >> 14) & 0x7FFF, key & 0x3FFF
    name = KIND_NAMES[kind]
    if name in ("op", "op_bwd"):
        return (name, low.ops[a], c)
    if name in ("edge", "edge_bwd"):
        return (name, low.ops[a], low.ops[b], c, d)
    return (name, low.ops[a], b, c)
