"""Test infrastructure: serialise parasim-API objects for the C oracle and call it.

Duck-typed over the reference package's objects and ours alike (``ops``,
``tensors``, ``topological_order()``, ``devices``, ``connection_between``,
``configs`` ...), so the same problem text can be produced from either side.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module; the product never does.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libparasim_oracle.so")

TAGS = ("MatMul", "Conv1D", "Conv2D", "Pool1D", "Pool2D", "Embedding", "ElementWise", "Concat")
DIMS = ("sample", "channel", "length", "height", "width")
KIND_NAMES = ("edge", "edge_bwd", "op", "op_bwd", "sync")


def build_oracle(force: bool = False) -> str:
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    src = os.path.join(HERE, "parasim_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", LIB_PATH,
                               src, "-lm", "-lpthread"])
    return LIB_PATH


def _hex(x: float) -> str:
    return float(x).hex()


def _shape(s) -> str:
    return f"{s.element_size} {len(s.dims)} " + " ".join(f"{DIMS.index(n)} {sz}" for n, sz in s.dims)


def _digest(op) -> str:
    doc = {"tag": op.kind.tag, "hp": sorted(op.kind.hyperparams.items()),
           "inputs": [[list(s.dims), s.element_size] for s in op.input_shapes]}
    return hashlib.md5(json.dumps(doc, sort_keys=True, separators=(",", ":")).encode()).hexdigest()[:12]


def problem_text(g, topo, profile, mode: str) -> str:
    ops = sorted(g.ops)
    rank = {oid: i for i, oid in enumerate(ops)}
    devs = topo.device_ids()
    kinds = sorted({topo.devices[d].kind for d in devs})
    fb = profile.fallback
    out = ["parasim-oracle 1", f"mode {1 if mode == 'full-iteration' else 0}",
           f"mult {_hex(profile.backward_multiplier)}",
           f"cost {_hex(fb.default_throughput)} {_hex(fb.overhead)}",
           f"kinds {len(kinds)}"]
    for k in kinds:
        out.append(f"{k} {_hex(fb.throughput[k]) if k in fb.throughput else 'nan'}")
    out.append(f"devices {len(devs)}")
    out += [f"{d} {kinds.index(topo.devices[d].kind)}" for d in devs]
    links = []
    for i, a in enumerate(devs):
        for j in range(i + 1, len(devs)):
            c = topo.connection_between(a, devs[j])
            if c is not None:
                links.append(f"{i} {j} {_hex(c.bandwidth)} {_hex(c.latency)}")
    out.append(f"links {len(links)}")
    out += links
    out.append(f"ops {len(ops)}")
    for oid in ops:
        op = g.ops[oid]
        hp = op.kind.hp
        axis = hp("axis")
        out.append(" ".join(str(v) for v in (
            "op", oid, TAGS.index(op.kind.tag), op.param_bytes,
            hp("kernel_h", 1), hp("kernel_w", 1), hp("stride_h", 1), hp("stride_w", 1),
            1 if hp("padding", "same") == "valid" else 0, hp("kernel", 1), hp("stride", 1),
            DIMS.index(axis) if axis in DIMS else -1)))
        out.append(_shape(op.output_shape))
        out.append(f"{len(op.input_shapes)} " + " ".join(_shape(s) for s in op.input_shapes))
    out.append(f"edges {len(g.tensors)}")
    out += [f"{rank[e.src]} {rank[e.dst]} {e.dst_slot}" for e in g.tensors]
    order = g.topological_order()
    out.append(f"topo {len(order)} " + " ".join(str(rank[o]) for o in order))
    over = []
    digests = {oid: _digest(g.ops[oid]) for oid in ops}
    for key, seconds in profile.entries.items():
        if key.device_kind not in kinds:
            continue
        for oid in ops:
            op = g.ops[oid]
            if op.kind.tag == key.kind and digests[oid] == key.digest and \
                    tuple(n for n, _ in key.region_dims) == op.output_shape.names():
                over.append(f"{rank[oid]} {kinds.index(key.device_kind)} {len(key.region_dims)} "
                            + " ".join(str(s) for _, s in key.region_dims) + f" {_hex(seconds)}")
    out.append(f"overrides {len(over)}")
    out += over
    return "\n".join(out) + "\n"


def _cfg_text(g, topo, oid, cfg) -> str:
    devs = topo.device_ids()
    op = g.ops[oid]
    degs = [cfg.degrees.get(n, 1) for n in op.output_shape.names()]
    asg = [devs.index(d) for d in cfg.assignment]
    return f"{len(degs)} " + " ".join(map(str, degs)) + f" {len(asg)} " + " ".join(map(str, asg))


def strategy_text(g, topo, strategy) -> str:
    return " ".join(_cfg_text(g, topo, oid, strategy.configs[oid]) for oid in sorted(g.ops))


class Oracle:
    """ctypes front end to oracle/_build/libparasim_oracle.so."""

    def __init__(self):
        self.lib = ctypes.CDLL(build_oracle())
        L = self.lib
        L.orc_simulate.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_long]
        L.orc_simulate_batch.argtypes = [ctypes.c_char_p, ctypes.c_char_p,
                                         ctypes.POINTER(ctypes.c_double), ctypes.c_int]
        L.orc_mcmc.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, ctypes.c_double, ctypes.c_int,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_int]
        L.orc_rng_words.argtypes = [ctypes.c_int, ctypes.c_ulonglong, ctypes.c_int, ctypes.c_void_p]
        L.orc_set_deadline.argtypes = [ctypes.c_double]
        L.orc_set_deadline.restype = None

    def simulate(self, g, topo, profile, mode, strategy, cap=1 << 26) -> dict:
        """Full build + simulate of one strategy.  Returns makespan, counts and
        an origin-keyed timeline {origin tuple: (ready, start, end, queue, exe, nbytes)}."""
        buf = ctypes.create_string_buffer(cap)
        rc = self.lib.orc_simulate(problem_text(g, topo, profile, mode).encode(),
                                   ("strategy " + strategy_text(g, topo, strategy)).encode(), buf, cap)
        text = buf.value.decode()
        ops = sorted(g.ops)
        res = {"rc": rc, "timeline": {}}
        for line in text.splitlines():
            f = line.split()
            if f[0] == "makespan":
                res["makespan"] = float.fromhex(f[1])
            elif f[0] == "tasks":
                res["tasks"] = int(f[1])
            elif f[0] == "edges":
                res["edges"] = int(f[1])
            elif f[0] == "comm":
                res["comm_tasks"] = int(f[1])
                res["comm_bytes"] = float.fromhex(f[2])
            elif f[0] == "error":
                devs = topo.device_ids()
                res["noroute"] = (devs[int(f[2])], devs[int(f[3])])
            elif f[0] == "t":
                kind, a, b, c, d = int(f[1]), int(f[2]), int(f[3]), int(f[4]), int(f[5])
                name = KIND_NAMES[kind]
                if name in ("op", "op_bwd"):
                    origin = (name, ops[a], c)
                elif name in ("edge", "edge_bwd"):
                    origin = (name, ops[a], ops[b], c, d)
                else:
                    origin = (name, ops[a], b, c)
                res["timeline"][origin] = (float.fromhex(f[9]), float.fromhex(f[10]), float.fromhex(f[11]),
                                           int(f[6]), float.fromhex(f[7]), float.fromhex(f[8]))
        return res

    def makespans(self, g, topo, profile, mode, strategies) -> np.ndarray:
        text = f"strategies {len(strategies)}\n" + "\n".join(strategy_text(g, topo, s) for s in strategies)
        out = np.zeros(len(strategies), dtype=np.float64)
        rc = self.lib.orc_simulate_batch(problem_text(g, topo, profile, mode).encode(), text.encode(),
                                         out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 1)
        assert rc == 0, rc
        return out

    def mcmc(self, g, topo, profile, mode, initial, seeds, max_proposals, max_degree,
             rng_mode="philox", beta=None, threads=1, deadline_s=None) -> dict:
        """polish=False MCMC, one chain per (initial strategy, seed).  ``deadline_s``
        (bounded baseline samples only) stops every chain between proposals once
        that much wall time has passed; summary[:, 2] says how far each got."""
        n = len(initial)
        nops = len(g.ops)
        maxsize = max(max(c.size() for c in s.configs.values()) for s in initial)
        maxsize = max(maxsize, max_degree, 1)
        text = f"chains {n}\n" + "\n".join(f"{seed} " + strategy_text(g, topo, s)
                                           for s, seed in zip(initial, seeds))
        summary = np.zeros((n, 6))
        cand = np.zeros((n, max(1, max_proposals)))
        ok = np.zeros((n, max(1, max_proposals)), dtype=np.uint8)
        bdeg = np.zeros((n, nops, 5), dtype=np.int32)
        basg = np.full((n, nops, maxsize), -1, dtype=np.int32)
        self.lib.orc_set_deadline(float(deadline_s or 0.0))
        rc = self.lib.orc_mcmc(problem_text(g, topo, profile, mode).encode(), text.encode(), max_proposals,
                               max_degree, 1 if rng_mode == "philox" else 0, beta is not None,
                               float(beta or 0.0), threads, summary.ctypes.data, cand.ctypes.data,
                               ok.ctypes.data, bdeg.ctypes.data, basg.ctypes.data, maxsize)
        self.lib.orc_set_deadline(0.0)
        assert rc == 0, rc
        return {"summary": summary, "cand": cand, "ok": ok, "best_deg": bdeg, "best_asg": basg}

    def rng_words(self, mode: str, seed: int, n: int) -> list[int]:
        out = np.zeros(n, dtype=np.uint32)
        self.lib.orc_rng_words(1 if mode == "philox" else 0, seed, n, out.ctypes.data)
        return [int(x) for x in out]
