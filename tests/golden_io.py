"""Loaders for tests/golden (fixtures generated from the reference by
scripts/make_golden.py)."""

import json
import os

import paper_1807_05358_b200 as ps

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def inputs(doc):
    g = ps.graph_from_json(doc["graph"])
    topo = ps.topology_from_json(doc["topology"])
    strategies = [ps.strategy_from_json(s) for s in doc["strategies"]]
    return g, topo, strategies


def fx(h):
    return float.fromhex(h)


def timeline_of(rec):
    """origin-string tuple -> (start, end, device)."""
    return {tuple(o): (fx(s), fx(e), d) for o, s, e, d in rec["timeline"]}


def origin_strings(origin):
    return tuple(map(str, origin))


def timeline_digest(table) -> str:
    """sha256 over the sorted (origin, start, end, device) rows of a
    timeline_table -- the digest scripts/make_golden.py records from the reference."""
    import hashlib
    rows = sorted((repr(tuple(o)), float(s).hex(), float(e).hex(), d) for o, (s, e, d) in table.items())
    return hashlib.sha256(json.dumps(rows, separators=(",", ":")).encode()).hexdigest()


def graph_digest(doc) -> str:
    import hashlib
    return hashlib.sha256(json.dumps(doc, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def queue_names(topo):
    """Oracle queue index -> device id / 'link:a|b' (devices, then links in (i < j) order)."""
    devs = topo.device_ids()
    names = list(devs)
    for i, a in enumerate(devs):
        for b in devs[i + 1:]:
            c = topo.connection_between(a, b)
            if c is not None:
                x, y = c.key()
                names.append(f"link:{x}|{y}")
    return names


def large_inputs(doc):
    """Graph / topology / strategies of a simulate_large.json case, rebuilt with
    this package's generators and checked against the digest the reference saw."""
    from paper_1807_05358_b200 import workloads as W
    gens = {"resnet101_16x4": lambda: W.resnet101(),
            "nmt40_16x4": lambda: W.nmt_like(steps=40, layers=2, batch=64, hidden=1024, vocab=32768),
            "random1k_4x4": lambda: W.random_dag(1000, seed=1000),
            "random10k_4x4": lambda: W.random_dag(10000, seed=1000)}
    text = ps.graph_to_json(gens[doc["name"]]())
    assert graph_digest(text) == doc["graph_sha256"], doc["name"]
    # through JSON, as the reference read it: ops in id order, which sets the
    # topological order and with it task creation order (total_comm_bytes sums)
    g = ps.graph_from_json(text)
    topo = ps.topology_from_json(doc["topology"])
    md = doc["max_degree"]
    strategies = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, md, s)
                                                        for s in doc["random_seeds"]]
    return g, topo, strategies
