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
