#!/usr/bin/env python3
"""Generate tests/golden/*.json from the REFERENCE implementation itself.

Run in the build container only (needs the read-only reference checkout):

    PYTHONDONTWRITEBYTECODE=1 python scripts/make_golden.py

Every fixture carries its inputs as the reference's own JSON documents
(formats.py FORMAT_VERSION 1) so the tests can rebuild identical inputs on a
machine without the reference, and the outputs the reference produced:
makespans / counts / timelines as float.hex, MCMC chain summaries and traces
(unmodified MT19937 and with PhiloxRandom injected as the module's Random).
"""

import json
import os
import random
import sys
import types

REF = "/root/reference/pkg"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
sys.path.insert(0, ROOT)

import parasim as R  # noqa: E402  (the reference)
import parasim.search as RS  # noqa: E402
from helpers import random_graph, random_topology  # noqa: E402  (reference test helpers)

from paper_1807_05358_b200.rng import PhiloxRandom  # noqa: E402  (stream under test)
from paper_1807_05358_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
H = float.hex


def sim_record(g, topo, strategy, mode, with_timeline=True):
    prof = R.CostProfile()
    tg = R.build_task_graph(g, topo, strategy, prof, mode)
    res = R.full_simulate(tg)
    rec = {"makespan": H(res.makespan), "oracle_makespan": H(R.oracle_simulate(tg)),
           "tasks": len(tg.tasks), "comm_tasks": sum(1 for t in tg.tasks.values() if t.kind == "comm"),
           "edges": sum(len(t.outputs) for t in tg.tasks.values()),
           "comm_bytes": H(float(tg.total_comm_bytes))}
    if with_timeline:
        rec["timeline"] = sorted([list(map(str, o)), H(s), H(e), d] for o, (s, e, d) in R.timeline_table(tg).items())
    return rec


def case_doc(g, topo, strategies, mode, md=None):
    return {"graph": R.graph_to_json(g), "topology": R.topology_to_json(topo), "mode": mode, "max_degree": md,
            "strategies": [R.strategy_to_json(s) for s in strategies]}


def simulate_cases():
    cases = []
    for seed in range(40):
        rng = random.Random(50000 + seed)
        g = random_graph(rng, 4, 14)
        topo = random_topology(rng, rng.choice((2, 4, 8, 16)))
        mode = R.MODE_FULL if seed % 2 else R.MODE_FORWARD
        md = rng.choice((2, 3, 4))
        strategies = [R.data_parallel_strategy(g, topo)] + [R.random_strategy(g, topo, md, seed * 10 + i)
                                                           for i in range(3)]
        doc = case_doc(g, topo, strategies, mode, md)
        doc["results"] = [sim_record(g, topo, s, mode) for s in strategies]
        cases.append(doc)
    return cases


def benchmark_cases():
    out = []
    specs = [("alexnet_like", W.alexnet_like(), W.single_node_topology(4), 4),
             ("inception_v3", W.inception_v3(), W.multi_node_topology(4, 4), 4),
             ("nmt_like_8", W.nmt_like(steps=8, layers=2, batch=64, hidden=1024, vocab=32768),
              W.multi_node_topology(4, 4), 8)]
    for name, g0, t0, md in specs:
        # round-trip through the reference's own formats so both sides read identical docs
        g = R.graph_from_json(W_json(g0))
        topo = R.topology_from_json(W_topo_json(t0))
        strategies = [R.data_parallel_strategy(g, topo)] + [R.random_strategy(g, topo, md, s) for s in range(2)]
        for mode in (R.MODE_FORWARD, R.MODE_FULL):
            doc = case_doc(g, topo, strategies, mode, md)
            doc["name"] = name
            doc["results"] = [sim_record(g, topo, s, mode, with_timeline=False) for s in strategies]
            out.append(doc)
    return out


def W_json(g):
    from paper_1807_05358_b200.formats import graph_to_json
    return graph_to_json(g)


def W_topo_json(t):
    from paper_1807_05358_b200.formats import topology_to_json
    return topology_to_json(t)


def mcmc_cases():
    out = []
    for seed in range(6):
        rng = random.Random(70000 + seed)
        g = random_graph(rng, 4, 10)
        topo = random_topology(rng, rng.choice((2, 4, 8)))
        mode = R.MODE_FULL if seed % 2 else R.MODE_FORWARD
        md = rng.choice((2, 4))
        init = [R.data_parallel_strategy(g, topo), R.random_strategy(g, topo, md, seed)]
        for rng_name in ("mt19937", "philox"):
            RS.random = types.SimpleNamespace(Random=PhiloxRandom) if rng_name == "philox" else random
            try:
                rep = R.mcmc_search(g, topo, R.CostProfile(), R.SearchParams(
                    max_proposals=100, seed=seed, max_degree=md, mode=mode, initial=init, polish=False))
            finally:
                RS.random = random
            doc = case_doc(g, topo, init, mode, md)
            doc.update({"rng": rng_name, "seed": seed, "max_proposals": 100,
                        "chains": [[H(c.initial_cost), H(c.best_cost), c.proposals, c.accepted, H(c.beta),
                                    c.termination] for c in rep.chains],
                        "trace": [[i, H(c), bool(a)] for i, c, a in rep.trace],
                        "best_cost": H(rep.best_cost),
                        "best_strategy": R.strategy_to_json(rep.best_strategy)})
            out.append(doc)
    return out


def search_report_cases():
    """Default mcmc_search (MT19937, polish on) -> the reference's own report JSON."""
    out = []
    tiny = R.OperatorGraph()
    tiny.add_op(R.Operation("a", R.OperatorKind("MatMul"), (R.shape(("sample", 4), ("channel", 4)),),
                            R.shape(("sample", 4), ("channel", 4)), param_bytes=64))
    tiny.add_op(R.Operation("b", R.OperatorKind("MatMul"), (R.shape(("sample", 4), ("channel", 4)),),
                            R.shape(("sample", 4), ("channel", 2)), param_bytes=32))
    tiny.add_tensor("a", "b")
    cases = [("tiny", tiny, R.single_node_topology(gpus=2), 2, R.MODE_FORWARD, 120, 5),
             ("lenet", R.lenet_like(batch=2, image=4, in_channels=1, conv_channels=(2, 2), fc_hidden=2, classes=2),
              R.single_node_topology(gpus=2), 2, R.MODE_FORWARD, 80, 4),
             ("rnn3-full", R.rnn3(steps=2, batch=4, hidden=4, vocab=4), R.single_node_topology(gpus=3), 2,
              R.MODE_FULL, 60, 1)]
    for name, g, topo, md, mode, props, seed in cases:
        rep = R.mcmc_search(g, topo, R.CostProfile(), R.SearchParams(max_proposals=props, seed=seed,
                                                                      max_degree=md, mode=mode))
        out.append({"name": name, "graph": R.graph_to_json(g), "topology": R.topology_to_json(topo),
                    "mode": mode, "max_degree": md, "max_proposals": props, "seed": seed,
                    "report": R.report_to_json(rep)})
    return out


def exhaustive_cases():
    out = []
    tiny = R.OperatorGraph()
    tiny.add_op(R.Operation("a", R.OperatorKind("MatMul"), (R.shape(("sample", 4), ("channel", 4)),),
                            R.shape(("sample", 4), ("channel", 4)), param_bytes=64))
    tiny.add_op(R.Operation("b", R.OperatorKind("MatMul"), (R.shape(("sample", 4), ("channel", 4)),),
                            R.shape(("sample", 4), ("channel", 2)), param_bytes=32))
    tiny.add_tensor("a", "b")
    cases = [("tiny", tiny, R.single_node_topology(gpus=2), 2, R.MODE_FORWARD),
             ("tiny-full", tiny, R.single_node_topology(gpus=2), 2, R.MODE_FULL),
             ("lenet", R.lenet_like(batch=2, image=4, in_channels=1, conv_channels=(2, 2), fc_hidden=2, classes=2),
              R.single_node_topology(gpus=2), 2, R.MODE_FORWARD),
             ("rnnlm", R.rnnlm_like(steps=2, layers=1, batch=2, hidden=2, vocab=2), R.single_node_topology(gpus=2),
              2, R.MODE_FORWARD)]
    for name, g, topo, md, mode in cases:
        res = R.exhaustive_optimal(g, topo, R.CostProfile(), max_degree=md, cap=1e15, mode=mode)
        out.append({"name": name, "graph": R.graph_to_json(g), "topology": R.topology_to_json(topo), "mode": mode,
                    "max_degree": md, "cost": H(res.cost), "visited": res.visited,
                    "space_estimate": res.space_estimate, "strategy": R.strategy_to_json(res.strategy)})
    return out


def rnn3_case():
    g = R.rnn3()
    topo = R.single_node_topology(gpus=3)
    s = R.rnn3_model_parallel_strategy(g, topo)
    doc = case_doc(g, topo, [s], R.MODE_FORWARD)
    doc["results"] = [sim_record(g, topo, s, R.MODE_FORWARD)]
    with open(os.path.join(REF, "tests", "data", "rnn3_model_parallel.json")) as fh:
        doc["reference_fixture"] = json.load(fh)
    return doc


def timeline_digest(table) -> str:
    """sha256 over the sorted (origin, start, end, device) rows of timeline_table
    (tests/golden_io.timeline_digest computes the same on the GPU side)."""
    import hashlib
    rows = sorted((repr(tuple(o)), H(s), H(e), d) for o, (s, e, d) in table.items())
    return hashlib.sha256(json.dumps(rows, separators=(",", ":")).encode()).hexdigest()


def graph_digest(doc) -> str:
    import hashlib
    return hashlib.sha256(json.dumps(doc, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def large_cases():
    """The BASELINE configs at their full sizes (64 devices; 1k- and 10k-op random
    DAGs), simulated by the reference itself.  Inputs are generated by this
    package's workload generators (the reference has none for these shapes) and
    pinned by a digest of their JSON; outputs are makespans, counts and a digest
    of the whole timeline."""
    specs = [("resnet101_16x4", lambda: W.resnet101(), lambda: W.multi_node_topology(16, 4), 8, 3),
             ("nmt40_16x4", lambda: W.nmt_like(steps=40, layers=2, batch=64, hidden=1024, vocab=32768),
              lambda: W.multi_node_topology(16, 4), 8, 3),
             ("random1k_4x4", lambda: W.random_dag(1000, seed=1000), lambda: W.multi_node_topology(4, 4), 4, 3),
             ("random10k_4x4", lambda: W.random_dag(10000, seed=1000), lambda: W.multi_node_topology(4, 4), 4, 2)]
    out = []
    for name, mk_g, mk_t, md, n_rand in specs:
        gdoc, tdoc = W_json(mk_g()), W_topo_json(mk_t())
        g = R.graph_from_json(gdoc)
        topo = R.topology_from_json(tdoc)
        strategies = [R.data_parallel_strategy(g, topo)] + [R.random_strategy(g, topo, md, s) for s in range(n_rand)]
        for mode in (R.MODE_FORWARD, R.MODE_FULL):
            recs = []
            for st in strategies:
                tg = R.build_task_graph(g, topo, st, R.CostProfile(), mode)
                res = R.full_simulate(tg)
                recs.append({"makespan": H(res.makespan), "tasks": len(tg.tasks),
                             "comm_tasks": sum(1 for t in tg.tasks.values() if t.kind == "comm"),
                             "edges": sum(len(t.outputs) for t in tg.tasks.values()),
                             "comm_bytes": H(float(tg.total_comm_bytes)),
                             "timeline_sha256": timeline_digest(R.timeline_table(tg))})
                print(name, mode, recs[-1]["tasks"], flush=True)
            out.append({"name": name, "mode": mode, "max_degree": md, "graph_sha256": graph_digest(gdoc),
                        "topology": tdoc, "random_seeds": list(range(n_rand)), "results": recs})
    return out


def profile_cases():
    """Measured-profile path (cost.py:105-121,136-198): a profile text with
    entries for some keys (perturbed analytic times), a fallback with its own
    rate and a nonzero overhead for the rest, and a non-default backward
    multiplier; simulated by the reference."""
    out = []
    specs = [("alexnet_1x4", lambda: W.alexnet_like(), lambda: W.single_node_topology(4), 4),
             ("inception_4x4", lambda: W.inception_v3(), lambda: W.multi_node_topology(4, 4), 4)]
    for name, mk_g, mk_t, md in specs:
        gdoc, tdoc = W_json(mk_g()), W_topo_json(mk_t())
        g = R.graph_from_json(gdoc)
        topo = R.topology_from_json(tdoc)
        strategies = [R.data_parallel_strategy(g, topo)] + [R.random_strategy(g, topo, md, s) for s in range(4)]
        # measured entries: every third key the analytic model produces, times 1.37 / 0.61
        probe = R.CostProfile()
        for st in strategies:
            R.build_task_graph(g, topo, st, probe, R.MODE_FULL)
        keys = sorted(probe.entries, key=lambda k: (k.kind, k.digest, k.region_dims, k.device_kind))
        measured = R.CostProfile()
        for i, k in enumerate(keys):
            if i % 3 == 0:
                measured.entries[k] = probe.entries[k] * (1.37 if i % 2 else 0.61)
        text = R.dumps_profile(measured)
        fallback = {"throughput": {"gpu": 4.0e11}, "default_throughput": 1.0e12, "overhead": 3.5e-6}
        for mode in (R.MODE_FORWARD, R.MODE_FULL):
            prof = R.loads_profile(text, R.AnalyticCostModel(**fallback))
            prof.backward_multiplier = 2.5
            mks = [H(R.full_simulate(R.build_task_graph(g, topo, st, prof, mode)).makespan) for st in strategies]
            out.append({"name": name, "mode": mode, "max_degree": md, "graph": gdoc, "topology": tdoc,
                        "strategies": [R.strategy_to_json(s) for s in strategies], "profile_text": text,
                        "fallback": fallback, "backward_multiplier": 2.5, "makespans": mks,
                        "fallback_evaluations": prof.fallback_evaluations})
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    if "--large" in sys.argv:  # the full-size / measured-profile fixtures only
        docs = {"simulate_large.json": large_cases(), "profiles.json": profile_cases()}
        for name, doc in docs.items():
            with open(os.path.join(OUT, name), "w") as fh:
                json.dump(doc, fh, separators=(",", ":"))
            print("wrote", name, os.path.getsize(os.path.join(OUT, name)))
        return
    docs = {"rnn3_model_parallel.json": rnn3_case(), "simulate_random.json": simulate_cases(),
            "simulate_benchmarks.json": benchmark_cases(), "mcmc.json": mcmc_cases(),
            "search_reports.json": search_report_cases(), "exhaustive.json": exhaustive_cases()}
    for name, doc in docs.items():
        with open(os.path.join(OUT, name), "w") as fh:
            json.dump(doc, fh, separators=(",", ":"))
        print("wrote", name, os.path.getsize(os.path.join(OUT, name)))


if __name__ == "__main__":
    main()
