"""The C oracle against vectors produced by the reference itself (CPU only).

The oracle is the parity checker for the GPU path, so it is pinned first:
every makespan, count, byte total, timeline and MCMC trajectory in
tests/golden must come out identical."""

import pytest

import paper_1807_05358_b200 as ps
from golden_io import fx, inputs, load, origin_strings, timeline_of


def test_formats_round_trip_reference_documents():
    for doc in load("simulate_random.json")[:10] + load("simulate_benchmarks.json")[:2]:
        g, topo, strategies = inputs(doc)
        assert ps.graph_to_json(g) == doc["graph"]
        assert ps.topology_to_json(topo) == doc["topology"]
        assert [ps.strategy_to_json(s) for s in strategies] == doc["strategies"]


def test_rnn3_golden(oracle):
    doc = load("rnn3_model_parallel.json")
    g, topo, (s,) = inputs(doc)
    ref = doc["reference_fixture"]
    got = oracle.simulate(g, topo, ps.CostProfile(), doc["mode"], s)
    assert got["makespan"] == ref["oracle_makespan"] == 3.5826560000000005e-06
    assert got["tasks"] == ref["task_count"] and got["comm_tasks"] == ref["comm_task_count"]
    assert got["edges"] == ref["dependency_edge_count"] and got["comm_bytes"] == ref["comm_bytes_total"]


@pytest.mark.parametrize("name", ["simulate_random.json", "simulate_benchmarks.json"])
def test_oracle_matches_reference_simulations(oracle, name):
    for doc in load(name):
        g, topo, strategies = inputs(doc)
        for s, rec in zip(strategies, doc["results"]):
            got = oracle.simulate(g, topo, ps.CostProfile(), doc["mode"], s)
            assert got["makespan"] == fx(rec["makespan"]) == fx(rec["oracle_makespan"])
            assert (got["tasks"], got["comm_tasks"], got["edges"]) == (rec["tasks"], rec["comm_tasks"], rec["edges"])
            assert got["comm_bytes"] == fx(rec["comm_bytes"])
            if "timeline" in rec:
                want = timeline_of(rec)
                have = {origin_strings(o): (v[1], v[2]) for o, v in got["timeline"].items()}
                assert have == {o: (s_, e_) for o, (s_, e_, _) in want.items()}


def test_oracle_matches_reference_mcmc(oracle):
    for doc in load("mcmc.json"):
        g, topo, init = inputs(doc)
        n = doc["max_proposals"]
        got = oracle.mcmc(g, topo, ps.CostProfile(), doc["mode"], init,
                          [doc["seed"] + 1000003 * c for c in range(len(init))], n, doc["max_degree"],
                          rng_mode="mt" if doc["rng"] == "mt19937" else "philox")
        trace = doc["trace"]
        for ci, ch in enumerate(doc["chains"]):
            s = got["summary"][ci]
            assert (s[0], s[1], int(s[2]), int(s[3]), s[4]) == (fx(ch[0]), fx(ch[1]), ch[2], ch[3], fx(ch[4]))
            seg = trace[ci * n:(ci + 1) * n]
            assert [fx(c) for _, c, _ in seg] == list(got["cand"][ci])
            assert [a for _, _, a in seg] == [bool(x) for x in got["ok"][ci]]


def test_philox_known_answer_and_stream(oracle):
    from paper_1807_05358_b200.rng import PhiloxRandom, philox4x32_10
    assert philox4x32_10((0, 0, 0, 0), (0, 0)) == (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)
    r = PhiloxRandom(123456789)
    assert oracle.rng_words("philox", 123456789, 11) == [r.getrandbits(32) for _ in range(11)]


def test_mt19937_matches_cpython(oracle):
    import random
    for seed in (0, 1, 1000003, 2 ** 32 + 5):
        r = random.Random(seed)
        assert oracle.rng_words("mt", seed, 700) == [r.getrandbits(32) for _ in range(700)]


def _oracle_table(res, topo):
    names = __import__("golden_io").queue_names(topo)
    return {o: (v[1], v[2], names[v[3]]) for o, v in res["timeline"].items()}


@pytest.mark.parametrize("name", ["resnet101_16x4", "nmt40_16x4", "random1k_4x4", "random10k_4x4"])
def test_oracle_matches_reference_at_full_size(oracle, name):
    """The BASELINE configs at full size (64 devices, 1k/10k-op DAGs): makespan,
    counts, byte totals and the whole timeline (digest) equal the reference's."""
    from golden_io import large_inputs, timeline_digest
    for doc in (d for d in load("simulate_large.json") if d["name"] == name):
        g, topo, strategies = large_inputs(doc)
        for s, rec in zip(strategies, doc["results"]):
            got = oracle.simulate(g, topo, ps.CostProfile(), doc["mode"], s, cap=1 << 28)
            assert got["makespan"] == fx(rec["makespan"]), (name, doc["mode"])
            assert (got["tasks"], got["comm_tasks"], got["edges"]) == (rec["tasks"], rec["comm_tasks"], rec["edges"])
            assert got["comm_bytes"] == fx(rec["comm_bytes"])
            assert timeline_digest(_oracle_table(got, topo)) == rec["timeline_sha256"], (name, doc["mode"])


def _profile_of(doc):
    prof = ps.loads_profile(doc["profile_text"], ps.AnalyticCostModel(**doc["fallback"]))
    prof.backward_multiplier = doc["backward_multiplier"]
    return prof


def test_oracle_matches_reference_with_a_measured_profile(oracle):
    """Profile-text entries + a fallback with its own rate and overhead + a
    non-default backward multiplier (cost.py:105-121,136-198)."""
    for doc in load("profiles.json"):
        g, topo, strategies = inputs(doc)
        got = oracle.makespans(g, topo, _profile_of(doc), doc["mode"], strategies)
        assert [float(x) for x in got] == [fx(h) for h in doc["makespans"]], (doc["name"], doc["mode"])
