"""GPU parity: every makespan / timeline / trajectory bit-identical to the C
oracle (itself pinned to the reference by tests/golden)."""

import math
import random

import numpy as np
import pytest

import paper_1807_05358_b200 as ps
from helpers import manual_task_graph, random_graph, random_topology

pytestmark = pytest.mark.gpu


def _random_case(seed):
    rng = random.Random(seed)
    g = random_graph(rng, 4, 14)
    topo = random_topology(rng, rng.choice((2, 4, 8, 16)))
    mode = ps.MODE_FULL if seed % 2 else ps.MODE_FORWARD
    md = rng.choice((2, 3, 4))
    return g, topo, mode, md


def test_batch_makespans_match_oracle_on_random_graphs(oracle):
    for seed in range(60):
        g, topo, mode, md = _random_case(seed)
        prof = ps.CostProfile()
        strategies = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, md, seed * 100 + i)
                                                            for i in range(8)]
        got = ps.evaluate_strategies(g, topo, prof, strategies, mode=mode, max_degree=md)
        want = oracle.makespans(g, topo, prof, mode, strategies)
        assert list(got) == list(want), seed


def test_timelines_match_oracle(oracle):
    for seed in range(25):
        g, topo, mode, md = _random_case(1000 + seed)
        prof = ps.CostProfile()
        s = ps.random_strategy(g, topo, md, seed)
        tg = ps.build_task_graph(g, topo, s, prof, mode)
        res = ps.full_simulate(tg)
        ref = oracle.simulate(g, topo, prof, mode, s)
        assert res.makespan == ref["makespan"]
        assert len(tg.tasks) == ref["tasks"]
        assert tg.total_comm_bytes == ref["comm_bytes"]
        assert sum(len(t.outputs) for t in tg.tasks.values()) == ref["edges"]
        tt = ps.timeline_table(tg)
        for origin, (start, end, dev) in tt.items():
            r = ref["timeline"][origin]
            assert (start, end) == (r[1], r[2]), origin


def test_rnn3_golden_fixture():
    g = ps.rnn3()
    topo = ps.single_node_topology(gpus=3)
    tg = ps.build_task_graph(g, topo, ps.rnn3_model_parallel_strategy(g, topo), ps.CostProfile(),
                             ps.MODE_FORWARD)
    comm = sum(1 for t in tg.tasks.values() if t.kind == "comm")
    assert (len(tg.tasks), len(tg.tasks) - comm, comm) == (12, 8, 4)
    assert sum(len(t.outputs) for t in tg.tasks.values()) == 11
    assert tg.total_comm_bytes == 16384.0
    assert ps.full_simulate(tg).makespan == 3.5826560000000005e-06
    assert ps.oracle_simulate(tg) == 3.5826560000000005e-06


def test_scheduler_known_answers():
    tg, ids = manual_task_graph([("a", "d0", 1.0), ("b", "d0", 2.0), ("c", "d0", 3.0)], [("a", "b"), ("b", "c")])
    res = ps.full_simulate(tg)
    assert res.makespan == 6.0
    assert [tg.timeline[ids[n]].start for n in "abc"] == [0.0, 1.0, 3.0]
    tg, _ = manual_task_graph([("a", "d0", 5.0), ("b", "d1", 5.0)], [])
    assert ps.full_simulate(tg).makespan == 5.0
    tg, ids = manual_task_graph([("src", "d0", 1.0), ("fast", "d0", 1.0), ("slow", "d1", 3.0), ("join", "d0", 1.0)],
                                [("src", "fast"), ("src", "slow"), ("fast", "join"), ("slow", "join")])
    res = ps.full_simulate(tg)
    assert tg.timeline[ids["join"]].ready == 4.0 and res.makespan == 5.0
    tg, ids = manual_task_graph([("z", "d0", 1.0), ("m", "d0", 1.0), ("a", "d0", 1.0)], [])
    ps.full_simulate(tg)
    assert sorted("zma", key=lambda n: tg.timeline[ids[n]].start) == sorted("zma")
    tg, ids = manual_task_graph([("a", "d0", 3.0), ("hog", "d1", 4.0), ("b", "d1", 1.0)], [("a", "b")])
    ps.full_simulate(tg)
    e = tg.timeline[ids["b"]]
    assert (e.ready, e.start, e.end) == (3.0, 4.0, 5.0)


def test_delta_tracks_chained_changes_exactly(oracle):
    for seed in range(8):
        g, topo, mode, md = _random_case(2000 + seed)
        prof = ps.CostProfile()
        rng = random.Random(seed)
        tg = ps.build_task_graph(g, topo, ps.random_strategy(g, topo, md, seed), prof, mode)
        ps.full_simulate(tg)
        for step in range(12):
            op_id = rng.choice(sorted(g.ops))
            cfg = rng.choice(ps.enumerate_configs(g.ops[op_id], topo, md))
            asg = tuple(rng.choice(topo.device_ids()) for _ in range(cfg.size()))
            _, changed = ps.update_task_graph(tg, g, topo, op_id, ps.ParallelizationConfig(dict(cfg.degrees), asg))
            res = ps.delta_simulate(tg, changed)
            fresh = ps.build_task_graph(g, topo, tg.strategy, prof, mode)
            assert res.makespan == ps.full_simulate(fresh).makespan
            assert ps.timeline_table(tg) == ps.timeline_table(fresh)
            assert res.makespan == oracle.simulate(g, topo, prof, mode, tg.strategy)["makespan"]


@pytest.mark.parametrize("rng_mode", ["mt19937", "philox"])
def test_mcmc_trajectories_match_oracle(oracle, rng_mode):
    for seed in range(10):
        g, topo, mode, md = _random_case(3000 + seed)
        prof = ps.CostProfile()
        init = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, md, seed + i) for i in range(3)]
        params = ps.SearchParams(max_proposals=120, seed=seed, max_degree=md, mode=mode, initial=init,
                                 polish=False, rng=rng_mode)
        rep = ps.mcmc_search(g, topo, prof, params)
        ref = oracle.mcmc(g, topo, prof, mode, init, [seed + 1000003 * c for c in range(4)], 120, md,
                          rng_mode="mt" if rng_mode == "mt19937" else "philox")
        for ci, ch in enumerate(rep.chains):
            s = ref["summary"][ci]
            assert (ch.initial_cost, ch.best_cost, ch.proposals, ch.accepted, ch.beta) == tuple(s[:5]), (seed, ci)
            tr = [c for _, c, _ in rep.trace[ci * 120:(ci + 1) * 120]]
            ok = [a for _, _, a in rep.trace[ci * 120:(ci + 1) * 120]]
            assert tr == list(ref["cand"][ci]) and ok == [bool(x) for x in ref["ok"][ci]], (seed, ci)


def test_benchmark_shapes_match_oracle(oracle):
    cases = [(ps.alexnet_like(), ps.single_node_topology(4), 4),
             (ps.inception_v3(), ps.multi_node_topology(4, 4), 4),
             (ps.nmt_like(steps=4, layers=2, batch=64, hidden=64, vocab=64), ps.multi_node_topology(4, 4), 4)]
    for g, topo, md in cases:
        prof = ps.CostProfile()
        strategies = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, md, s) for s in range(4)]
        for mode in (ps.MODE_FORWARD, ps.MODE_FULL):
            got = ps.evaluate_strategies(g, topo, prof, strategies, mode=mode, max_degree=md)
            want = oracle.makespans(g, topo, prof, mode, strategies)
            assert list(got) == list(want)


def test_missing_link_is_reported_like_the_reference():
    g = ps.OperatorGraph()
    g.add_op(ps.Operation("a", ps.OperatorKind("MatMul"), (ps.shape(("sample", 4), ("channel", 8)),),
                          ps.shape(("sample", 4), ("channel", 8)), param_bytes=256))
    g.add_op(ps.Operation("b", ps.OperatorKind("MatMul"), (ps.shape(("sample", 4), ("channel", 8)),),
                          ps.shape(("sample", 4), ("channel", 4)), param_bytes=128))
    g.add_tensor("a", "b")
    topo = ps.DeviceTopology()
    for d in ("d0", "d1", "d2"):
        topo.add_device(d)
    topo.add_connection("d0", "d1", 1e9, 0.0)
    strat = ps.ParallelizationStrategy({
        "a": ps.ParallelizationConfig({"sample": 1, "channel": 1}, ("d0",)),
        "b": ps.ParallelizationConfig({"sample": 1, "channel": 1}, ("d2",))})
    with pytest.raises(ps.NoRouteError, match="no route between device d0 and device d2"):
        ps.build_task_graph(g, topo, strat, ps.CostProfile(), ps.MODE_FORWARD)


def test_ready_set_capacity_regrows_transparently(oracle):
    """A deliberately tiny ready-set capacity must still give the exact answer
    (the problem is regrown 4x until every candidate fits)."""
    from paper_1807_05358_b200.lowering import lower
    from paper_1807_05358_b200.search import _eval_encoded
    g = ps.nmt_like(steps=4, layers=2, batch=64, hidden=64, vocab=64)
    topo = ps.multi_node_topology(4, 4)
    prof = ps.CostProfile()
    strategies = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, 4, s) for s in range(3)]
    for mode in (ps.MODE_FORWARD, ps.MODE_FULL):
        low = lower(g, topo, prof, mode, max_degree=4, strategies=strategies, ready_capacity=2)
        maps = np.zeros((len(strategies), low.n_ops), dtype=np.int32)
        asg = np.zeros((len(strategies), low.n_slots), dtype=np.uint8)
        for i, s in enumerate(strategies):
            low.encode(s, maps[i], asg[i])
        got = _eval_encoded(low, maps, asg, strategies)
        assert list(got) == list(oracle.makespans(g, topo, prof, mode, strategies))


def test_large_ready_sets_take_the_multi_chunk_path(oracle):
    """NMT data-parallel graphs put > 32 tasks in the ready set at once."""
    g = ps.nmt_like(steps=8, layers=2, batch=64, hidden=64, vocab=64)
    topo = ps.multi_node_topology(4, 4)
    prof = ps.CostProfile()
    strategies = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, 8, s) for s in range(3)]
    for mode in (ps.MODE_FORWARD, ps.MODE_FULL):
        got = ps.evaluate_strategies(g, topo, prof, strategies, mode=mode, max_degree=8)
        assert list(got) == list(oracle.makespans(g, topo, prof, mode, strategies))


def test_mcmc_chains_survive_ready_set_overflow(oracle):
    """Chains whose ready set outgrows shared memory re-run that simulation with
    the ready set in global memory: same trajectory, no failed chains."""
    from paper_1807_05358_b200.lowering import lower
    g = ps.nmt_like(steps=4, layers=2, batch=64, hidden=64, vocab=64)
    topo = ps.multi_node_topology(4, 4)
    prof = ps.CostProfile()
    init = [ps.data_parallel_strategy(g, topo), ps.random_strategy(g, topo, 4, 1)]
    import paper_1807_05358_b200.search as S
    orig = S.lower
    S.lower = lambda *a, **k: orig(*a, **{**k, "ready_capacity": 4})
    try:
        rep = ps.mcmc_search(g, topo, prof, ps.SearchParams(max_proposals=60, seed=2, max_degree=4, initial=init,
                                                            polish=False, mode=ps.MODE_FULL, rng="philox"))
    finally:
        S.lower = orig
    ref = oracle.mcmc(g, topo, prof, ps.MODE_FULL, init, [2 + 1000003 * c for c in range(2)], 60, 4,
                      rng_mode="philox")
    for ci, ch in enumerate(rep.chains):
        assert (ch.initial_cost, ch.best_cost, ch.proposals, ch.accepted) == tuple(ref["summary"][ci][:4])


def test_search_api_semantics_on_gpu():
    """Reference test_search.py behaviours through the GPU path."""
    import math
    g = ps.OperatorGraph()
    g.add_op(ps.Operation("a", ps.OperatorKind("MatMul"), (ps.shape(("sample", 4), ("channel", 4)),),
                          ps.shape(("sample", 4), ("channel", 4)), param_bytes=64))
    g.add_op(ps.Operation("b", ps.OperatorKind("MatMul"), (ps.shape(("sample", 4), ("channel", 4)),),
                          ps.shape(("sample", 4), ("channel", 2)), param_bytes=32))
    g.add_tensor("a", "b")
    topo = ps.single_node_topology(gpus=2)
    prof = ps.CostProfile()
    p = ps.SearchParams(max_proposals=120, seed=5, max_degree=2)
    a, b = ps.mcmc_search(g, topo, prof, p), ps.mcmc_search(g, topo, prof, p)
    assert a == b and a.proposals == 240 and all(c.termination == "proposal-limit" for c in a.chains)
    with pytest.raises(ValueError, match="budget_seconds or max_proposals"):
        ps.mcmc_search(g, topo, prof, ps.SearchParams())
    r = ps.mcmc_search(g, topo, prof, ps.SearchParams(max_proposals=150, seed=1, max_degree=2, beta=math.inf,
                                                      initial=[ps.data_parallel_strategy(g, topo)], polish=False))
    acc = [c for _, c, ok in r.trace if ok]
    assert acc and all(y <= x for x, y in zip(acc, acc[1:]))
    r = ps.mcmc_search(g, topo, prof, ps.SearchParams(max_proposals=1, seed=0, max_degree=2))
    for c in r.chains:
        assert c.beta == pytest.approx(math.log(10.0) / (0.05 * c.initial_cost))
    ps.mcmc_search(g, topo, prof, ps.SearchParams(max_proposals=60, seed=3, max_degree=2, check_interval=1))
    raw = ps.mcmc_search(g, topo, prof, ps.SearchParams(max_proposals=40, seed=9, max_degree=2, polish=False))
    pol = ps.mcmc_search(g, topo, prof, ps.SearchParams(max_proposals=40, seed=9, max_degree=2))
    assert pol.best_cost <= raw.best_cost
    assert ps.local_optimality_check(pol.best_strategy, g, topo, prof, max_degree=2) is None
    bad = ps.ParallelizationStrategy({oid: ps.ParallelizationConfig({"sample": 1, "channel": 1}, ("ghost-device",))
                                      for oid in g.ops})
    rep = ps.mcmc_search(g, topo, prof, ps.SearchParams(max_proposals=30, seed=0, max_degree=2,
                                                        initial=[bad, ps.data_parallel_strategy(g, topo)]))
    assert rep.chains[0].termination.startswith("error") and rep.chains[0].proposals == 0
    assert math.isfinite(rep.best_cost)
    with pytest.raises(ps.SearchError, match="every chain failed"):
        ps.mcmc_search(g, topo, prof, ps.SearchParams(max_proposals=5, initial=[bad]))


def test_polish_and_local_check_match_reference_semantics(oracle):
    """Greedy polish on the GPU reaches the same strategy/cost as the reference's
    sequential first-improvement scan (golden: run here against the oracle by
    re-scoring every accepted move)."""
    g = ps.lenet_like(batch=2, image=4, in_channels=1, conv_channels=(2, 2), fc_hidden=2, classes=2)
    topo = ps.single_node_topology(gpus=2)
    prof = ps.CostProfile()
    rep = ps.mcmc_search(g, topo, prof, ps.SearchParams(max_proposals=50, seed=4, max_degree=2))
    assert rep.best_cost == oracle.simulate(g, topo, prof, ps.MODE_FORWARD, rep.best_strategy)["makespan"]
    assert ps.local_optimality_check(rep.best_strategy, g, topo, prof, max_degree=2) is None


def test_default_search_report_is_byte_identical_to_the_reference():
    """mcmc_search with default parameters (CPython MT19937 stream, greedy
    polish) reproduces the reference's report JSON byte for byte."""
    from golden_io import load
    for doc in load("search_reports.json"):
        g = ps.graph_from_json(doc["graph"])
        topo = ps.topology_from_json(doc["topology"])
        rep = ps.mcmc_search(g, topo, ps.CostProfile(), ps.SearchParams(
            max_proposals=doc["max_proposals"], seed=doc["seed"], max_degree=doc["max_degree"], mode=doc["mode"]))
        assert ps.report_to_json(rep) == doc["report"], doc["name"]


def test_exhaustive_optimal_matches_the_reference():
    """Same optimum, same strategy, same number of visited search nodes."""
    from golden_io import fx, load
    for doc in load("exhaustive.json"):
        g = ps.graph_from_json(doc["graph"])
        topo = ps.topology_from_json(doc["topology"])
        res = ps.exhaustive_optimal(g, topo, ps.CostProfile(), max_degree=doc["max_degree"], cap=1e15,
                                    mode=doc["mode"])
        assert res.cost == fx(doc["cost"]), doc["name"]
        assert res.visited == doc["visited"], doc["name"]
        assert res.space_estimate == doc["space_estimate"]
        assert ps.strategy_to_json(res.strategy) == doc["strategy"], doc["name"]


@pytest.mark.parametrize("hook", ["PS_FORCE_ASG_GLOBAL", "PS_FORCE_GLOBAL_ALL"])
def test_global_memory_layouts(oracle, monkeypatch, hook):
    """Very wide problems keep device assignments in global memory, and problems
    too big for shared memory keep every table there; force each layout on a
    small problem and check batch evaluation, timelines and MCMC parity."""
    monkeypatch.setenv(hook, "1")
    g, topo, mode, md = _random_case(4242)
    prof = ps.CostProfile()
    strategies = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, md, s) for s in range(6)]
    got = ps.evaluate_strategies(g, topo, prof, strategies, mode=mode, max_degree=md)
    assert list(got) == list(oracle.makespans(g, topo, prof, mode, strategies))
    tg = ps.build_task_graph(g, topo, strategies[1], prof, mode=mode)
    assert ps.full_simulate(tg).makespan == got[1]
    init = strategies[:3]
    rep = ps.mcmc_search(g, topo, prof, ps.SearchParams(max_proposals=80, seed=7, max_degree=md, mode=mode,
                                                        initial=init, polish=False, rng="philox"))
    ref = oracle.mcmc(g, topo, prof, mode, init, [7 + 1000003 * c for c in range(3)], 80, md, rng_mode="philox")
    for ci, ch in enumerate(rep.chains):
        assert (ch.initial_cost, ch.best_cost, ch.proposals, ch.accepted) == tuple(ref["summary"][ci][:4])


# ---------------------------------------------------------------- full sizes
# BASELINE.json configs at their own sizes (not reduced): the GPU path against
# the oracle, strategy by strategy, and the 1024-chain MCMC the bench times.

def _full_size_cases():
    return [
        ("resnet101_16x4", ps.resnet101(), ps.multi_node_topology(16, 4), 8),
        ("nmt40_16x4", ps.nmt_like(steps=40, layers=2, batch=64, hidden=1024, vocab=32768),
         ps.multi_node_topology(16, 4), 8),
        ("random1k_4x4", ps.random_dag(1000, seed=1000), ps.multi_node_topology(4, 4), 4),
    ]


@pytest.mark.parametrize("case", range(3))
def test_full_size_configs_match_oracle(oracle, case):
    name, g, topo, md = _full_size_cases()[case]
    prof = ps.CostProfile()
    strategies = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, md, s) for s in range(3)]
    for mode in (ps.MODE_FULL, ps.MODE_FORWARD):
        got = ps.evaluate_strategies(g, topo, prof, strategies, mode=mode, max_degree=md)
        want = oracle.makespans(g, topo, prof, mode, strategies)
        assert list(got) == list(want), (name, mode)


def test_bench_config_mcmc_matches_oracle(oracle):
    """Inception-v3 on 4x4 devices, full-iteration, 1024 chains (the bench
    workload, Philox streams): every chain's summary and best strategy."""
    import os
    g, topo, md = ps.inception_v3(), ps.multi_node_topology(4, 4), 4
    prof = ps.CostProfile()
    C, P = 1024, 128
    init = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, md, c) for c in range(1, C)]
    seeds = [1000003 * c for c in range(C)]
    params = ps.SearchParams(max_proposals=P, seed=0, max_degree=md, mode=ps.MODE_FULL, initial=init,
                             polish=False, rng="philox")
    rep = ps.mcmc_search(g, topo, prof, params)
    ref = oracle.mcmc(g, topo, prof, ps.MODE_FULL, init, seeds, P, md, rng_mode="philox",
                      threads=os.cpu_count() or 1)
    got = [(ch.initial_cost, ch.best_cost, ch.proposals, ch.accepted, ch.beta) for ch in rep.chains]
    want = [tuple(s[:5]) for s in ref["summary"]]
    assert got == want
    cand = np.array([c for _, c, _ in rep.trace]).reshape(C, P)
    assert np.array_equal(cand, ref["cand"])


def _hetero_topology(rng):
    """Two device kinds and three distinct link speeds: the multi-kind time table
    and the per-transfer division path (more than two link classes)."""
    topo = ps.DeviceTopology()
    devs = []
    for n in range(2):
        for i in range(4):
            kind = "gpu" if i < 2 else "tpu"
            d = f"n{n}{kind}{i}"
            topo.add_device(d, kind, f"node{n}")
            devs.append((n, kind, d))
    for x in range(len(devs)):
        for y in range(x + 1, len(devs)):
            (na, ka, a), (nb, kb, b) = devs[x], devs[y]
            if na != nb:
                bw, lat = 7e9, 5e-6
            elif ka == kb == "tpu":
                bw, lat = 32e9, 5e-7
            else:
                bw, lat = rng.choice(((16e9, 1e-6), (12e9, 2e-6)))
            topo.add_connection(a, b, bw, lat)
    return topo


@pytest.mark.parametrize("shape", ["hetero8", "mesh64"])
def test_randomised_sweep_matches_oracle(oracle, shape):
    rng = random.Random(2026 if shape == "hetero8" else 2027)
    for case in range(24):
        g = ps.random_dag(rng.randint(10, 50), seed=rng.randrange(1 << 30))
        if shape == "hetero8":
            topo = _hetero_topology(rng)
            prof = ps.CostProfile(fallback=ps.AnalyticCostModel(throughput={"tpu": 3e12}))
        else:
            topo = ps.multi_node_topology(16, 4)
            prof = ps.CostProfile()
        md = rng.choice((2, 4, 8))
        strategies = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, md, rng.randrange(1 << 20))
                                                            for _ in range(3)]
        for mode in (ps.MODE_FULL, ps.MODE_FORWARD):
            got = ps.evaluate_strategies(g, topo, prof, strategies, mode=mode, max_degree=md)
            want = oracle.makespans(g, topo, prof, mode, strategies)
            assert list(got) == list(want), (shape, case, mode)


def test_mcmc_on_heterogeneous_topology_matches_oracle(oracle):
    rng = random.Random(99)
    g = ps.random_dag(30, seed=1234)
    topo = _hetero_topology(rng)
    prof = ps.CostProfile(fallback=ps.AnalyticCostModel(throughput={"tpu": 3e12}))
    init = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, 4, s) for s in range(3)]
    for mode in (ps.MODE_FULL, ps.MODE_FORWARD):
        rep = ps.mcmc_search(g, topo, prof, ps.SearchParams(max_proposals=100, seed=11, max_degree=4, mode=mode,
                                                            initial=init, polish=False, rng="philox"))
        ref = oracle.mcmc(g, topo, prof, mode, init, [11 + 1000003 * c for c in range(4)], 100, 4, rng_mode="philox")
        for ci, ch in enumerate(rep.chains):
            assert (ch.initial_cost, ch.best_cost, ch.proposals, ch.accepted) == tuple(ref["summary"][ci][:4]), (mode, ci)


def test_time_boxed_segments_are_exact_prefixes(oracle):
    """ps_mcmc_run_budget stops chains at data-dependent points (its time budget
    and each chain's mean proposal time): whatever it stopped at, every chain's
    state must equal the oracle's after that many proposals."""
    import ctypes
    from paper_1807_05358_b200 import _native as nat
    from paper_1807_05358_b200.lowering import lower
    g, topo, mode, md = _random_case(77)
    prof = ps.CostProfile()
    C = 48
    init = [ps.data_parallel_strategy(g, topo)] + [ps.random_strategy(g, topo, md, c) for c in range(1, C)]
    seeds = np.array([5 + 1000003 * c for c in range(C)], dtype=np.uint64)
    low = lower(g, topo, prof, ps.MODE_FULL, max_degree=md, strategies=init)
    maps = np.zeros((C, low.n_ops), dtype=np.int32)
    asg = np.zeros((C, low.n_slots), dtype=np.uint8)
    for i, s in enumerate(init):
        low.encode(s, maps[i], asg[i])
    L = nat.lib()
    mp = nat.PsMcmcParams(nat.PS_RNG_PHILOX, 0, 0.0, math.log(10.0), 0, 0)
    h = ctypes.c_void_p()
    nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), C, nat.ptr(maps), nat.ptr(asg), nat.ptr(seeds), None,
                               ctypes.byref(h)), "ps_mcmc_create")
    try:
        for _ in range(3):
            nat.check(L.ps_mcmc_run_budget(h, 1 << 30, 300_000, None), "ps_mcmc_run_budget")  # 0.3 ms segments
        summ = (nat.PsChainSummary * C)()
        nat.check(L.ps_mcmc_read(h, summ, None, None, None, None), "ps_mcmc_read")
    finally:
        L.ps_mcmc_destroy(h)
    counts = sorted({s.proposals for s in summ})
    assert counts[-1] > 0
    for p in counts:
        idx = [c for c in range(C) if summ[c].proposals == p]
        ref = oracle.mcmc(g, topo, prof, ps.MODE_FULL, [init[c] for c in idx], [int(seeds[c]) for c in idx], p, md,
                          rng_mode="philox")
        for j, c in enumerate(idx):
            s = summ[c]
            assert (s.initial_cost, s.best_cost, s.proposals, s.accepted) == tuple(ref["summary"][j][:4]), (c, p)


def _run_mcmc_raw(low, init, seeds, proposals, delta, record=0):
    import ctypes
    from paper_1807_05358_b200 import _native as nat
    C = len(init)
    maps = np.zeros((C, low.n_ops), dtype=np.int32)
    asg = np.zeros((C, low.n_slots), dtype=np.uint8)
    for i, s in enumerate(init):
        low.encode(s, maps[i], asg[i])
    L = nat.lib()
    mp = nat.PsMcmcParams(nat.PS_RNG_PHILOX, 0, 0.0, math.log(10.0), 1 if record else 0, record, delta)
    h = ctypes.c_void_p()
    sd = np.array(seeds, dtype=np.uint64)
    nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), C, nat.ptr(maps), nat.ptr(asg), nat.ptr(sd), None,
                               ctypes.byref(h)), "ps_mcmc_create")
    try:
        for done in range(0, proposals, 50):
            nat.check(L.ps_mcmc_run(h, min(50, proposals - done), None), "ps_mcmc_run")
        summ = (nat.PsChainSummary * C)()
        bm = np.zeros((C, low.n_ops), dtype=np.int32)
        ba = np.zeros((C, low.n_slots), dtype=np.uint8)
        tc = np.zeros((C, max(record, 1)))
        nat.check(L.ps_mcmc_read(h, summ, nat.ptr(bm), nat.ptr(ba), nat.ptr(tc) if record else None, None),
                  "ps_mcmc_read")
    finally:
        L.ps_mcmc_destroy(h)
    return summ, bm, ba, tc


@pytest.mark.parametrize("mode", [ps.MODE_FULL, ps.MODE_FORWARD])
def test_delta_evaluation_equals_from_scratch_and_oracle(oracle, mode):
    """Checkpointed delta evaluation (resume from the last snapshot before the
    changed op's first dependent round) gives the same trajectories, best
    strategies and trace as re-simulating every proposal from time zero, and
    the oracle's; and it does skip rounds."""
    from paper_1807_05358_b200.lowering import lower
    g, topo, md = ps.inception_v3(), ps.multi_node_topology(4, 4), 4
    prof = ps.CostProfile()
    C, P = 96, 150
    init = [ps.data_parallel_strategy(g, topo)] + ps.random_strategies(g, topo, md, list(range(1, C)))
    seeds = [1000003 * c for c in range(C)]
    low = lower(g, topo, prof, mode, max_degree=md, strategies=init)
    a, am, aa, at = _run_mcmc_raw(low, init, seeds, P, 1, record=P)
    b, bm, ba, bt = _run_mcmc_raw(low, init, seeds, P, 0, record=P)
    key = lambda s: (s.initial_cost, s.best_cost, s.cost, s.proposals, s.accepted, s.beta, s.status)
    assert [key(s) for s in a] == [key(s) for s in b]
    assert np.array_equal(am, bm) and np.array_equal(aa, ba) and np.array_equal(at, bt)
    reused = sum(s.rounds_reused for s in a)
    run = sum(s.rounds_run for s in a)
    assert reused > 0.05 * (reused + run), (reused, run, [(s.rounds_run, s.rounds_reused, s.status, s.proposals) for s in a[:8]])
    assert all(s.rounds_reused == 0 for s in b)
    ref = oracle.mcmc(g, topo, prof, mode, init[:16], seeds[:16], P, md, rng_mode="philox", threads=8)
    assert [key(s)[:2] + key(s)[3:5] for s in a[:16]] == [(r[0], r[1], r[2], r[3]) for r in ref["summary"]]
    assert np.array_equal(at[:16], ref["cand"])


def test_delta_evaluation_on_large_and_heterogeneous_problems(oracle):
    """Delta evaluation where the counters live in global memory (ResNet-101 on
    64 devices), with capacity reruns, and on a heterogeneous topology."""
    from paper_1807_05358_b200.lowering import lower
    rng = random.Random(5)
    cases = [(ps.resnet101(), ps.multi_node_topology(16, 4), 8, ps.CostProfile(), 24, 40),
             (ps.random_dag(40, seed=77), _hetero_topology(rng),
              4, ps.CostProfile(fallback=ps.AnalyticCostModel(throughput={"tpu": 3e12})), 32, 120)]
    for g, topo, md, prof, C, P in cases:
        for mode in (ps.MODE_FULL, ps.MODE_FORWARD):
            init = [ps.data_parallel_strategy(g, topo)] + ps.random_strategies(g, topo, md, list(range(1, C)))
            seeds = [7 + 1000003 * c for c in range(C)]
            low = lower(g, topo, prof, mode, max_degree=md, strategies=init, ready_capacity=16)
            a, am, aa, at = _run_mcmc_raw(low, init, seeds, P, 1, record=P)
            ref = oracle.mcmc(g, topo, prof, mode, init, seeds, P, md, rng_mode="philox", threads=8)
            assert [(s.initial_cost, s.best_cost, s.proposals, s.accepted) for s in a] == \
                [tuple(r[:4]) for r in ref["summary"]], mode
            assert np.array_equal(at, ref["cand"])


@pytest.mark.parametrize("mode", [ps.MODE_FULL, ps.MODE_FORWARD])
def test_delta_batch_abi_matches_full_evaluation(oracle, mode):
    """ps_delta_batch (the C-ABI form of update_task_graph + delta_simulate):
    per chain, 40 rounds of a given single-op change, committed or rolled back
    at random; every makespan equals a from-scratch batch evaluation of the
    changed strategy, the chains' live strategies follow the commits, and a
    sample matches the oracle."""
    import ctypes
    from paper_1807_05358_b200 import _native as nat
    from paper_1807_05358_b200.lowering import lower
    g, topo, md = ps.inception_v3(), ps.multi_node_topology(4, 4), 4
    prof = ps.CostProfile()
    C = 64
    init = [ps.data_parallel_strategy(g, topo)] + ps.random_strategies(g, topo, md, list(range(1, C)))
    low = lower(g, topo, prof, mode, max_degree=md, strategies=init)
    maps = np.zeros((C, low.n_ops), dtype=np.int32)
    asg = np.zeros((C, low.n_slots), dtype=np.uint8)
    for i, s in enumerate(init):
        low.encode(s, maps[i], asg[i])
    L = nat.lib()
    mp = nat.PsMcmcParams(nat.PS_RNG_PHILOX, 0, 0.0, math.log(10.0), 0, 0, 1)
    h = ctypes.c_void_p()
    sd = np.zeros(C, dtype=np.uint64)
    nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), C, nat.ptr(maps), nat.ptr(asg), nat.ptr(sd), None,
                               ctypes.byref(h)), "ps_mcmc_create")
    rng = np.random.default_rng(3)
    nmaps = low.arrays["op_nmaps_enum"]
    stride = int(max(low.arrays["map_size"]))
    checked = []
    try:
        for step in range(40):
            op = rng.integers(0, low.n_ops, C).astype(np.int32)
            op[rng.random(C) < 0.1] = -1  # some chains sit this round out
            mi = np.array([rng.integers(0, nmaps[o]) if o >= 0 else 0 for o in op], dtype=np.int32)
            dv = rng.integers(0, topo.device_ids().__len__(), (C, stride)).astype(np.uint8)
            commit = (rng.random(C) < 0.5).astype(np.uint8)
            mk = np.zeros(C)
            st = np.zeros(C, dtype=np.int32)
            nat.check(L.ps_delta_batch(h, nat.ptr(op), nat.ptr(mi), nat.ptr(dv), stride, nat.ptr(commit), nat.ptr(mk),
                                       nat.ptr(st), nat.PS_HOST_PTRS, None), "ps_delta_batch")
            assert (st == nat.PS_STATUS_OK).all()
            # the changed strategies, scored from scratch
            cm, ca = maps.copy(), asg.copy()
            for i in range(C):
                if op[i] < 0:
                    continue
                r = int(op[i])
                cm[i, r] = mi[i]
                size = int(low.arrays["map_size"][low.arrays["op_map_off"][r] + mi[i]])
                base = int(low.slot_off[r])
                ca[i, base:base + size] = dv[i, :size]
            live = op >= 0
            fresh = np.zeros(C)
            fst = np.zeros(C, dtype=np.int32)
            nat.check(L.ps_simulate_batch(low.handle(), nat.ptr(cm), nat.ptr(ca), C, nat.ptr(fresh), nat.ptr(fst),
                                          nat.PS_HOST_PTRS, None), "ps_simulate_batch")
            assert np.array_equal(mk[live], fresh[live]), step
            keep = live & (commit != 0)
            maps[keep], asg[keep] = cm[keep], ca[keep]
            if step % 10 == 9:
                checked.append((low.decode(cm[1], ca[1]), float(mk[1])))
        sm = np.zeros_like(maps)
        sa = np.zeros_like(asg)
        nat.check(L.ps_mcmc_read_state(h, nat.ptr(sm), nat.ptr(sa)), "ps_mcmc_read_state")
        assert np.array_equal(sm, maps)
        for i in range(C):  # live strategies: compare the used slots of each op
            for r in range(low.n_ops):
                size = int(low.arrays["map_size"][low.arrays["op_map_off"][r] + maps[i, r]])
                base = int(low.slot_off[r])
                assert np.array_equal(sa[i, base:base + size], asg[i, base:base + size])
        summ = (nat.PsChainSummary * C)()
        nat.check(L.ps_mcmc_read(h, summ, None, None, None, None), "ps_mcmc_read")
        assert sum(s.rounds_reused for s in summ) > 0
    finally:
        L.ps_mcmc_destroy(h)
    want = oracle.makespans(g, topo, prof, mode, [s for s, _ in checked])
    assert [m for _, m in checked] == list(want)


def test_api_delta_resumes_on_the_resident_handle(oracle):
    """update_task_graph + delta_simulate through the drop-in API: the task
    graph keeps a resident delta handle, ``changed`` is computed lazily and
    equals the eager definition, and results match fresh builds."""
    from paper_1807_05358_b200.taskgraph import ChangedTasks
    g, topo, md = ps.inception_v3(), ps.multi_node_topology(4, 4), 4
    prof = ps.CostProfile()
    rng = random.Random(11)
    tg = ps.build_task_graph(g, topo, ps.random_strategy(g, topo, md, 1), prof, ps.MODE_FULL)
    ps.full_simulate(tg)
    for step in range(30):
        op_id = rng.choice(sorted(g.ops))
        cfg = rng.choice(ps.enumerate_configs(g.ops[op_id], topo, md))
        asg = tuple(rng.choice(topo.device_ids()) for _ in range(cfg.size()))
        before = tg.strategy.copy()
        _, changed = ps.update_task_graph(tg, g, topo, op_id, ps.ParallelizationConfig(dict(cfg.degrees), asg))
        res = ps.delta_simulate(tg, changed)
        assert tg._dh is not None and tg._dh_pending == []
        fresh = ps.build_task_graph(g, topo, tg.strategy, prof, ps.MODE_FULL)
        assert res.makespan == ps.full_simulate(fresh).makespan
        if step % 10 == 0 and isinstance(changed, ChangedTasks):
            old = ps.build_task_graph(g, topo, before, prof, ps.MODE_FULL)
            prev = {t.origin: (t.exe_time, t.device, frozenset(old.tasks[p].origin for p in t.inputs))
                    for t in old.tasks.values()}
            want = sorted(tid for tid, t in fresh.tasks.items()
                          if t.op_id == op_id or (t.origin[0] in ("edge", "edge_bwd", "sync") and op_id in t.origin[1:3])
                          or prev.get(t.origin) != (t.exe_time, t.device,
                                                    frozenset(fresh.tasks[p].origin for p in t.inputs)))
            assert list(changed) == want
            assert ps.timeline_table(tg) == ps.timeline_table(fresh)
    assert tg._dh is not None
    assert oracle.simulate(g, topo, prof, ps.MODE_FULL, tg.strategy)["makespan"] == res.makespan


@pytest.mark.parametrize("budget", [None, 0.5])
def test_sharded_search_equals_single_gpu_search(budget):
    """mcmc_search(devices=[...]): chains split into contiguous shards, one host
    thread and problem copy per GPU (here two shards on GPU 0), merged with the
    reference's earliest-chain rule (search.py:256).  With a proposal limit the
    report is byte-identical to the one-GPU run of the same chains; time-boxed,
    every chain's trajectory is an exact prefix of the same stream."""
    g, topo, md = ps.inception_v3(), ps.multi_node_topology(4, 4), 4
    prof = ps.CostProfile()
    C = 48
    init = [ps.data_parallel_strategy(g, topo)] + ps.random_strategies(g, topo, md, list(range(1, C)))
    kw = dict(seed=3, max_degree=md, mode=ps.MODE_FULL, initial=init, polish=False, rng="philox")
    if budget is None:
        kw["max_proposals"] = 60
    else:
        kw["budget_seconds"] = budget
    one = ps.mcmc_search(g, topo, prof, ps.SearchParams(**kw))
    two = ps.mcmc_search(g, topo, prof, ps.SearchParams(devices=[0, 0], **kw))
    if budget is None:
        assert ps.formats.report_to_json(one) == ps.formats.report_to_json(two)
        # a three-way split with an uneven last shard
        three = ps.mcmc_search(g, topo, prof, ps.SearchParams(devices=[0, 0, 0], **kw))
        assert ps.formats.report_to_json(one) == ps.formats.report_to_json(three)
    else:
        for a, b in zip(one.chains, two.chains):
            assert a.initial_cost == b.initial_cost and a.beta == b.beta
        # chain-by-chain: the shorter run's trace is a prefix of the longer one's
        off_a = off_b = 0
        for a, b in zip(one.chains, two.chains):
            ta = [c for _, c, _ in one.trace[off_a:off_a + a.proposals]]
            tb = [c for _, c, _ in two.trace[off_b:off_b + b.proposals]]
            k = min(len(ta), len(tb))
            assert ta[:k] == tb[:k]
            off_a += a.proposals
            off_b += b.proposals


def test_sharded_evaluation_equals_one_launch():
    g, topo, md = ps.inception_v3(), ps.multi_node_topology(4, 4), 4
    prof = ps.CostProfile()
    strategies = ps.random_strategies(g, topo, md, list(range(37)))
    a = ps.evaluate_strategies(g, topo, prof, strategies, mode=ps.MODE_FULL, max_degree=md)
    b = ps.evaluate_strategies(g, topo, prof, strategies, mode=ps.MODE_FULL, max_degree=md, devices=[0, 0, 0])
    assert list(a) == list(b)


@pytest.mark.parametrize("cap,warp_global", [(2, False), (8, True), (128, False), (128, True), (16, "all")])
def test_two_level_ready_set_matches_oracle(oracle, monkeypatch, cap, warp_global):
    """The wide-problem variants (front ready set in shared memory, unsorted
    back set in global memory with a lower bound on its ready times, refill /
    trim / combined slow rounds; optionally warp slices in global memory)
    forced onto small problems with tiny front capacities: batch makespans and
    MCMC trajectories (delta evaluation on) equal the oracle's."""
    from paper_1807_05358_b200.lowering import lower
    from paper_1807_05358_b200.search import _eval_encoded
    monkeypatch.setenv("PS_FORCE_WIDE", "1")
    if warp_global == "all":  # block tables and warp slices in global memory
        monkeypatch.setenv("PS_FORCE_GLOBAL_ALL", "1")
    elif warp_global:  # warp slices in global memory, per-round state in shared memory
        monkeypatch.setenv("PS_FORCE_WARP_GLOBAL", "1")
    rng = random.Random(cap)
    cases = [(ps.nmt_like(steps=8, layers=2, batch=64, hidden=64, vocab=64), ps.multi_node_topology(4, 4), 8),
             (ps.random_dag(300, seed=cap), ps.multi_node_topology(4, 4), 4),
             (ps.inception_v3(), ps.multi_node_topology(4, 4), 4)]
    for g, topo, md in cases:
        prof = ps.CostProfile()
        strategies = [ps.data_parallel_strategy(g, topo)] + ps.random_strategies(g, topo, md, [rng.randrange(10**6) for _ in range(7)])
        for mode in (ps.MODE_FORWARD, ps.MODE_FULL):
            low = lower(g, topo, prof, mode, max_degree=md, strategies=strategies, ready_capacity=cap)
            maps = np.zeros((len(strategies), low.n_ops), dtype=np.int32)
            asg = np.zeros((len(strategies), low.n_slots), dtype=np.uint8)
            for i, s in enumerate(strategies):
                low.encode(s, maps[i], asg[i])
            got = _eval_encoded(low, maps, asg, strategies)
            assert list(got) == list(oracle.makespans(g, topo, prof, mode, strategies)), (g, mode)
            C = 16
            init = (strategies * 2)[:C]
            seeds = [5 + 1000003 * c for c in range(C)]
            a, _, _, at = _run_mcmc_raw(low, init, seeds, 30, 1, record=30)
            ref = oracle.mcmc(g, topo, prof, mode, init, seeds, 30, md, rng_mode="philox", threads=8)
            assert [(s.initial_cost, s.best_cost, s.proposals, s.accepted) for s in a] == \
                [tuple(r[:4]) for r in ref["summary"]], (mode, cap)
            assert np.array_equal(at, ref["cand"])


@pytest.mark.parametrize("budget,mux", [(False, False), (True, False), (False, True), (True, True)])
def test_more_chains_than_resident_warps(oracle, monkeypatch, budget, mux):
    """More chains than resident warps: later blocks wait for a resident one to
    finish, or (PS_MCMC_MUX) the resident warps run their chains in turn with
    the time box split among them.  Every chain's summary and trace equal the
    oracle's for the proposals it made."""
    if mux:
        monkeypatch.setenv("PS_MCMC_MUX", "1")
    import ctypes
    from paper_1807_05358_b200 import _native as nat
    from paper_1807_05358_b200.lowering import lower
    g, topo, md = ps.alexnet_like(), ps.single_node_topology(4), 4
    prof = ps.CostProfile()
    C = 2600
    init = [ps.data_parallel_strategy(g, topo)] + ps.random_strategies(g, topo, md, list(range(1, C)))
    seeds = [11 + 1000003 * c for c in range(C)]
    low = lower(g, topo, prof, ps.MODE_FULL, max_degree=md, strategies=init)
    assert low.info().resident_warps_per_sm * 148 < C
    maps = np.zeros((C, low.n_ops), dtype=np.int32)
    asg = np.zeros((C, low.n_slots), dtype=np.uint8)
    for i, s in enumerate(init):
        low.encode(s, maps[i], asg[i])
    L = nat.lib()
    P = 40
    mp = nat.PsMcmcParams(nat.PS_RNG_PHILOX, 0, 0.0, math.log(10.0), 1, P, 1)
    h = ctypes.c_void_p()
    sd = np.array(seeds, dtype=np.uint64)
    nat.check(L.ps_mcmc_create(low.handle(), ctypes.byref(mp), C, nat.ptr(maps), nat.ptr(asg), nat.ptr(sd), None,
                               ctypes.byref(h)), "ps_mcmc_create")
    try:
        if budget:
            nat.check(L.ps_mcmc_run_budget(h, P, 2_000_000, None), "ps_mcmc_run_budget")  # 2 ms, split per warp
        else:
            nat.check(L.ps_mcmc_run(h, P, None), "ps_mcmc_run")
        summ = (nat.PsChainSummary * C)()
        tc = np.zeros((C, P))
        nat.check(L.ps_mcmc_read(h, summ, None, None, nat.ptr(tc), None), "ps_mcmc_read")
    finally:
        L.ps_mcmc_destroy(h)
    counts = sorted({s.proposals for s in summ})
    assert counts[-1] > 0 and all(s.status == nat.PS_STATUS_OK for s in summ)
    if not budget:
        assert counts == [P]
    for p in counts:
        idx = [c for c in range(C) if summ[c].proposals == p][:64]  # a sample per proposal count
        ref = oracle.mcmc(g, topo, prof, ps.MODE_FULL, [init[c] for c in idx], [seeds[c] for c in idx], p, md,
                          rng_mode="philox", threads=8)
        for j, c in enumerate(idx):
            s = summ[c]
            assert (s.initial_cost, s.best_cost, s.proposals, s.accepted) == tuple(ref["summary"][j][:4]), (c, p)
            assert list(tc[c, :p]) == list(ref["cand"][j, :p]), (c, p)
