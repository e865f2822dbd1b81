"""Host-side API (CPU only): data model, SOAP partition math, cost model,
profile format, lowering tables, RNG streams, and the C-ABI library surface.
Known answers follow the reference's own unit tests (test_graph.py,
test_partition.py, test_cost.py)."""

import ctypes
import itertools
import math
import os
import random
import re

import numpy as np
import pytest

import paper_1807_05358_b200 as ps
from paper_1807_05358_b200 import _native as nat
from paper_1807_05358_b200.lowering import lower

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# -- graph ---------------------------------------------------------------------

def test_shape_accessors():
    s = ps.shape(("sample", 4), ("channel", 8), element_size=2)
    assert s.names() == ("sample", "channel") and s.sizes() == (4, 8)
    assert s.size("channel") == 8 and s.has("sample") and not s.has("width")
    assert s.volume() == 32 and s.nbytes() == 64
    with pytest.raises(KeyError):
        s.size("height")


def test_conv_arithmetic():
    assert [ps.conv_out_size(8, 3, 1, "same"), ps.conv_out_size(8, 3, 1, "valid"), ps.conv_out_size(8, 3, 2, "same"),
            ps.conv_out_size(8, 2, 2, "valid"), ps.conv_out_size(7, 3, 2, "same")] == [8, 6, 4, 4, 4]
    assert [ps.pad_before(8, 3, 1, "same"), ps.pad_before(8, 3, 1, "valid"), ps.pad_before(8, 2, 2, "same")] == [1, 0, 0]


def _ew(name):
    s = ps.shape(("sample", 2))
    return ps.Operation(name, ps.OperatorKind("ElementWise"), (s,), s)


def test_topological_order_and_cycles():
    g = ps.OperatorGraph()
    for n in "abc":
        g.add_op(_ew(n))
    g.add_tensor("a", "b")
    g.add_tensor("b", "c")
    assert g.topological_order() == ["a", "b", "c"]
    assert g.predecessors("c") == ["b"] and g.successors("a") == ["b"]
    with pytest.raises(ValueError, match="duplicate"):
        g.add_op(_ew("a"))
    g.add_tensor("c", "a")
    with pytest.raises(ValueError):
        g.topological_order()
    assert any("cycle" in i for i in ps.validate_graph(g).issues)


def test_dimension_classes():
    mm = ps.Operation("mm", ps.OperatorKind("MatMul"), (ps.shape(("sample", 4), ("channel", 8)),),
                      ps.shape(("sample", 4), ("channel", 16)), param_bytes=512)
    assert ps.parallelizable_dims(mm) == {"sample": "sample", "channel": "parameter"}
    emb = ps.Operation("em", ps.OperatorKind("Embedding", {"vocab_size": 16}), (ps.shape(("sample", 4)),),
                       ps.shape(("sample", 4), ("channel", 8)), param_bytes=512)
    assert ps.parallelizable_dims(emb) == {"sample": "sample", "channel": "parameter"}


def test_generators_validate_and_match_reference_sizes():
    for name, gen in ps.MODEL_GENERATORS.items():
        assert ps.validate_graph(gen()).ok, name
    inc, res = ps.inception_v3(), ps.resnet101()
    assert len(inc.ops) == 125 and ps.validate_graph(inc).ok
    assert len(res.ops) == 141 and ps.validate_graph(res).ok
    assert round(sum(o.param_bytes for o in inc.ops.values()) / 1e6, 1) == 95.2
    assert round(sum(o.param_bytes for o in res.ops.values()) / 1e6, 1) == 177.8
    g = ps.random_dag(400, seed=3)
    assert len(g.ops) == 400 and ps.validate_graph(g).ok
    tags = {op.kind.tag for seed in range(12) for op in ps.random_dag(60, seed=seed).ops.values()}
    assert tags == set(ps.graph.KIND_TAGS)


def test_topology_validation():
    topo = ps.DeviceTopology()
    topo.add_device("a")
    topo.add_device("b")
    topo.add_connection("a", "b", 1e9, 1e-6)
    assert ps.validate_topology(topo).ok
    topo.connections += [ps.Connection("a", "ghost", 1e9), ps.Connection("a", "a", 1e9), ps.Connection("b", "a", -5.0, -1.0)]
    issues = "\n".join(ps.validate_topology(topo).issues)
    for frag in ("unknown device ghost", "endpoints must differ", "duplicate connection", "bandwidth must be positive",
                 "negative latency"):
        assert frag in issues


# -- partition -----------------------------------------------------------------

def _mm(sample=4, cin=4, cout=4):
    return ps.Operation("mm", ps.OperatorKind("MatMul"), (ps.shape(("sample", sample), ("channel", cin)),),
                        ps.shape(("sample", sample), ("channel", cout)), param_bytes=cin * cout * 4)


def test_enumerate_configs_order():
    cfgs = ps.enumerate_configs(_mm(), ps.single_node_topology(gpus=4), max_degree=4)
    assert [(c.degrees["sample"], c.degrees["channel"]) for c in cfgs] == [(1, 1), (1, 2), (1, 4), (2, 1), (2, 2), (4, 1)]
    assert max(c.size() for c in ps.enumerate_configs(_mm(), ps.single_node_topology(gpus=2), 64)) == 2
    assert ps.divisors(16) == [1, 2, 4, 8, 16]


def test_output_region_row_major_and_tiling():
    cfg = ps.ParallelizationConfig({"sample": 2, "channel": 2})
    op = _mm()
    assert [ps.output_region(op, cfg, k) for k in range(4)] == [
        ps.region(("sample", 0, 2), ("channel", 0, 2)), ps.region(("sample", 0, 2), ("channel", 2, 4)),
        ps.region(("sample", 2, 4), ("channel", 0, 2)), ps.region(("sample", 2, 4), ("channel", 2, 4))]
    with pytest.raises(IndexError):
        ps.output_region(op, cfg, 4)
    with pytest.raises(ValueError):
        ps.output_region(op, ps.ParallelizationConfig({"sample": 3}), 0)


def test_receptive_field_and_param_slice():
    op = ps.Operation("cv", ps.OperatorKind("Conv1D", {"kernel": 3, "stride": 1, "padding": "same"}),
                      (ps.shape(("sample", 2), ("length", 16), ("channel", 2)),),
                      ps.shape(("sample", 2), ("length", 16), ("channel", 4)), param_bytes=96)
    needs = dict(ps.input_regions(op, ps.region(("sample", 0, 2), ("length", 8, 16), ("channel", 0, 4))))
    assert needs[0].range_of("length") == (7, 16) and needs[0].range_of("channel") == (0, 2)
    assert needs["param"] == ps.region(("rows", 0, 4), ("cols", 0, 6))


def test_halo_matches_brute_force():
    rng = random.Random(3)
    for _ in range(120):
        kernel, stride, padding = rng.randint(1, 4), rng.randint(1, 3), rng.choice(("same", "valid"))
        in_len = rng.randint(max(kernel, 4), 18)
        out_len = ps.conv_out_size(in_len, kernel, stride, padding)
        if out_len < 1:
            continue
        op = ps.Operation("cv", ps.OperatorKind("Conv1D", {"kernel": kernel, "stride": stride, "padding": padding}),
                          (ps.shape(("sample", 2), ("length", in_len), ("channel", 2)),),
                          ps.shape(("sample", 2), ("length", out_len), ("channel", 2)))
        pad = ps.pad_before(in_len, kernel, stride, padding)
        for lo in range(out_len):
            for hi in range(lo + 1, out_len + 1):
                cells = {o * stride - pad + t for o in range(lo, hi) for t in range(kernel)}
                cells = {c for c in cells if 0 <= c < in_len}
                need = dict(ps.input_regions(op, ps.region(("sample", 0, 2), ("length", lo, hi), ("channel", 0, 2))))
                assert need[0].range_of("length") == (min(cells), max(cells) + 1)


def test_strategies_and_issues():
    g = ps.alexnet_like()
    topo = ps.single_node_topology(gpus=4)
    dp = ps.data_parallel_strategy(g, topo)
    assert ps.strategy_issues(g, topo, dp) == []
    assert all(c.degrees["sample"] == 4 for c in dp.configs.values())
    rs = ps.random_strategy(g, topo, 4, 7)
    assert ps.strategy_issues(g, topo, rs) == [] and rs == ps.random_strategy(g, topo, 4, 7)
    bad = ps.ParallelizationConfig({"sample": 3}, ("gpu00",))
    assert any("does not divide" in i for i in ps.config_issues(g.ops["conv1"], bad, topo))


# -- cost ----------------------------------------------------------------------

def test_analytic_known_answers():
    op = _mm(32, 1024, 1024)
    dev = ps.single_node_topology(gpus=1).devices["gpu00"]
    t = ps.CostProfile().task_exe_time(op, ps.region(("sample", 0, 32), ("channel", 0, 1024)), dev)
    assert t == 2.0 * 1024 * (32 * 1024) / 1e12 == 6.7108864e-05
    model = ps.AnalyticCostModel(throughput={"gpu": 2e12}, overhead=1e-6)
    key = ps.cost_key_for(_mm(4, 8, 8), ps.region(("sample", 0, 4), ("channel", 0, 8)), "gpu")
    assert model.time(_mm(4, 8, 8), key) == 2.0 * 8 * 32 / 2e12 + 1e-6
    conn = ps.Connection("a", "b", 1e9, 1e-3)
    assert ps.comm_time(conn, 4_000_000) == 1e-3 + 4e-3 and ps.comm_time(conn, 0) == 1e-3


def test_cache_and_profile_format():
    op = _mm(8, 16, 8)
    dev = ps.single_node_topology(gpus=1).devices["gpu00"]
    out = ps.region(("sample", 0, 8), ("channel", 0, 8))
    p = ps.CostProfile()
    p.task_exe_time(op, out, dev)
    p.task_exe_time(op, out, dev)
    assert p.fallback_evaluations == 1
    key = ps.cost_key_for(op, out, "gpu")
    dims = ",".join(f"{n}={s}" for n, s in key.region_dims)
    q = ps.loads_profile(f"# measured\n{key.kind};{key.digest};{dims};gpu;7e-4\n")
    assert q.task_exe_time(op, out, dev) == 7e-4 and q.fallback_evaluations == 0
    assert ps.loads_profile(ps.dumps_profile(q)).entries == q.entries
    with pytest.raises(ps.ProfileFormatError, match="line 2.*5 ';'-separated"):
        ps.loads_profile("# ok\nMatMul;abc;sample=4;gpu\n")
    with pytest.raises(ps.ProfileFormatError, match="non-positive time"):
        ps.loads_profile("MatMul;abc;sample=4;gpu;0\n")
    merged = ps.merge_profiles(ps.loads_profile("MatMul;abc;sample=4;gpu;1e-5\n"),
                               ps.loads_profile("MatMul;abc;sample=4;gpu;9e-5\n"))
    assert list(merged.entries.values()) == [9e-5]


def test_digest_separates_equal_output_shapes():
    a, b = _mm(8, 16, 8), _mm(8, 32, 8)
    assert a.output_shape == b.output_shape and ps.cost_digest(a) != ps.cost_digest(b)


# -- search helpers ---------------------------------------------------------------

def test_accept_rule():
    assert ps.accept_probability(1.0, 0.5, 3.0) == 1.0 and ps.accept_probability(1.0, 1.0, 3.0) == 1.0
    assert ps.accept_probability(1.0, 1.5, 2.0) == pytest.approx(math.exp(-1.0))
    assert ps.accept_probability(2.0, 3.0, math.inf) == 0.0
    rng = random.Random(0)
    hits = sum(ps.accept(1.0, 2.0, 1.0, rng) for _ in range(20000))
    assert hits / 20000 == pytest.approx(math.exp(-1.0), abs=0.01)


def test_propose_changes_at_most_one_op():
    g = ps.alexnet_like()
    topo = ps.single_node_topology(gpus=2)
    base = ps.data_parallel_strategy(g, topo)
    for seed in range(10):
        new = ps.propose(base, g, topo, 2, random.Random(seed))
        assert ps.strategy_issues(g, topo, new) == []
        assert sum(new.configs[o] != base.configs[o] for o in g.ops) <= 1


def test_philox_random_is_a_random_subclass():
    r = ps.PhiloxRandom(5)
    xs = [r.choice(range(10)) for _ in range(1000)]
    assert set(xs) == set(range(10))
    r2 = ps.PhiloxRandom(5)
    assert [r2.choice(range(10)) for _ in range(1000)] == xs
    assert 0.0 <= ps.PhiloxRandom(1).random() < 1.0


# -- lowering and the C ABI -------------------------------------------------------

def test_lowering_tables_are_consistent():
    g = ps.inception_v3()
    topo = ps.multi_node_topology(4, 4)
    dp = ps.data_parallel_strategy(g, topo)
    low = lower(g, topo, ps.CostProfile(), ps.MODE_FULL, max_degree=4, strategies=[dp])
    a = low.arrays
    assert low.ops == sorted(g.ops) and low.devices == topo.device_ids()
    assert len(low.link_pairs) == 120
    for r, oid in enumerate(low.ops):
        enum = ps.enumerate_configs(g.ops[oid], topo, 4)
        assert low.n_enum[r] == len(enum)
        assert [low.maps[r][i] for i in range(len(enum))] == [
            tuple(c.degrees.get(n, 1) for n in g.ops[oid].output_shape.names()) for c in enum]
    m, asg = low.encode(dp)
    assert low.decode(m, asg, template=dp) == dp
    assert a["combo_off"][-1] == sum(len(low.maps[s]) * len(low.maps[d]) for s, d in low.pairs)
    # exe table == profile lookups, backward = forward * multiplier
    assert np.all(a["exe_bwd"] == a["exe_fwd"] * 2.0)


def test_native_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "parasim.h")).read()
    declared = set(re.findall(r"\b(ps_[a-z_]+)\s*\(", header))
    assert {"ps_problem_create", "ps_simulate_batch", "ps_mcmc_run", "ps_simulate_explicit"} <= declared
    lib = ctypes.CDLL(nat.LIB_PATH)  # loads without a GPU; no compute calls here
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert missing == []
    assert nat.lib().ps_abi_version() == nat.ABI_VERSION


def test_product_path_has_no_cpu_fallback(monkeypatch):
    monkeypatch.setattr(nat, "_lib", None)
    monkeypatch.setattr(nat, "_load_error", None)
    monkeypatch.setattr(nat, "LIB_PATH", "/nonexistent/libparasim_cuda.so")
    g = ps.alexnet_like()
    topo = ps.single_node_topology(gpus=4)
    with pytest.raises(nat.NativeUnavailable):
        ps.build_task_graph(g, topo, ps.data_parallel_strategy(g, topo), ps.CostProfile())


def test_random_strategies_batch_equals_single_draws():
    g, topo = ps.inception_v3(), ps.multi_node_topology(4, 4)
    seeds = [0, 1, 17, 1000003]
    batch = ps.random_strategies(g, topo, 4, seeds)
    for s, b in zip(seeds, batch):
        one = ps.random_strategy(g, topo, 4, s)
        assert {k: (c.degrees, c.assignment) for k, c in one.configs.items()} == \
            {k: (c.degrees, c.assignment) for k, c in b.configs.items()}


# -- lowering cache and task-time validation (host side) --------------------------

def test_lowering_cache_tracks_in_place_edits_and_keeps_profile_picklable():
    import copy
    import pickle
    from paper_1807_05358_b200.taskgraph import _problem_for
    g = ps.alexnet_like()
    topo = ps.single_node_topology(4)
    prof = ps.CostProfile()
    s = ps.data_parallel_strategy(g, topo)
    a = _problem_for(g, topo, prof, ps.MODE_FULL, s)
    assert _problem_for(g, topo, prof, ps.MODE_FULL, s) is a  # cache hit
    # the cache lives outside the profile: it still pickles and deep-copies
    pickle.loads(pickle.dumps(prof))
    copy.deepcopy(prof)
    # an in-place edit of a profile entry lowers again with the new value
    key = next(iter(prof.entries))
    prof.entries[key] = prof.entries[key] * 3.0
    b = _problem_for(g, topo, prof, ps.MODE_FULL, s)
    assert b is not a and key in prof.entries
    assert _problem_for(g, topo, prof, ps.MODE_FULL, s) is b
    # so does a changed link (a new Connection registered on the topology)
    topo.connections.append(ps.Connection("gpu0", "gpu1", 1.0, 0.0))
    assert _problem_for(g, topo, prof, ps.MODE_FULL, s) is not b
    # and a replaced operation
    oid = sorted(g.ops)[0]
    op = g.ops[oid]
    g.ops[oid] = ps.Operation(op.id, op.kind, op.input_shapes, op.output_shape, op.param_bytes + 4)
    c = _problem_for(g, topo, prof, ps.MODE_FULL, s)
    assert _problem_for(g, topo, prof, ps.MODE_FULL, s) is c


def test_negative_task_times_are_rejected_by_the_lowering():
    g = ps.alexnet_like()
    topo = ps.single_node_topology(4)
    prof = ps.CostProfile(fallback=ps.AnalyticCostModel(overhead=-1.0))
    with pytest.raises(ValueError, match="negative"):
        lower(g, topo, prof, ps.MODE_FORWARD, max_degree=2)
    # zero times are legal (the reference schedules them; the GPU replay is exact for them)
    lower(g, topo, ps.CostProfile(fallback=ps.AnalyticCostModel(default_throughput=math.inf)), ps.MODE_FORWARD,
          max_degree=2)
