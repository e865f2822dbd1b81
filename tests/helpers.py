"""Shared test builders (same roles as the reference's tests/helpers.py:
random valid DAGs over all eight kinds, random topologies, hand-built task
graphs), written against this package's API."""

import random

import paper_1807_05358_b200 as ps
from paper_1807_05358_b200.taskgraph import TaskGraph


def random_graph(rng: random.Random, min_ops=4, max_ops=12) -> ps.OperatorGraph:
    """A small random DAG; sizes drawn so every kind appears across seeds."""
    return ps.random_dag(rng.randint(min_ops, max_ops), seed=rng.randrange(1 << 30))


def random_topology(rng: random.Random, devices: int) -> ps.DeviceTopology:
    if devices >= 4 and devices % 2 == 0 and rng.random() < 0.5:
        return ps.multi_node_topology(nodes=2, gpus_per_node=devices // 2,
                                      intra_bandwidth=rng.choice((8e9, 16e9)),
                                      inter_bandwidth=rng.choice((2e9, 7e9)),
                                      intra_latency=rng.choice((0.0, 1e-6)),
                                      inter_latency=rng.choice((1e-6, 5e-6)))
    return ps.single_node_topology(gpus=devices, bandwidth=rng.choice((1e9, 8e9, 32e9)),
                                   latency=rng.choice((0.0, 1e-6)))


def manual_task_graph(specs, edges, devices=("d0", "d1")):
    """Bare task graph from (name, device, exe) rows; returns (tg, name->id)."""
    topo = ps.DeviceTopology()
    for d in devices:
        topo.add_device(d)
    tg = TaskGraph(ps.OperatorGraph(), topo, ps.ParallelizationStrategy({}), ps.CostProfile(), ps.MODE_FORWARD)
    ids = {}
    for name, dev, exe in specs:
        ids[name] = tg._new_task("normal", dev, exe, ("op", name, 0), name, 0).id
    for a, b in edges:
        tg._link(ids[a], ids[b])
    return tg, ids
