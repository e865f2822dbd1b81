"""Multi-process (gloo, world_size 2) checks of the N>1 host logic: chain
sharding and the end-of-search exchange (earliest chain wins ties)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1807_05358_b200.parallel import global_best, shard


def test_shard_covers_every_chain_once():
    for n in (1, 7, 1024, 1025):
        for w in (1, 2, 3, 8):
            got = [c for r in range(w) for c in shard(r, w, n)]
            assert got == list(range(n))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        for costs, chains in cases:
            m = np.full(5, rank * 10 + 1, dtype=np.int32)
            a = np.full(7, rank + 3, dtype=np.uint8)
            res.append(global_best(costs[rank], chains[rank], m, a))
        out.put((rank, [(c, i, None if mm is None else mm.tolist(), None if aa is None else aa.tolist())
                        for c, i, mm, aa in res]))
    finally:
        dist.destroy_process_group()


def test_global_best_gloo_world2():
    inf = float("inf")
    cases = [
        ((2.0, 1.0), (0, 600)),        # rank 1 wins outright
        ((1.0, 1.0), (5, 512)),        # tie: earliest chain (rank 0's chain 5) wins
        ((1.0, 1.0), (700, 3)),        # tie: chain 3 on rank 1 is earlier
        ((inf, 0.5), (-1, 513)),       # rank 0 has no live chain
    ]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [(1.0, 600, 1), (1.0, 5, 0), (1.0, 3, 1), (0.5, 513, 1)]
    for r in range(2):
        for (cost, chain, m, a), (wc, wch, owner) in zip(results[r], want):
            assert (cost, chain) == (wc, wch)
            assert m == [owner * 10 + 1] * 5 and a == [owner + 3] * 7
