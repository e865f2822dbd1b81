"""Chain sharding across GPUs and the one exchange step at the end of a search.

Chains are independent given (initial strategy, seed), so rank
r of W owns the contiguous block of chains ``shard(r, W, n)`` and nothing
crosses GPUs while chains run.  When the search ends, the global winner is the
chain with the smallest best cost, earliest chain index on ties -- the
reference's strict-``<`` scan over chains in order (search.py:256) -- found with
two MIN all-reduces over 8-byte scalars, followed by a broadcast of the winning
strategy (a few KB) from its owner.  Works over NCCL (GPU tensors) and gloo
(CPU tensors, used by the tests).
"""

from __future__ import annotations

import numpy as np

__all__ = ["shard", "global_best"]


def shard(rank: int, world: int, n: int) -> range:
    """Contiguous block of chain indices owned by ``rank``."""
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return range(lo, hi)


def global_best(best_cost: float, best_chain: int, map_local: np.ndarray, assign: np.ndarray, device=None):
    """(cost, chain, map_local, assign) of the global winner on every rank.

    ``best_chain`` is the rank's winning *global* chain index (or -1 if all of
    its chains failed, with best_cost = inf)."""
    import torch
    import torch.distributed as dist

    dev = device if device is not None else torch.device("cpu")
    cost = torch.tensor([best_cost], dtype=torch.float64, device=dev)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(cost, op=dist.ReduceOp.MIN)
    win_cost = float(cost.item())
    big = np.iinfo(np.int64).max
    mine = best_chain if (best_chain >= 0 and best_cost == win_cost) else big
    chain = torch.tensor([mine], dtype=torch.int64, device=dev)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(chain, op=dist.ReduceOp.MIN)
    win_chain = int(chain.item())
    if win_chain == big:
        return win_cost, -1, None, None
    m = torch.as_tensor(np.ascontiguousarray(map_local, dtype=np.int32)).to(dev)
    a = torch.as_tensor(np.ascontiguousarray(assign, dtype=np.uint8)).to(dev)
    if dist.is_initialized() and dist.get_world_size() > 1:
        owner = torch.tensor([dist.get_rank() if mine == win_chain else -1], dtype=torch.int64, device=dev)
        dist.all_reduce(owner, op=dist.ReduceOp.MAX)
        dist.broadcast(m, src=int(owner.item()))
        dist.broadcast(a, src=int(owner.item()))
    return win_cost, win_chain, m.cpu().numpy(), a.cpu().numpy()
