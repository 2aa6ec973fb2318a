"""Multi-GPU realization sharding (one process per GPU, torch.distributed).

Realizations are independent -- realization r is a pure function of
(TI, config, mix64(master, r + 1)) (simulator.hpp:523-566) -- so
an ensemble shards across ranks with no data-path collective: rank k of W
simulates the realizations r with r % W == k.  The only communication is the
optional gather of results to one rank.  The output is identical for every
world size, as the reference requires for every worker count
(test_simulator.cpp:543-551).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import ccwsim as cs


def shard_indices(n_total: int, rank: int, world: int) -> List[int]:
    """Global realization indices owned by `rank` (round-robin)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    return list(range(rank, n_total, world))


def shard_seeds(master_seed: int, n_total: int, rank: int, world: int) -> List[Tuple[int, int]]:
    """(global index, seed) pairs of this rank's realizations."""
    return [(r, cs.mix64(master_seed, r + 1)) for r in shard_indices(n_total, rank, world)]


def simulate_shard(ti: cs.CategoricalGrid, cfg: cs.SimConfig, rank: int, world: int,
                   simulate: Optional[Callable[[Sequence[int]], np.ndarray]] = None,
                   device: Optional[cs.Device] = None) -> Tuple[List[int], np.ndarray]:
    """Simulate this rank's share of cfg.n_realizations.  Returns the global
    indices and an (n_local, sg_h, sg_w) uint8 array.  `simulate` (seeds ->
    array) replaces the device call, e.g. for CPU tests with the oracle."""
    pairs = shard_seeds(cfg.master_seed, cfg.n_realizations, rank, world)
    idx = [r for r, _ in pairs]
    seeds = [s for _, s in pairs]
    if not seeds:
        return idx, np.zeros((0, cfg.sg_height, cfg.sg_width), np.uint8)
    if simulate is not None:
        return idx, np.asarray(simulate(seeds), np.uint8)
    res = cs.simulate_batch(ti, cfg, seeds, None, device)
    return idx, np.stack([r.realization.cells for r in res])


def gather_ensemble(idx: List[int], local: np.ndarray, n_total: int, dst: int = 0,
                    group=None) -> Optional[np.ndarray]:
    """Gather every rank's shard to `dst`, ordered by realization index
    (torch.distributed; works with nccl and gloo).  Returns None off `dst`."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    objs = [None] * world if rank == dst else None
    dist.gather_object((idx, local), objs, dst=dst, group=group)
    if rank != dst:
        return None
    h, w = local.shape[1:]
    out = np.zeros((n_total, h, w), np.uint8)
    for ids, arr in objs:
        for j, r in enumerate(ids):
            out[r] = arr[j]
    return out
