"""Multi-GPU sharding (one process per GPU, torch.distributed).

Two decompositions:

* realization shards -- below;
* candidate-position shards of one realization -- simulate_position_sharded.

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


# ------------------------------------------------ candidate-position shards --
#
# A single realization has no independent units, but every placement's score
# map does: the reference scores the npos TI windows in row-major order and
# keeps the K best (matcher.hpp:147-204).  Shard s of S screens the windows
# [position_range(npos, s, S)) and ranks them locally under the reference's
# rule (fp64 score descending, earlier position on ties); the global top-K is
# the merge of the S local top-K lists, because each of its windows is among
# the K best of its own shard.  On the GPU the lists (16 B per candidate) are
# all-gathered with ncclAllGather once per placement wave and merged on every
# rank (libccwgpu.so, shard_merge_kernel); the functions below restate the
# partition and the merge for host tests.

def position_range(npos: int, shard: int, nshards: int) -> Tuple[int, int]:
    """[p0, p1) of shard `shard` (the C++ split in sim.cu run_simulation)."""
    if nshards < 1 or not 0 <= shard < nshards:
        raise ValueError(f"bad shard {shard} of {nshards}")
    return npos * shard // nshards, npos * (shard + 1) // nshards


def local_top_k(scores: np.ndarray, p0: int, p1: int, k: int) -> List[Tuple[float, int]]:
    """A shard's top-K (score, global position) under the reference ranking."""
    flat = np.asarray(scores, np.float64).ravel()
    pos = np.arange(p0, p1)
    order = sorted(pos.tolist(), key=lambda p: (-flat[p], p))
    return [(float(flat[p]), int(p)) for p in order[:min(k, p1 - p0)]]


def merge_top_k(lists: Sequence[Sequence[Tuple[float, int]]], k: int) -> List[Tuple[float, int]]:
    """Global top-K from the shards' lists (shard_merge_kernel's rule)."""
    allc = [c for lst in lists for c in lst]
    allc.sort(key=lambda c: (-c[0], c[1]))
    return allc[:k]


def simulate_position_sharded(ti: cs.CategoricalGrid, cfg: cs.SimConfig, seeds: Sequence[int],
                              device: Optional[cs.Device] = None, group=None,
                              virtual_shards: int = 1):
    """Simulate `seeds` with every placement's window positions sharded over
    the ranks of `group` (torch.distributed, one GPU per rank).  Rank 0 draws
    the NCCL unique id and broadcasts it; each rank's context joins one NCCL
    communicator; every rank returns the same SimResult list."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = device or cs.default_device()
    box = [cs.nccl_unique_id() if rank == 0 else None]
    # src is a global rank: group rank 0 of `group` (itself when group is None)
    src = 0 if group is None else dist.get_global_rank(group, 0)
    dist.broadcast_object_list(box, src=src, group=group)
    try:
        dev.set_position_shards(world, rank, box[0], virtual_shards)
        return cs.simulate_batch(ti, cfg, list(seeds), None, dev)
    finally:
        dev.set_position_shards(1, 0, None, 1)


# ------------------------------------------- 3D candidate-position shards --
# The 3D screen (csrc/sim3d.cu) scores boxes of TI window positions; shard s
# of S owns the boxes [s * bps, min((s + 1) * bps, nbox)) with
# bps = ceil(nbox / S), keeps each box's top-K packed keys and the per-wave
# box lists are all-gathered (ncclAllGather, rank-major) before every rank
# merges them (select3d_kernel).  Scores are exact integers, so the packed
# key alone orders candidates: (score + 2^31) << 32 | (2^32 - 1 - position).

def box_range(nbox: int, shard: int, nshards: int) -> Tuple[int, int]:
    bps = -(-nbox // nshards)
    return min(nbox, shard * bps), min(nbox, (shard + 1) * bps)


def pack_key3d(score: int, position: int) -> int:
    return ((int(score) + (1 << 31)) & 0xFFFFFFFF) << 32 | (0xFFFFFFFF - int(position))


def unpack_key3d(key: int) -> Tuple[int, int]:
    return (key >> 32) - (1 << 31), 0xFFFFFFFF - (key & 0xFFFFFFFF)


def merge_box_keys(keys: Sequence[int], k: int) -> List[int]:
    """select3d_kernel's merge: the k largest keys, descending (0 = empty)."""
    return sorted((int(x) for x in keys if x), reverse=True)[:k]
