"""World-size-2 gloo test of the realization-sharded ensemble path
(paper_2404_00441_b200/distributed.py), with the oracle as the CPU compute:
the gathered ensemble equals the single-process ensemble, in order."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    import pyoracle
    from paper_2404_00441_b200 import ccwsim as cs, distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(5)
    ti_a = rng.integers(0, 3, (64, 64)).astype(np.uint8)
    ti = cs.CategoricalGrid(64, 64, 3, ti_a)
    cfg = cs.SimConfig(48, 56, 16, 4, 2, 3, n_realizations=7, master_seed=99)
    o = pyoracle.restatement()
    sim = lambda seeds: [o.simulate_one(ti_a, 3, cfg, None, seed=s)["realization"] for s in seeds]
    idx, local = D.simulate_shard(ti, cfg, rank, world, simulate=sim)
    assert idx == list(range(rank, 7, world))
    full = D.gather_ensemble(idx, local, cfg.n_realizations)
    if rank == 0:
        np.save(out_path, full)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_ensemble_matches_single_process(tmp_path, oracle):
    port = _free_port()
    out = str(tmp_path / "ens.npy")
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    rng = np.random.default_rng(5)
    ti_a = rng.integers(0, 3, (64, 64)).astype(np.uint8)
    import pyoracle
    cfg = pyoracle.Cfg(sg_height=48, sg_width=56, template_size=16, overlap=4, dwt_level=2,
                       candidates=3, n_realizations=7, master_seed=99)
    ref, _ = oracle.simulate_ensemble(ti_a, 3, cfg, None, workers=2)
    assert np.array_equal(got, ref)


def test_shard_indices_partition():
    from paper_2404_00441_b200 import distributed as D
    for n in (0, 1, 7, 100):
        for world in (1, 2, 3, 8):
            parts = [D.shard_indices(n, r, world) for r in range(world)]
            assert sorted(i for p in parts for i in p) == list(range(n))
    with pytest.raises(ValueError):
        D.shard_indices(5, 3, 2)


def _pos_worker(rank, world, port, out_path):
    """One placement's score map, window positions sharded over the ranks:
    local top-K per rank, all-gathered over gloo, merged on every rank."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    import pyoracle
    from paper_2404_00441_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = pyoracle.restatement()
    results = []
    for trial in range(6):
        rng = np.random.default_rng(300 + trial)
        b = 4
        # blocky apex planes: many exact ties, some across shard boundaries
        ti = np.repeat(np.repeat(rng.integers(0, 2, (3, 12, 12)), 2, 1), 2, 2).astype(np.float64) * b
        tm = rng.integers(0, 2, (3, 6, 6)).astype(np.float64) * b
        mask = np.zeros((6, 6))
        mask[:2, :] = 1
        mask[:, :2] = 1
        tm *= mask
        s = o.score_map_channels(ti, tm, mask)
        k = int(rng.integers(1, 9))
        p0, p1 = D.position_range(s.size, rank, world)
        mine = D.local_top_k(s, p0, p1, k)
        lists = [None] * world
        dist.all_gather_object(lists, mine)
        merged = D.merge_top_k(lists, k)
        results.append([(p // s.shape[1], p % s.shape[1], v) for v, p in merged])
    if rank == 0:
        np.save(out_path, np.array(results, dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_position_sharded_top_k_matches_reference(tmp_path, oracle, world):
    """8(e) single-realization decomposition: merging the ranks' local top-K
    lists reproduces the reference's top_k (matcher.hpp:177-204) exactly,
    including its earlier-position tie rule."""
    port = _free_port()
    out = str(tmp_path / "topk.npy")
    mp.start_processes(_pos_worker, args=(world, port, out), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out, allow_pickle=True)
    for trial in range(6):
        rng = np.random.default_rng(300 + trial)
        ti = np.repeat(np.repeat(rng.integers(0, 2, (3, 12, 12)), 2, 1), 2, 2).astype(np.float64) * 4
        tm = rng.integers(0, 2, (3, 6, 6)).astype(np.float64) * 4
        mask = np.zeros((6, 6))
        mask[:2, :] = 1
        mask[:, :2] = 1
        tm *= mask
        s = oracle.score_map_channels(ti, tm, mask)
        k = int(rng.integers(1, 9))
        assert [tuple(c) for c in got[trial]] == oracle.top_k(s, k)


def test_position_ranges_partition():
    from paper_2404_00441_b200 import distributed as D
    for npos in (1, 7, 49, 12100):
        for S in range(1, min(npos, 9) + 1):
            rs = [D.position_range(npos, s, S) for s in range(S)]
            assert rs[0][0] == 0 and rs[-1][1] == npos
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(p1 > p0 for p0, p1 in rs)
    with pytest.raises(ValueError):
        D.position_range(10, 2, 2)


def _worker3d(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist
    import pyoracle3d as P3
    from paper_2404_00441_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o3 = P3.oracle3()
    rng = np.random.default_rng(11)
    ti = rng.integers(0, 3, (24, 28, 32)).astype(np.uint8)
    cnt = o3.block_counts(ti, 3, 1)
    n = rng.integers(0, 8, (3, 4, 4, 4)).astype(np.int32)
    mask = np.zeros((4, 4, 4), np.uint8)
    mask[:2] = 1
    mask[:, :2] = 1
    n[:, mask == 0] = 0
    S = o3.score_map(cnt, n, mask)  # (9, 11, 13) positions
    K = 4
    # boxes of 3 x 4 x 8 positions, shard = this rank's box range
    nb = [-(-S.shape[0] // 3), -(-S.shape[1] // 4), -(-S.shape[2] // 8)]
    nbox = nb[0] * nb[1] * nb[2]
    b0, b1 = D.box_range(nbox, rank, world)
    bps = -(-nbox // world)
    mine = np.zeros((bps, K), np.uint64)
    for b in range(b0, b1):
        q2, q1, q0 = b % nb[2], (b // nb[2]) % nb[1], b // (nb[2] * nb[1])
        keys = []
        for p0 in range(q0 * 3, min(S.shape[0], q0 * 3 + 3)):
            for p1 in range(q1 * 4, min(S.shape[1], q1 * 4 + 4)):
                for p2 in range(q2 * 8, min(S.shape[2], q2 * 8 + 8)):
                    pos = (p0 * S.shape[1] + p1) * S.shape[2] + p2
                    keys.append(D.pack_key3d(int(S[p0, p1, p2]), pos))
        top = D.merge_box_keys(keys, K)
        mine[b - b0, :len(top)] = top
    # ncclAllGather stand-in: gloo all_gather of the rank's box lists
    t = torch.from_numpy(mine.view(np.int64).copy())
    parts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    allk = np.concatenate([p.numpy().view(np.uint64).ravel() for p in parts])
    merged = D.merge_box_keys([int(x) for x in allk], K)
    if rank == 0:
        np.save(out_path, np.array([D.unpack_key3d(k) for k in merged], np.int64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_3d_position_shards_merge(tmp_path, world):
    """3D position shards over gloo: per-rank box top-K lists of an exact
    score map, all-gathered and merged, equal the map's global top-K
    (score desc, earlier row-major position on ties)."""
    port = _free_port()
    out = str(tmp_path / "m3.npy")
    mp.start_processes(_worker3d, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    got = np.load(out)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle3d as P3
    o3 = P3.oracle3()
    rng = np.random.default_rng(11)
    ti = rng.integers(0, 3, (24, 28, 32)).astype(np.uint8)
    cnt = o3.block_counts(ti, 3, 1)
    n = rng.integers(0, 8, (3, 4, 4, 4)).astype(np.int32)
    mask = np.zeros((4, 4, 4), np.uint8)
    mask[:2] = 1
    mask[:, :2] = 1
    n[:, mask == 0] = 0
    flat = o3.score_map(cnt, n, mask).ravel()
    best = sorted(range(flat.size), key=lambda q: (-flat[q], q))[:4]
    assert got.tolist() == [[int(flat[q]), q] for q in best]
