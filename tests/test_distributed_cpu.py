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
