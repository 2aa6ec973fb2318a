"""CPU checks of the 3D extension's oracle (oracle/ccw3d_oracle.c): the C
restatement against the independent pure-Python loop restatement of the same
definition (oracle/pyoracle3d.py, written from ccw3d_oracle.h), validation
messages, plan geometry and the wave-key ordering property the device
schedule relies on.  The reference has no 3D, so these two
restatements pin each other ("parity restatement-pinned")."""
import itertools

import numpy as np
import pytest

import pyoracle3d as P3


@pytest.fixture(scope="module")
def o3():
    return P3.oracle3()


def blocky(rng, shape, nf, cell=2):
    g = rng.integers(0, nf, tuple(-(-s // cell) for s in shape))
    for a in range(3):
        g = g.repeat(cell, a)
    return np.ascontiguousarray(g[:shape[0], :shape[1], :shape[2]]).astype(np.uint8)


@pytest.mark.parametrize("block", range(3))
def test_c_restatement_equals_python_loops(o3, block):
    rng = np.random.default_rng(70 + block)
    for trial in range(6):
        J = int(rng.integers(1, 3))
        B = 1 << J
        tcb = int(rng.integers(2, 4))
        T = B * tcb
        anys = trial % 2 == 1
        OV = int(rng.integers(1, T)) if anys else B * int(rng.integers(1, tcb))
        nf = int(rng.integers(1, 5))
        dims = tuple(int(B * rng.integers(tcb + 1, tcb + 3) + (int(rng.integers(0, B)) if anys else 0))
                     for _ in range(3))
        ti = blocky(rng, dims, nf, int(rng.integers(1, 3)))
        sg = tuple(int(v) for v in rng.integers(T, T + 2 * (T - OV) + 3, 3))
        cfg = P3.Cfg3(sg=sg, template_size=T, overlap=OV, dwt_level=J,
                      candidates=int(rng.integers(1, 5)), any_support=anys)
        hd = None
        if trial >= 3:
            cells = rng.choice(int(np.prod(sg)), 12, replace=False)
            hd = [(*np.unravel_index(int(c), sg), int(rng.integers(0, nf))) for c in cells]
            hd = [tuple(int(v) for v in h) for h in hd]
        for seed in (5, 6):
            a = o3.simulate_one(ti, nf, cfg, hd, seed)
            b, mism = P3.py_simulate_one(ti, nf, cfg, hd, seed)
            assert np.array_equal(a["realization"], b), (block, trial, seed)
            assert a["diagnostics"]["pre_overwrite_mismatches"] == mism
            c = o3.simulate_one(ti, nf, cfg, hd, seed, threads=3)
            assert np.array_equal(c["realization"], b)


def test_block_counts_and_score_map(o3):
    rng = np.random.default_rng(3)
    ti = blocky(rng, (12, 16, 20), 3, 1)
    cnt = o3.block_counts(ti, 3, 2)
    ref = np.stack([(ti == f).reshape(3, 4, 4, 4, 5, 4).sum(axis=(1, 3, 5)) for f in range(3)])
    assert np.array_equal(cnt, ref)
    n = rng.integers(0, 10, (3, 2, 2, 2)).astype(np.int32)
    mask = np.array([1, 0, 1, 1, 0, 1, 1, 1], np.uint8).reshape(2, 2, 2)
    n[:, mask == 0] = 0
    S = o3.score_map(cnt, n, mask)
    exp = np.zeros((2, 3, 4), np.int64)
    for p in itertools.product(range(2), range(3), range(4)):
        exp[p] = sum(int(cnt[f, p[0] + m0, p[1] + m1, p[2] + m2]) * int(n[f, m0, m1, m2])
                     for f in range(3) for m0 in range(2) for m1 in range(2) for m2 in range(2)
                     if mask[m0, m1, m2])
    assert np.array_equal(S, exp)


def test_validation_messages(o3):
    ok = P3.Cfg3(sg=(32, 32, 32), template_size=16, overlap=4, dwt_level=2)
    o3.validate(ok, (32, 32, 32), 2)
    with pytest.raises(P3.Oracle3Error, match="overlap: 6 not divisible"):
        o3.validate(P3.Cfg3(sg=(32, 32, 32), template_size=16, overlap=6, dwt_level=2))
    o3.validate(P3.Cfg3(sg=(32, 32, 32), template_size=16, overlap=6, dwt_level=2, any_support=True))
    with pytest.raises(P3.Oracle3Error, match="not divisible by 2\\^dwt_level"):
        o3.validate(ok, (32, 30, 32), 2)
    o3.validate(P3.Cfg3(sg=(32, 32, 32), template_size=16, overlap=4, dwt_level=2, any_support=True),
                (32, 30, 32), 2)
    with pytest.raises(P3.Oracle3Error, match="exceeds training image"):
        o3.validate(ok, (32, 12, 32), 2)
    with pytest.raises(P3.Oracle3Error, match="outside 32x32x32 grid"):
        o3.validate(ok, (32, 32, 32), 2, [(0, 0, 32, 1)])
    with pytest.raises(P3.Oracle3Error, match="duplicate hard data"):
        o3.validate(ok, (32, 32, 32), 2, [(1, 2, 3, 1), (1, 2, 3, 0)])
    with pytest.raises(P3.Oracle3Error, match="facies 2 outside"):
        o3.validate(ok, (32, 32, 32), 2, [(1, 2, 3, 2)])


def test_plan_geometry(o3):
    """Stride lattice per axis, padded work extents (simulator.hpp:125-131 per
    axis), all 8 corners x 6 axis orders reachable, shapes = slabs on the axes
    whose traversal index is > 0, raster order = outer/middle/inner."""
    cfg = P3.Cfg3(sg=(40, 50, 70), template_size=16, overlap=4, dwt_level=2)
    seen = set()
    for seed in range(1, 400):
        p = o3.plan(cfg, seed)
        seen.add((p["corner"], p["order"]))
        assert p["work"] == (40, 52, 76)
        assert len(p["shapes"]) == 3 * 4 * 6
        assert p["shapes"][0] == 0 and (p["shapes"][1:] != 0).all()
        outer, middle, inner = P3.ORDERS[p["order"]]
        org = p["origins"]
        # the inner axis varies fastest
        assert org[1][inner] != org[0][inner] and org[1][outer] == org[0][outer]
    assert len(seen) == 48


def test_wave_keys_order_overlapping_placements(o3):
    """The device schedule runs placements in waves keyed
    (d+1)^2 io + (d+1) im + ii: every overlapping pair is ordered as in the
    raster loop, and placements sharing a wave never overlap."""
    for T, OV in ((16, 4), (16, 8), (24, 16), (12, 10)):
        cfg = P3.Cfg3(sg=(40, 44, 48), template_size=T, overlap=OV, dwt_level=1)
        stride = T - OV
        d = -(-T // stride) - 1
        for seed in (1, 2, 3, 4):
            p = o3.plan(cfg, seed)
            order = P3.ORDERS[p["order"]]
            org = p["origins"]
            idx = []
            for k in range(len(org)):
                pos = []
                for a in range(3):
                    lat = org[k][a] // stride
                    n = (p["work"][a] - T) // stride + 1
                    pos.append(lat if not (p["corner"] >> a) & 1 else n - 1 - lat)
                idx.append(pos)
            idx = np.array(idx)
            key = (d + 1) ** 2 * idx[:, order[0]] + (d + 1) * idx[:, order[1]] + idx[:, order[2]]
            o = org.astype(np.int64)
            overlap = (np.abs(o[:, None, :] - o[None, :, :]) < T).all(axis=2)
            later = np.arange(len(o))[:, None] < np.arange(len(o))[None, :]  # raster order a < b
            bad = overlap & later & ~(key[:, None] < key[None, :])
            assert not bad.any(), (T, OV, seed)
