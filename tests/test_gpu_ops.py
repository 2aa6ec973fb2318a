"""The fp64 operator surface on the device (ccw_dwt2_f64 / ccw_idwt2_f64 /
ccw_score_map_f64 / ccw_top_k_f64 / ccw_select_conditional /
ccw_min_cut_stitch) against the reference's outputs (tests/golden), the oracle,
and the known answers of the reference's Catch2 suite restated through the
Python mirror of ``namespace ccwsim``."""
import numpy as np
import pytest

from _golden import load
from paper_2404_00441_b200 import ccwsim as cs

pytestmark = pytest.mark.gpu


def test_wavelet_bit_exact_vs_reference():
    z = load("wavelet.npz")
    for i in range(6):
        x, lv = z[f"x_{i}"], int(z[f"lv_{i}"])
        pyr = cs.dwt2(x, lv)
        assert np.array_equal(pyr.apex, z[f"apex_{i}"])
        packed = np.concatenate([np.ravel(p) for sb in pyr.details
                                 for p in (sb.detail_h, sb.detail_v, sb.detail_d)])
        assert np.array_equal(packed, z[f"det_{i}"])
        assert np.array_equal(cs.idwt2(pyr), z[f"back_{i}"])
        s = cs.dwt2_single(x)
        assert np.array_equal(np.stack([s.approx, s.detail_h, s.detail_v, s.detail_d]), z[f"single_{i}"])
    for lv in (1, 2, 3):
        assert np.array_equal(cs.dwt2(z["bin"], lv).apex, z[f"bin_apex_{lv}"])


def test_ti_pyramid_apex_bit_exact(oracle):
    """The device TI pyramid (built once, ccw_ti_create) equals dwt2(...).apex
    of every indicator / raw-code plane (simulator.hpp:429-435)."""
    rng = np.random.default_rng(5)
    for nf, lv, mode in [(2, 2, 0), (3, 3, 0), (4, 1, 1), (5, 2, 1)]:
        a = rng.integers(0, nf, (64, 96)).astype(np.uint8)
        h = cs.TrainingImage(cs.CategoricalGrid(64, 96, nf, a), lv, mode)
        apex = h.apex()
        planes = [(a == f).astype(np.float64) for f in range(nf)] if mode == 0 else [a.astype(np.float64)]
        for f, p in enumerate(planes):
            assert np.array_equal(apex[f], oracle.dwt2(p, lv)[0])
        h.close()


def test_score_map_bit_exact_vs_reference():
    z = load("matcher.npz")
    for i in range(12):
        ti, tm, mask = z[f"ti_{i}"], z[f"tm_{i}"], z[f"mask_{i}"]
        mode = "normalized" if int(z[f"scoring_{i}"]) else "raw"
        out = cs.ccw_score_map_channels(list(ti), list(tm), mask, mode)
        assert np.array_equal(out.scores, z[f"out_{i}"])


def test_top_k_bit_exact_vs_reference():
    z = load("matcher.npz")
    for i in range(6):
        got = cs.top_k(cs.ScoreMap(z[f"topk_s_{i}"]), int(z[f"topk_k_{i}"]))
        assert np.array_equal(np.array([(c.row, c.col, c.score) for c in got.entries]), z[f"topk_{i}"])


def test_top_k_stable_sort_oracle():
    # test_matcher.cpp:185-207
    rng = cs.Mt19937_64(36)
    for _ in range(10):
        s = np.array([[float(cs.bounded(rng, 50)) for _ in range(20)] for _ in range(20)])
        got = cs.top_k(cs.ScoreMap(s), 7).entries
        order = sorted(range(400), key=lambda i: -s.flat[i])  # stable
        assert [(c.row, c.col) for c in got] == [divmod(i, 20) for i in order[:7]]


def test_matcher_known_answers():
    # test_matcher.cpp:57-116
    rng = np.random.default_rng(31)
    ti = rng.uniform(-1, 1, (8, 8))
    m = cs.ccw_score_map(ti, np.zeros((3, 3)), np.ones((3, 3)))
    assert m.scores.shape == (6, 6) and (m.scores == 0).all()
    ti = rng.uniform(-1, 1, (10, 10))
    tm = ti[4:8, 3:7].copy()
    m = cs.ccw_score_map(ti, tm, np.ones((4, 4)))
    assert abs(m.scores[4, 3] - (tm ** 2).sum()) < 1e-9
    ti = np.ones((8, 8))
    with pytest.raises(cs.StructureError):
        cs.ccw_score_map(ti, np.zeros((3, 3)), np.ones((3, 4)))
    with pytest.raises(cs.DimensionError):
        cs.ccw_score_map(ti, np.zeros((9, 3)), np.ones((9, 3)))
    bad = np.ones((3, 3))
    bad[1, 1] = 0.5
    with pytest.raises(cs.StructureError):
        cs.ccw_score_map(ti, np.zeros((3, 3)), bad)
    mask = np.ones((3, 3))
    mask[2, 2] = 0
    with pytest.raises(cs.StructureError):
        cs.ccw_score_map(ti, np.ones((3, 3)), mask)
    norm = cs.ccw_score_map_channels([np.zeros((6, 6))], [np.ones((2, 2))], np.ones((2, 2)),
                                     "normalized")
    assert (norm.scores == 0).all()


def test_score_map_corpus_vs_oracle(oracle):
    # acceptance.cpp:263-306 shape: 100 instances, J in {1,2}
    rng = np.random.default_rng(303)
    for trial in range(100):
        lv = int(rng.integers(1, 3))
        b = 1 << lv
        oh, ow = b * int(rng.integers(1, 16 // b + 1)), b * int(rng.integers(1, 16 // b + 1))
        th_, tw_ = b * int(rng.integers(oh // b, 64 // b + 1)), b * int(rng.integers(ow // b, 64 // b + 1))
        ti_ca = cs.dwt2(rng.uniform(-1, 1, (th_, tw_)), lv).apex
        or_ca = cs.dwt2(rng.uniform(-1, 1, (oh, ow)), lv).apex
        mask = (rng.integers(0, 10, or_ca.shape) < 7).astype(np.float64)
        or_ca = or_ca * mask
        got = cs.ccw_score_map(ti_ca, or_ca, mask).scores
        assert np.array_equal(got, oracle.score_map_channels(ti_ca, or_ca, mask, 0))


def test_select_conditional_fixtures():
    # test_matcher.cpp:247-315
    cells = np.array([[(r + c) % 2 for c in range(8)] for r in range(8)], np.uint8)
    cells[5, 5] = 1
    ti = cs.CategoricalGrid(8, 8, 2, cells)
    C = cs.Candidate
    s = cs.CandidateSet([C(1, 1, 9.0), C(0, 0, 8.0)])
    p = cs.select_conditional(s, [], ti, 1)
    assert (p.candidate.row, p.candidate.col, p.mismatches) == (1, 1, 0)
    s = cs.CandidateSet([C(0, 0, 9.0), C(1, 0, 8.0), C(2, 2, 7.0)])
    p = cs.select_conditional(s, [cs.HardDatum(1, 1, 1)], ti, 1)
    assert (p.candidate.row, p.candidate.col, p.mismatches) == (2, 2, 0)
    s = cs.CandidateSet([C(0, 0, 9.0), C(1, 0, 8.0)])
    p = cs.select_conditional(s, [cs.HardDatum(0, 0, 0), cs.HardDatum(0, 1, 0)], ti, 1)
    assert p.mismatches == 1 and p.candidate.score == 9.0
    with pytest.raises(cs.EmptyInputError):
        cs.select_conditional(cs.CandidateSet(), [], ti, 1)


def test_min_cut_stitch_vs_oracle(oracle):
    rng = np.random.default_rng(9)
    for trial in range(30):
        t = int(rng.integers(4, 40))
        ov = int(rng.integers(1, t))
        shape = int(rng.integers(0, 4))
        vl, ht = int(rng.integers(0, 2)), int(rng.integers(0, 2))
        e = rng.integers(0, 3, (t, t)).astype(np.uint8)
        i = rng.integers(0, 3, (t, t)).astype(np.uint8)
        got = cs.min_cut_stitch(cs.CategoricalGrid(t, t, 3, e), cs.CategoricalGrid(t, t, 3, i),
                                cs.OrGeometry(shape, bool(vl), bool(ht), ov))
        assert np.array_equal(got.cells, oracle.min_cut_stitch(e, i, shape, vl, ht, ov))


def test_wavelet_roundtrip_and_locality():
    # acceptance.cpp:235-261 (criteria 1-2), :308-347 (criterion 4)
    rng = np.random.default_rng(101)
    worst = 0.0
    for _ in range(60):
        lv = int(rng.integers(1, 4))
        b = 1 << lv
        x = rng.uniform(-1, 1, (b * int(rng.integers(2, 128 // b + 1)), b * int(rng.integers(2, 128 // b + 1))))
        pyr = cs.dwt2(x, lv)
        worst = max(worst, np.abs(cs.idwt2(pyr) - x).max())
        e = (pyr.apex ** 2).sum() + sum((sb.detail_h ** 2).sum() + (sb.detail_v ** 2).sum() +
                                        (sb.detail_d ** 2).sum() for sb in pyr.details)
        assert abs(e - (x ** 2).sum()) <= 1e-9 * (x ** 2).sum()
    assert worst < 1e-9
    x = rng.uniform(-1, 1, (64, 64))
    full = cs.dwt2(x, 2)
    sub = cs.dwt2(x[8:40, 4:36], 2)
    assert np.abs(sub.apex - full.apex[2:10, 1:9]).max() < 1e-12
    with pytest.raises(cs.DimensionError):
        cs.dwt2_single(np.zeros((3, 4)))
    with pytest.raises(cs.DimensionError):
        cs.dwt2(np.zeros((12, 16)), 3)
