"""The metrics restatement (oracle/ccw_metrics_oracle.c) pinned on the
reference's own known answers (proj/tests/test_metrics.cpp, restated: Catch2
and Eigen are absent here) and on independent numpy enumerations."""
import math
from collections import Counter

import numpy as np
import pytest

import pymetrics as M


def test_variogram_known_answers():
    # test_metrics.cpp:141-170
    g, pr = M.variogram(np.ones((6, 6), np.uint8), 1, 0, 4)
    assert (g == 0).all() and pr
    stripes = np.tile(np.arange(6) % 2, (6, 1)).astype(np.uint8)
    g, _ = M.variogram(stripes, 1, 0, 3)
    assert g.tolist() == [0.5, 0.0, 0.5]
    assert (M.variogram(stripes, 1, 1, 3)[0] == 0).all()
    g, pr = M.variogram(np.zeros((4, 4), np.uint8), 2, 0, 2)
    assert not pr and (g == 0).all()


def test_variogram_matches_pair_enumeration():
    rng = np.random.default_rng(3)
    for _ in range(5):
        g = rng.integers(0, 3, (17, 23)).astype(np.uint8)
        for d in (0, 1):
            got, _ = M.variogram(g, 1, d, 9)
            ind = (g == 1).astype(np.int64)
            for h in range(1, 10):
                a, b = (ind[:, :-h], ind[:, h:]) if d == 0 else (ind[:-h], ind[h:])
                assert got[h - 1] == 0.5 * float(((a - b) ** 2).sum()) / a.size


def test_connectivity_known_answers():
    # test_metrics.cpp:212-258
    g = np.zeros((6, 6), np.uint8)
    g[3, :] = 1
    assert (M.connectivity(g, 1, 0, 5) == 1.0).all()
    g = np.zeros((6, 6), np.uint8)
    g[:, 1] = 1
    g[:, 4] = 1
    s = M.connectivity(g, 1, 0, 4)
    assert s[2] == 0.0 and math.isnan(s[0])
    cb = (np.add.outer(np.arange(6), np.arange(6)) % 2).astype(np.uint8)
    s = M.connectivity(cb, 1, 0, 5)
    for h in range(1, 6):
        assert math.isnan(s[h - 1]) if h % 2 else s[h - 1] == 0.0
    assert np.isnan(M.connectivity(np.zeros((5, 5), np.uint8), 2, 0, 3)).all()


def _bfs_labels(g, f):
    h, w = g.shape
    lab = -np.ones((h, w), np.int64)
    k = 0
    for r in range(h):
        for c in range(w):
            if g[r, c] != f or lab[r, c] >= 0:
                continue
            stack = [(r, c)]
            lab[r, c] = k
            while stack:
                y, x = stack.pop()
                for dy, dx in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                    yy, xx = y + dy, x + dx
                    if 0 <= yy < h and 0 <= xx < w and g[yy, xx] == f and lab[yy, xx] < 0:
                        lab[yy, xx] = k
                        stack.append((yy, xx))
            k += 1
    return lab


def test_connectivity_matches_bfs():
    rng = np.random.default_rng(5)
    for _ in range(4):
        g = rng.integers(0, 2, (15, 19)).astype(np.uint8)
        lab = _bfs_labels(g, 1)
        for d in (0, 1):
            got = M.connectivity(g, 1, d, 8)
            for h in range(1, 9):
                a, b = (lab[:, :-h], lab[:, h:]) if d == 0 else (lab[:-h], lab[h:])
                both = (a >= 0) & (b >= 0)
                exp = (a == b)[both].mean() if both.any() else float("nan")
                assert (math.isnan(exp) and math.isnan(got[h - 1])) or got[h - 1] == exp


def test_ensemble_average_and_downsample():
    ones = np.ones((3, 4), np.uint8)
    assert (M.ensemble_average(np.stack([ones, ones]), 1) == 1.0).all()
    assert (M.ensemble_average(np.stack([ones, np.zeros_like(ones)]), 1) == 0.5).all()
    d = M.downsample_majority(np.array([[0, 1, 1, 2], [1, 1, 2, 1]], np.uint8), 3, 2)  # test_metrics.cpp:419-426
    assert d.tolist() == [[1, 1]]
    assert M.downsample_majority(np.ones((5, 7), np.uint8), 2, 2).shape == (2, 3)


def test_pattern_histogram_and_js():
    # test_metrics.cpp:319-356
    lst, total = M.pattern_histogram(np.ones((5, 5), np.uint8), 2)
    assert total == 16 and lst == [(b"\x01" * 4, 16)]
    rng = np.random.default_rng(45)
    g = rng.integers(0, 3, (10, 10)).astype(np.uint8)
    lst, total = M.pattern_histogram(g, 3)
    exp = Counter(g[r:r + 3, c:c + 3].tobytes() for r in range(8) for c in range(8))
    assert total == 64 and dict(lst) == dict(exp)
    assert M.pattern_histogram(rng.integers(0, 2, (9, 9)).astype(np.uint8), 3, 3)[1] == 9
    # js_divergence (test_metrics.cpp:360-415) on 1x1 windows
    p = ([(b"a", 1)], 1)
    q = ([(b"a", 1), (b"b", 1)], 2)
    assert abs(M.js_divergence(p, q, 1) - 0.31128) < 1e-4
    assert M.js_divergence(p, p, 1) == 0.0
    disj = M.js_divergence(([(b"a", 2), (b"b", 2)], 4), ([(b"c", 1), (b"d", 3)], 4), 1)
    assert abs(disj - 1.0) < 1e-12


def _anodi_case(seed=49):
    rng = np.random.default_rng(seed)
    ti = np.zeros((32, 32), np.uint8)
    ti[8:12, :] = 1
    ti[20:23, 3:29] = 1
    a = rng.integers(0, 2, (3, 32, 32)).astype(np.uint8)
    b = rng.integers(0, 2, (3, 32, 32)).astype(np.uint8)
    return a, b, ti


def test_anodi_known_answers():
    # test_metrics.cpp:440-523, acceptance.cpp:610-630
    a, b, ti = _anodi_case()
    lv, agg = M.anodi(a, a, ti, 2, 3, 4)
    assert lv.shape == (3, 8)
    for row in lv:
        assert abs(row[4] - 1) < 1e-12 and abs(row[5] - 1) < 1e-12 and abs(row[6] - 1) < 1e-12
        assert abs(row[7] - 1 / 3) < 1e-12
    assert abs(agg - 1) < 1e-9
    lv, agg = M.anodi(a, b, ti, 2, 2, 4)
    assert abs(agg - float((lv[:, 7] * lv[:, 6]).sum())) < 1e-12
    lv, agg = M.anodi(a, b, ti, 2, 2, 4, [0.75, 0.25])
    assert lv[0, 7] == 0.75 and lv[1, 7] == 0.25
    assert abs(agg - (0.75 * lv[0, 6] + 0.25 * lv[1, 6])) < 1e-12
    with pytest.raises(RuntimeError, match="DegeneracyError"):
        M.anodi(np.stack([ti, ti]), np.stack([ti, ti]), ti, 2, 2, 4)
    with pytest.raises(RuntimeError, match="EmptyInputError"):
        M.anodi(a[:1], b, ti, 2, 2, 4)


def test_anodi_matches_from_scratch_evaluation():
    # test_metrics.cpp:474-513: every level statistic from downsample + histogram + JS
    a, b, ti = _anodi_case(7)
    win = 4
    lv, _ = M.anodi(a, b, ti, 2, 2, win)
    for level in (1, 2):
        f = 1 << (level - 1)
        hist = lambda g: M.pattern_histogram(M.downsample_majority(g, 2, f) if f > 1 else g, win)
        th = hist(ti)

        def pairwise(e):
            v = [M.js_divergence(hist(e[i]), hist(e[j]), win) for i in range(len(e)) for j in range(i + 1, len(e))]
            return sum(v) / len(v)

        def vs_ti(e):
            return sum(M.js_divergence(hist(g), th, win) for g in e) / len(e)

        row = lv[level - 1]
        assert abs(row[0] - pairwise(a)) < 1e-9 and abs(row[1] - pairwise(b)) < 1e-9
        assert abs(row[2] - vs_ti(a)) < 1e-9 and abs(row[3] - vs_ti(b)) < 1e-9
        assert abs(row[6] - (row[0] / row[1]) / (row[2] / row[3])) < 1e-9
