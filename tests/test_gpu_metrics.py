"""On-device validation metrics (csrc/metrics.cu) against the metrics
restatement (oracle/ccw_metrics_oracle.c, pinned in test_metrics_cpu.py):
integer-derived quantities (variograms, connectivity, ensemble averages,
histogram counts, downsampling) exactly; JS divergence within 1e-12 (the
reference sums over an unordered_map, so its term order is unspecified)."""
import math

import numpy as np
import pytest

import pymetrics as M
from paper_2404_00441_b200 import ccwsim as cs
from paper_2404_00441_b200 import metrics as G
from paper_2404_00441_b200 import synth

pytestmark = pytest.mark.gpu


def ensemble(n=6, h=96, w=130, seed=3):
    ti_a = synth.channel_levee_ti(160, 160, 77)
    ti = cs.CategoricalGrid(160, 160, 3, ti_a)
    cfg = cs.SimConfig(h, w, 32, 8, 2, 3)
    res = cs.simulate_batch(ti, cfg, [cs.mix64(seed, r + 1) for r in range(n)])
    return np.stack([r.realization.cells for r in res]), ti_a


def test_variograms_exact():
    grids, _ = ensemble()
    for f in (0, 1, 2):
        for d in (0, 1):
            lag = 40 if d == 0 else 30
            g, pr = G.indicator_variograms(grids, f, d, lag)
            for r in range(len(grids)):
                e, ep = M.variogram(grids[r], f, d, lag)
                assert np.array_equal(g[r], e) and pr[r] == ep, (f, d, r)
    # wide grids: lags that cross 64-cell words
    rng = np.random.default_rng(1)
    wide = rng.integers(0, 2, (3, 20, 333)).astype(np.uint8)
    g, _ = G.indicator_variograms(wide, 1, 0, 200)
    for r in range(3):
        assert np.array_equal(g[r], M.variogram(wide[r], 1, 0, 200)[0])


def test_connectivity_exact():
    grids, _ = ensemble()
    for f in (0, 1):
        for d in (0, 1):
            p = G.connectivity_functions(grids, f, d, 25)
            for r in range(len(grids)):
                e = M.connectivity(grids[r], f, d, 25)
                assert np.array_equal(np.isnan(p[r]), np.isnan(e))
                assert np.array_equal(p[r][~np.isnan(e)], e[~np.isnan(e)]), (f, d, r)
    # long sinuous components (union-find under contention)
    ti = synth.channel_ti(400, 500, 5)
    p = G.connectivity_functions(ti, 1, 0, 300)[0]
    e = M.connectivity(ti, 1, 0, 300)
    assert np.array_equal(p[~np.isnan(e)], e[~np.isnan(e)])


def test_known_answers_on_device():
    # test_metrics.cpp:141-170, 212-258 through the product API
    stripes = cs.CategoricalGrid(6, 6, 2, np.tile(np.arange(6) % 2, (6, 1)).astype(np.uint8))
    assert G.indicator_variogram(stripes, 1, "east_west", 3).gamma == [0.5, 0.0, 0.5]
    assert not G.indicator_variogram(cs.CategoricalGrid(4, 4, 3, fill=0), 2, "east_west", 2).facies_present
    with pytest.raises(cs.DimensionError, match="max_lag"):
        G.indicator_variogram(cs.CategoricalGrid(4, 6, 2, fill=0), 0, "east_west", 6)
    g = np.zeros((6, 6), np.uint8)
    g[:, 1] = 1
    g[:, 4] = 1
    s = G.connectivity_function(cs.CategoricalGrid(6, 6, 2, g), 1, "east_west", 4)
    assert s.probability[0] is None and s.probability[2] == 0.0


def test_ensemble_average_exact_on_device_buffer():
    """The ensemble straight from ccw_simulate_device's output buffer (HBM)."""
    import ctypes as C
    import torch
    from paper_2404_00441_b200 import _abi
    ti_a = synth.channel_levee_ti(160, 160, 77)
    ti = cs.CategoricalGrid(160, 160, 3, ti_a)
    cfg = cs.SimConfig(96, 130, 32, 8, 2, 3)
    dev = cs.default_device()
    tih = cs.TrainingImage(ti, 2, "indicator", dev)
    seeds = np.array([cs.mix64(3, r + 1) for r in range(6)], np.uint64)
    d_out = torch.empty((6, 96, 130), dtype=torch.uint8, device="cuda:0")
    dev.check(dev._lib.ccw_simulate_device(dev.handle, tih.handle, C.byref(cfg.to_c()),
                                           seeds.ctypes.data_as(_abi.U64P), 6, None, 0,
                                           C.c_void_p(d_out.data_ptr()), None))
    torch.cuda.synchronize()
    host = d_out.cpu().numpy()
    for f in range(3):
        assert np.array_equal(G.ensemble_average(d_out, f), M.ensemble_average(host, f))
    g, _ = G.indicator_variograms(d_out, 1, 1, 20)
    for r in range(6):
        assert np.array_equal(g[r], M.variogram(host[r], 1, 1, 20)[0])


def test_pattern_histograms_and_js():
    grids, ti_a = ensemble()
    for win, stride in ((3, 1), (4, 2), (7, 1)):
        ht = G.pattern_histogram(ti_a, win, stride, num_facies=3)
        et, tt = M.pattern_histogram(ti_a, win, stride)
        assert ht.total == tt and ht.counts == dict(et)
        for r in range(3):
            hr = G.pattern_histogram(grids[r], win, stride, num_facies=3)
            er = M.pattern_histogram(grids[r], win, stride)
            assert hr.counts == dict(er[0])
            js = G.js_divergence(hr, ht)
            assert abs(js - M.js_divergence(er, (et, tt), win)) < 1e-12
            assert abs(js - G.js_divergence(ht, hr)) < 1e-12
            assert 0.0 <= js <= 1.0
        assert G.js_divergence(ht, ht) == 0.0


def test_downsample_exact():
    grids, _ = ensemble(n=2)
    for factor in (1, 2, 3, 5):
        g = cs.CategoricalGrid(grids.shape[1], grids.shape[2], 3, grids[0])
        d = G.downsample_majority(g, factor)
        assert np.array_equal(d.cells, M.downsample_majority(grids[0], 3, factor))


def test_anodi_matches_restatement():
    grids, ti_a = ensemble(n=8)
    ga, gb = grids[:4], grids[4:]
    for levels, win, wts in ((3, 3, None), (2, 4, [0.75, 0.25])):
        res = G.anodi(ga, gb, ti_a, levels, win, wts, num_facies=3)
        exp, agg = M.anodi(ga, gb, ti_a, 3, levels, win, wts)
        got = np.array([[l.between_a, l.between_b, l.within_a, l.within_b, l.d_between, l.d_within, l.ratio,
                         l.weight] for l in res.levels])
        assert np.allclose(got, exp, rtol=0, atol=1e-9), (got, exp)
        assert abs(res.aggregate - agg) < 1e-9
    # identical ensembles: r = 1 (test_metrics.cpp:449-459); on-device input
    import torch
    d = torch.from_numpy(ga).cuda()
    res = G.anodi(d, d, ti_a, 2, 3, num_facies=3)
    assert abs(res.aggregate - 1.0) < 1e-9
    with pytest.raises(cs.DegeneracyError):
        G.anodi([ti_a[:96, :130]] * 2, [ti_a[:96, :130]] * 2, ti_a[:96, :130], 2, 3, num_facies=3)
    with pytest.raises(cs.EmptyInputError):
        G.anodi(ga[:1], gb, ti_a, 2, 3, num_facies=3)
