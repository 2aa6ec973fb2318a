"""Pin the C restatement (oracle/ccw_oracle.c) before trusting it as the
checker: against golden vectors produced by the reference itself
(tests/golden, oracle/gen_golden.py), against the compiled reference directly
when oracle/_ref is built, and against the known answers of the reference's
Catch2 suite (proj/tests/test_{wavelet,matcher,simulator}.cpp)."""
import numpy as np
import pytest

import pyoracle
from _golden import load, sim_cases


def cfg_of(d):
    return pyoracle.Cfg(**d)


@pytest.mark.parametrize("case", sim_cases(), ids=lambda c: c["name"])
def test_simulate_matches_reference_golden(oracle, case):
    cfg = cfg_of(case["cfg"])
    for i, seed in enumerate(case["seeds"]):
        r = oracle.simulate_one(case["ti"], case["nf"], cfg, case["hd"], seed=seed, trace=True)
        assert np.array_equal(r["realization"], case["real"][i])
        assert r["diagnostics"]["pre_overwrite_mismatches"] == case["mism"][i]
        assert r["diagnostics"]["origin"] == case["origin"][i]
        assert int(r["diagnostics"]["column_major"]) == case["colmajor"][i]
        assert np.array_equal(r["trace"]["ti_row"], case["ti_row"][i])
        assert np.array_equal(r["trace"]["ti_col"], case["ti_col"][i])


def test_ensemble_matches_reference_golden(oracle):
    z = load("ensemble_channel64.npz")
    cfg = pyoracle.Cfg(n_realizations=6, master_seed=int(z["master"]))
    for workers in (1, 3):
        out, diags = oracle.simulate_ensemble(z["ti"], 2, cfg, None, workers=workers)
        assert np.array_equal(out, z["real"])
        assert [d["seed"] for d in diags] == [oracle.mix64(cfg.master_seed, r + 1) for r in range(6)]


def test_wavelet_matches_reference_golden(oracle):
    z = load("wavelet.npz")
    for i in range(6):
        x, lv = z[f"x_{i}"], int(z[f"lv_{i}"])
        apex, det = oracle.dwt2(x, lv)
        assert np.array_equal(apex, z[f"apex_{i}"])
        packed = np.concatenate([np.ravel(p) for lvl in det for p in lvl])
        assert np.array_equal(packed, z[f"det_{i}"])
        back = oracle.idwt2(apex, det, x.shape[0], x.shape[1], lv)
        assert np.array_equal(back, z[f"back_{i}"])
        assert np.array_equal(np.stack(oracle.dwt2_single(x)), z[f"single_{i}"])
    for lv in (1, 2, 3):
        assert np.array_equal(oracle.dwt2(z["bin"], lv)[0], z[f"bin_apex_{lv}"])


def test_matcher_matches_reference_golden(oracle):
    z = load("matcher.npz")
    for i in range(12):
        out = oracle.score_map_channels(z[f"ti_{i}"], z[f"tm_{i}"], z[f"mask_{i}"],
                                        int(z[f"scoring_{i}"]))
        assert np.array_equal(out, z[f"out_{i}"])
    for i in range(6):
        got = np.array(oracle.top_k(z[f"topk_s_{i}"], int(z[f"topk_k_{i}"])), np.float64)
        assert np.array_equal(got, z[f"topk_{i}"])


# -- known answers restated from the reference's Catch2 suite ----------------

def test_known_answer_dwt_block(oracle):
    # test_wavelet.cpp:81-88
    a, dh, dv, dd = oracle.dwt2_single(np.array([[1.0, 1.0], [0.0, 0.0]]))
    assert abs(a[0, 0] - 1) < 1e-12 and abs(dh[0, 0] - 1) < 1e-12
    assert abs(dv[0, 0]) < 1e-12 and abs(dd[0, 0]) < 1e-12


def test_known_answer_constant_plane(oracle):
    # test_wavelet.cpp:90-103, :152-157
    a, dh, dv, dd = oracle.dwt2_single(np.full((6, 4), 3.25))
    assert a.shape == (3, 2) and np.allclose(a, 6.5, atol=1e-12, rtol=0)
    assert np.allclose(dh, 0, atol=1e-12) and np.allclose(dd, 0, atol=1e-12)
    apex, _ = oracle.dwt2(np.full((8, 8), 1.5), 3)
    assert np.allclose(apex, 12.0, atol=1e-12, rtol=0)


def test_known_answer_errors(oracle):
    # test_wavelet.cpp:116-119, :159-162
    with pytest.raises(pyoracle.OracleError) as e:
        oracle.dwt2_single(np.zeros((3, 4)))
    assert e.value.kind == "DimensionError"
    with pytest.raises(pyoracle.OracleError) as e:
        oracle.dwt2(np.zeros((12, 16)), 3)
    assert e.value.kind == "DimensionError"


def test_known_answer_top_k(oracle):
    # test_matcher.cpp:164-183, :209-214
    got = oracle.top_k(np.array([[3.0, 1.0], [2.0, 5.0]]), 2)
    assert got == [(1, 1, 5.0), (0, 0, 3.0)]
    got = oracle.top_k(np.full((2, 3), 4.0), 3)
    assert [(r, c) for r, c, _ in got] == [(0, 0), (0, 1), (0, 2)]
    assert len(oracle.top_k(np.ones((2, 2)), 10)) == 4
    with pytest.raises(pyoracle.OracleError) as e:
        oracle.top_k(np.ones((2, 2)), 0)
    assert e.value.kind == "ConfigError"


def test_known_answer_config_errors(oracle):
    # test_simulator.cpp:29-71
    ti = np.zeros((64, 64), np.uint8)
    bad = pyoracle.Cfg(template_size=32, overlap=6)
    with pytest.raises(pyoracle.OracleError) as e:
        oracle.simulate_one(ti, 2, bad, None, 1)
    assert e.value.kind == "ConfigError" and "overlap" in e.value.msg
    bad = pyoracle.Cfg(template_size=18, overlap=8)
    with pytest.raises(pyoracle.OracleError) as e:
        oracle.simulate_one(ti, 2, bad, None, 1)
    assert "template" in e.value.msg


def test_known_answer_plan(oracle):
    # test_simulator.cpp:74-106
    p = oracle.plan_raster_path(pyoracle.Cfg(sg_height=512, sg_width=512, template_size=32,
                                             overlap=8), 1)
    assert (p["work_height"], p["work_width"], len(p["tops"])) == (512, 512, 441)
    p = oracle.plan_raster_path(pyoracle.Cfg(sg_height=70), 3)
    assert p["work_height"] == 76 and p["work_width"] == 64


def test_seam_matches_exhaustive(oracle):
    # test_simulator.cpp:319-350
    rng = np.random.default_rng(8)
    for _ in range(20):
        cost = rng.integers(0, 3, (4, 8)).astype(np.int32)
        seam = oracle.min_cost_seam(cost)
        assert all(abs(int(seam[r]) - int(seam[r - 1])) <= 1 for r in range(1, 4))
        best = min(sum(cost[l, p[l]] for l in range(4))
                   for p in np.ndindex(8, 8, 8, 8)
                   if all(abs(p[l] - p[l - 1]) <= 1 for l in range(1, 4)))
        assert sum(cost[l, seam[l]] for l in range(4)) == best


@pytest.mark.skipif(not pyoracle.reference_available(), reason="oracle/_ref not built")
def test_restatement_equals_reference_randomized(oracle, reference):
    """Restatement vs the compiled reference on a seeded corpus of configs."""
    rng = np.random.default_rng(2026)
    for trial in range(24):
        J = int(rng.integers(1, 4))
        b = 1 << J
        T = b * int(rng.integers(2, 6))
        OV = b * int(rng.integers(1, T // b))
        nf = int(rng.integers(1, 5))
        H = b * int(rng.integers(T // b + 1, 96 // b + 1))
        W = b * int(rng.integers(T // b + 1, 96 // b + 1))
        ti = rng.integers(0, nf, (H, W)).astype(np.uint8)
        sg_h = int(rng.integers(T, 80))
        sg_w = int(rng.integers(T, 80))
        cfg = pyoracle.Cfg(sg_height=sg_h, sg_width=sg_w, template_size=T, overlap=OV,
                           dwt_level=J, candidates=int(rng.integers(1, 9)),
                           scoring=int(rng.integers(0, 2)), facies_mode=int(rng.integers(0, 2)),
                           min_cut=bool(rng.integers(0, 2)))
        hd = None
        if trial % 3 == 0:
            cells = rng.choice(sg_h * sg_w, size=int(rng.integers(1, 12)), replace=False)
            hd = [(int(c // sg_w), int(c % sg_w), int(rng.integers(0, nf))) for c in cells]
        seed = int(rng.integers(0, 2**63))
        a = oracle.simulate_one(ti, nf, cfg, hd, seed=seed)
        r = reference.simulate_one(ti, nf, cfg, hd, seed=seed)
        assert np.array_equal(a["realization"], r["realization"]), (trial, cfg)
        assert a["diagnostics"]["pre_overwrite_mismatches"] == r["diagnostics"]["pre_overwrite_mismatches"]


@pytest.mark.skipif(not pyoracle.reference_available(), reason="oracle/_ref not built")
def test_rng_matches_reference(oracle, reference):
    for seed in (0, 1, 5489, 2**64 - 1):
        assert np.array_equal(oracle.mt64_draws(seed, 700), reference.mt64_draws(seed, 700))
        ns = np.array([1, 2, 3, 4, 5, 7, 2**63 + 5, 10**18], np.uint64)
        assert np.array_equal(oracle.bounded_draws(seed, ns), reference.bounded_draws(seed, ns))
        assert oracle.mix64(seed, 3) == reference.mix64(seed, 3)
