"""Parity of the CUDA simulation path (libccwgpu.so) with the reference:
bit-identical realizations, diagnostics and provenance traces against the
reference's own outputs (tests/golden) and against the oracle restatement on a
seeded corpus; size-independent properties at the BASELINE configs' sizes."""
import numpy as np
import pytest

import pyoracle
from _golden import load, sim_cases
from paper_2404_00441_b200 import ccwsim as cs

pytestmark = pytest.mark.gpu


def to_cfg(d, hd=None):
    names = {0: "raw", 1: "normalized"}
    modes = {0: "indicator", 1: "raw_codes"}
    cfg = cs.SimConfig(sg_height=d["sg_height"], sg_width=d["sg_width"],
                       template_size=d["template_size"], overlap=d["overlap"],
                       dwt_level=d["dwt_level"], candidates=d["candidates"],
                       n_realizations=d.get("n_realizations", 1),
                       master_seed=d.get("master_seed", 0), scoring=names[d.get("scoring", 0)],
                       facies_mode=modes[d.get("facies_mode", 0)],
                       min_cut=bool(d.get("min_cut", 0)))
    if hd:
        cfg.hard_data = cs.HardDataSet([cs.HardDatum(*p) for p in hd])
    return cfg


@pytest.mark.parametrize("case", sim_cases(), ids=lambda c: c["name"])
def test_golden_realizations_bit_exact(case):
    ti = cs.CategoricalGrid(case["ti"].shape[0], case["ti"].shape[1], case["nf"], case["ti"])
    cfg = to_cfg(case["cfg"], case["hd"])
    traces = [cs.SimTrace() for _ in case["seeds"]]
    res = cs.simulate_batch(ti, cfg, case["seeds"], traces)
    for i, r in enumerate(res):
        assert np.array_equal(r.realization.cells, case["real"][i])
        assert r.diagnostics.pre_overwrite_mismatches == case["mism"][i]
        assert r.diagnostics.origin == case["origin"][i]
        assert int(r.diagnostics.column_major) == case["colmajor"][i]
        assert [e.ti_row for e in traces[i].events] == case["ti_row"][i].tolist()
        assert [e.ti_col for e in traces[i].events] == case["ti_col"][i].tolist()


def test_golden_ensemble():
    z = load("ensemble_channel64.npz")
    ti = cs.CategoricalGrid(64, 64, 2, z["ti"])
    cfg = cs.SimConfig(64, 64, 16, 4, 2, 4, n_realizations=6, master_seed=int(z["master"]))
    res = cs.simulate_ensemble(ti, cfg, workers=4)
    assert np.array_equal(np.stack([r.realization.cells for r in res]), z["real"])


def random_case(rng, trial):
    J = int(rng.integers(1, 4))
    b = 1 << J
    T = b * int(rng.integers(2, 7))
    OV = b * int(rng.integers(1, T // b))
    nf = int(rng.integers(1, 6))
    H = b * int(rng.integers(T // b + 1, 128 // b + 1))
    W = b * int(rng.integers(T // b + 1, 128 // b + 1))
    if trial % 2:
        ti = rng.integers(0, nf, (H, W)).astype(np.uint8)
    else:  # blocky TI -> many exact score ties
        ti = np.repeat(np.repeat(rng.integers(0, nf, (H // b, W // b)), b, 0), b, 1).astype(np.uint8)
    sg_h, sg_w = int(rng.integers(T, 96)), int(rng.integers(T, 96))
    d = dict(sg_height=sg_h, sg_width=sg_w, template_size=T, overlap=OV, dwt_level=J,
             candidates=int(rng.integers(1, 12)), scoring=int(rng.integers(0, 2)) if trial % 4 == 0 else 0,
             facies_mode=int(rng.integers(0, 2)), min_cut=int(rng.integers(0, 2)))
    hd = None
    if trial % 3 == 0:
        cells = rng.choice(sg_h * sg_w, size=int(rng.integers(1, 30)), replace=False)
        hd = [(int(c // sg_w), int(c % sg_w), int(rng.integers(0, nf))) for c in cells]
    return ti, nf, d, hd


@pytest.mark.parametrize("block", range(4))
def test_randomized_corpus_vs_oracle(oracle, block):
    rng = np.random.default_rng(1000 + block)
    for trial in range(12):
        ti_a, nf, d, hd = random_case(rng, trial)
        ti = cs.CategoricalGrid(ti_a.shape[0], ti_a.shape[1], nf, ti_a)
        cfg = to_cfg(d, hd)
        seeds = [int(s) for s in rng.integers(0, 2**63, 3)]
        res = cs.simulate_batch(ti, cfg, seeds)
        for s, r in zip(seeds, res):
            o = oracle.simulate_one(ti_a, nf, pyoracle.Cfg(**d), hd, seed=s)
            assert np.array_equal(r.realization.cells, o["realization"]), (block, trial, d)
            assert r.diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]


def test_large_k_and_conditioning(oracle):
    # acceptance.cpp:383-436 shape: K=64 and dense hard data from a reference realization
    ti_a = pyoracle.reference().make_channel_ti(256, 256, 2026) if pyoracle.reference_available() \
        else load("sim_channel128_J3.npz")["ti"]
    ti = cs.CategoricalGrid(ti_a.shape[0], ti_a.shape[1], 2, ti_a)
    d = dict(sg_height=256, sg_width=256, template_size=32, overlap=8, dwt_level=2, candidates=64)
    ref_real = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**d), None, seed=777)["realization"]
    rng = np.random.default_rng(606)
    cells = rng.choice(256 * 256, size=1000, replace=False)
    hd = [(int(c // 256), int(c % 256), int(ref_real[c // 256, c % 256])) for c in cells]
    cfg = to_cfg(d, hd)
    res = cs.simulate_batch(ti, cfg, [11, 12])
    for s, r in zip([11, 12], res):
        o = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**d), hd, seed=s)
        assert np.array_equal(r.realization.cells, o["realization"])
        assert r.diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]
        assert all(r.realization.cells[a, b] == f for a, b, f in hd)


@pytest.mark.parametrize("k", [1, 2, 5])
def test_large_tie_groups_bulk_path(oracle, k):
    """Binary TI at J=3 (BASELINE config 2 regime): the exact screen ties
    hundreds to thousands of windows at the K-th score, which the warp select
    hands to the bulk rescoring kernel.  Bit-exact against the oracle, with
    and without hard data."""
    from paper_2404_00441_b200 import synth
    ti_a = synth.channel_ti(640, 640, 77, scale=6.0)
    ti = cs.CategoricalGrid(640, 640, 2, ti_a)
    d = dict(sg_height=600, sg_width=700, template_size=96, overlap=24, dwt_level=3, candidates=k)
    dev = cs.default_device()
    seeds = [cs.mix64(5, k), cs.mix64(6, k)]
    ref0 = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**d), None, seed=seeds[0])["realization"]
    hd = synth.hard_data_from(ref0, 0.01, 9 + k)
    for cond in (None, [tuple(int(v) for v in row) for row in hd]):
        cfg = to_cfg(d, cond)
        res = cs.simulate_batch(ti, cfg, seeds)
        assert dev.last_timing()["bulk_jobs"] > 0
        for s, r in zip(seeds, res):
            o = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**d), cond, seed=s)
            assert np.array_equal(r.realization.cells, o["realization"]), (k, cond is None)
            assert r.diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]


@pytest.mark.parametrize("nf", [2, 3, 5, 17])
def test_streamed_output_matches_device(nf):
    """Host results are streamed as bit-packed bands (1/2/4 bits per cell for
    F <= 2/4/16, bytes above) and unpacked by host threads (sim.cu
    pack_band_kernel, unpack_band): into pageable and page-locked buffers, with
    hard data (mismatch counts), they must equal the device-resident results."""
    import ctypes as C
    import torch
    from paper_2404_00441_b200 import _abi, synth
    rng = np.random.default_rng(100 + nf)
    ti_a = (synth.channel_ti(152, 172, 5 + nf, scale=4.0).astype(np.int64) * 7 +
            rng.integers(0, 3, (152, 172))) % nf
    ti_a = ti_a.astype(np.uint8)
    ti = cs.CategoricalGrid(152, 172, nf, ti_a)
    d = dict(sg_height=230, sg_width=190, template_size=24, overlap=8, dwt_level=2, candidates=4)
    seeds = [cs.mix64(77, i) for i in range(12)]
    hd = [(int(r), int(c), int(rng.integers(0, nf))) for r, c in zip(rng.integers(0, 230, 40), rng.integers(0, 190, 40))]
    hd = list({(r, c): (r, c, f) for r, c, f in hd}.values())
    cfg = to_cfg(d, hd)
    host = cs.simulate_batch(ti, cfg, seeds)                      # pageable numpy buffer
    dev = cs.default_device()
    lib = _abi.lib()
    h = cs._ti_handle(ti, cfg, None)
    c = cfg.to_c()
    n = len(seeds)
    sa = np.array(seeds, np.uint64)
    hda = np.array(hd, np.int32).reshape(-1, 3)
    diags = (_abi.DiagC * n)()
    d_out = torch.empty(n * 230 * 190, dtype=torch.uint8, device="cuda")
    dev.check(lib.ccw_simulate_device(dev.handle, h.handle, C.byref(c), sa.ctypes.data_as(_abi.U64P), n,
                                      hda.ctypes.data_as(_abi.I32P), hda.shape[0], C.c_void_p(d_out.data_ptr()), diags))
    ref = d_out.cpu().numpy().reshape(n, 230, 190)
    ref_mism = [diags[r].pre_overwrite_mismatches for r in range(n)]
    pinned = torch.empty(n * 230 * 190, dtype=torch.uint8).pin_memory()
    dev.check(lib.ccw_simulate(dev.handle, h.handle, C.byref(c), sa.ctypes.data_as(_abi.U64P), n,
                               hda.ctypes.data_as(_abi.I32P), hda.shape[0],
                               C.cast(C.c_void_p(pinned.data_ptr()), _abi.U8P), diags, None))
    assert dev.last_timing()["d2h_bytes"] < n * 230 * 190 or nf > 16
    got = pinned.numpy().reshape(n, 230, 190)
    for r in range(n):
        assert np.array_equal(host[r].realization.cells, ref[r]), r
        assert np.array_equal(got[r], ref[r]), r
        assert host[r].diagnostics.pre_overwrite_mismatches == ref_mism[r]
        assert diags[r].pre_overwrite_mismatches == ref_mism[r]


@pytest.mark.parametrize("hard", [False, True])
def test_device_schedule_replay(oracle, hard, monkeypatch):
    """The job schedule is drawn on the device (schedule.cu); a draw rejected
    by bounded() sends the realization to a sequential replay.  Forcing that
    path for every realization must give the same realizations."""
    from paper_2404_00441_b200 import synth
    ti_a = synth.channel_ti(160, 160, 41, scale=5.0)
    ti = cs.CategoricalGrid(160, 160, 2, ti_a)
    d = dict(sg_height=150, sg_width=170, template_size=24, overlap=8, dwt_level=2, candidates=3)
    seeds = [cs.mix64(13, i) for i in range(3)]
    hd = None
    if hard:
        ref = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**d), None, seed=seeds[0])["realization"]
        hd = [tuple(int(v) for v in row) for row in synth.hard_data_from(ref, 0.01, 3)]
    with cs.default_device().options(sched_replay=1):
        res = cs.simulate_batch(ti, to_cfg(d, hd), seeds)
    for s, r in zip(seeds, res):
        o = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**d), hd, seed=s)
        assert np.array_equal(r.realization.cells, o["realization"])


@pytest.mark.parametrize("help_min", [2, 8])
def test_shared_rescoring(oracle, help_min, monkeypatch):
    """Equal-score groups of at least help_min windows are rescored in chunks
    claimed by the launch's other CTAs (select.cu hb_rescore); a low
    threshold makes most unconditional picks go that way.  Bit-exact."""
    from paper_2404_00441_b200 import synth
    ti_a = synth.channel_ti(200, 200, 31, scale=5.0)
    ti = cs.CategoricalGrid(200, 200, 2, ti_a)
    d = dict(sg_height=260, sg_width=230, template_size=32, overlap=8, dwt_level=2, candidates=5)
    dev = cs.default_device()
    seeds = [cs.mix64(9, i) for i in range(6)]
    # (uniform-window reduction off: it would shrink the groups below help_min)
    with dev.options(help_min=help_min, uniform=0):
        res = cs.simulate_batch(ti, to_cfg(d, None), seeds)
        assert dev.last_timing()["shared_groups"] > 0
    for s, r in zip(seeds, res):
        o = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**d), None, seed=s)
        assert np.array_equal(r.realization.cells, o["realization"])


@pytest.mark.parametrize("k", [4, 8])
def test_k_above_tile_count_with_ties(oracle, k):
    """Fewer 128-position tiles than K and a blocky TI (every window ties):
    the tile-maximum bound degenerates, the candidate list overflows and the
    placement goes to the bulk path with an all-positions threshold."""
    rng = np.random.default_rng(77 + k)
    ti_a = np.repeat(np.repeat(rng.integers(0, 3, (17, 21)), 4, 0), 4, 1).astype(np.uint8)
    ti = cs.CategoricalGrid(68, 84, 3, ti_a)
    for mode in (0, 1):
        d = dict(sg_height=38, sg_width=94, template_size=12, overlap=4, dwt_level=2, candidates=k,
                 facies_mode=mode)
        cfg = to_cfg(d)
        seeds = [3 + k, 4 + k]
        res = cs.simulate_batch(ti, cfg, seeds)
        for s, r in zip(seeds, res):
            o = oracle.simulate_one(ti_a, 3, pyoracle.Cfg(**d), None, seed=s)
            assert np.array_equal(r.realization.cells, o["realization"]), (k, mode)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("k", [1, 5])
def test_normalized_screen(oracle, mode, k):
    """Normalized scoring through the int8 screen (S = S' + C_job over the
    exact norm map): bit-exact against the oracle on a channel TI and on a
    blocky, tie-heavy TI, with hard data."""
    from paper_2404_00441_b200 import synth
    rng = np.random.default_rng(900 + 10 * mode + k)
    tis = [synth.channel_levee_ti(192, 160, 31),
           np.repeat(np.repeat(rng.integers(0, 3, (48, 40)), 4, 0), 4, 1).astype(np.uint8)]
    dev = cs.default_device()
    for ti_a in tis:
        nf = 3
        ti = cs.CategoricalGrid(ti_a.shape[0], ti_a.shape[1], nf, ti_a)
        d = dict(sg_height=150, sg_width=170, template_size=32, overlap=8, dwt_level=2, candidates=k,
                 scoring=1, facies_mode=mode)
        seeds = [cs.mix64(17, k), cs.mix64(18, k)]
        ref0 = oracle.simulate_one(ti_a, nf, pyoracle.Cfg(**d), None, seed=seeds[0])["realization"]
        cells = rng.choice(150 * 170, size=40, replace=False)
        hd = [(int(c // 170), int(c % 170), int(ref0[c // 170, c % 170])) for c in cells]
        for cond in (None, hd):
            res = cs.simulate_batch(ti, to_cfg(d, cond), seeds)
            assert dev.last_timing()["ccf_variant"] == 2  # screened
            for s_, r in zip(seeds, res):
                o = oracle.simulate_one(ti_a, nf, pyoracle.Cfg(**d), cond, seed=s_)
                assert np.array_equal(r.realization.cells, o["realization"]), (mode, k, cond is None)
                assert r.diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]


@pytest.mark.parametrize("case", ["long_runs", "many_tiles", "k8", "long_runs_hd"])
def test_fast_select_geometries(oracle, case):
    """Fast-select corners against the oracle: mask rows longer than one
    rescoring item (Tc = 32), score rows with more than 512 tiles (the scan
    streams the tile maxima), K = 8 (the register top-K limit), hard data."""
    from paper_2404_00441_b200 import synth
    if case in ("long_runs", "long_runs_hd"):
        ti_a, nf = synth.channel_levee_ti(192, 192, 5), 3
        d = dict(sg_height=160, sg_width=176, template_size=64, overlap=16, dwt_level=1, candidates=3)
    elif case == "many_tiles":
        ti_a, nf = synth.channel_ti(600, 600, 11), 2
        d = dict(sg_height=64, sg_width=72, template_size=16, overlap=4, dwt_level=1, candidates=5)
    else:
        ti_a, nf = synth.channel_levee_ti(256, 256, 6), 3
        d = dict(sg_height=200, sg_width=200, template_size=32, overlap=8, dwt_level=2, candidates=8)
    ti = cs.CategoricalGrid(ti_a.shape[0], ti_a.shape[1], nf, ti_a)
    seeds = [cs.mix64(23, 1), cs.mix64(23, 2)]
    hd = None
    if case == "long_runs_hd":
        ref0 = oracle.simulate_one(ti_a, nf, pyoracle.Cfg(**d), None, seed=seeds[0])["realization"]
        rng = np.random.default_rng(5)
        cells = rng.choice(d["sg_height"] * d["sg_width"], size=120, replace=False)
        hd = [(int(c // d["sg_width"]), int(c % d["sg_width"]),
               int(ref0[c // d["sg_width"], c % d["sg_width"]])) for c in cells]
    res = cs.simulate_batch(ti, to_cfg(d, hd), seeds)
    for s_, r in zip(seeds, res):
        o = oracle.simulate_one(ti_a, nf, pyoracle.Cfg(**d), hd, seed=s_)
        assert np.array_equal(r.realization.cells, o["realization"]), case
        assert r.diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]


def fast_case(rng, trial):
    """Fast-select geometries (raw scoring, K <= 8, no min-cut), mid-size."""
    J = int(rng.integers(1, 4))
    b = 1 << J
    T = b * int(rng.integers(3, 9))
    OV = b * int(rng.integers(1, max(2, (T // b) // 2 + 1)))
    nf = int(rng.integers(2, 5))
    H = b * int(rng.integers(max(T // b + 4, 24), 72))
    W = b * int(rng.integers(max(T // b + 4, 24), 72))
    if trial % 3 == 0:
        ti = np.repeat(np.repeat(rng.integers(0, nf, (H // b, W // b)), b, 0), b, 1).astype(np.uint8)
    else:
        ti = rng.integers(0, nf, (H, W)).astype(np.uint8)
        ti = np.where(rng.random((H, W)) < 0.7, np.roll(ti, 1, axis=1), ti).astype(np.uint8)
    sg_h, sg_w = int(rng.integers(T + 8, 3 * T + 40)), int(rng.integers(T + 8, 3 * T + 40))
    d = dict(sg_height=sg_h, sg_width=sg_w, template_size=T, overlap=OV, dwt_level=J,
             candidates=int(rng.integers(1, 9)), facies_mode=int(rng.integers(0, 2)))
    hd = None
    if trial % 2:
        cells = rng.choice(sg_h * sg_w, size=int(rng.integers(5, 80)), replace=False)
        hd = [(int(c // sg_w), int(c % sg_w), int(rng.integers(0, nf))) for c in cells]
    return ti, nf, d, hd


@pytest.mark.parametrize("block", range(3))
def test_fast_path_corpus_vs_oracle(oracle, block):
    """Randomized fast-select configurations (equal-score ranking, tile
    queueing, bulk deferral, streamed result bands) against the oracle."""
    rng = np.random.default_rng(5000 + block)
    for trial in range(20):
        ti_a, nf, d, hd = fast_case(rng, trial)
        if nf > 2 and d["dwt_level"] == 3 and d["facies_mode"] == 1:
            d["facies_mode"] = 0  # raw-code block sums above 127 leave the int8 screen (covered elsewhere)
        ti = cs.CategoricalGrid(ti_a.shape[0], ti_a.shape[1], nf, ti_a)
        seeds = [int(s) for s in rng.integers(0, 2**63, 4)]
        res = cs.simulate_batch(ti, to_cfg(d, hd), seeds)
        for s_, r in zip(seeds, res):
            o = oracle.simulate_one(ti_a, nf, pyoracle.Cfg(**d), hd, seed=s_)
            assert np.array_equal(r.realization.cells, o["realization"]), (block, trial, d)
            assert r.diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]


@pytest.mark.parametrize("F", [6, 8, 12])
def test_many_facies_and_odd_templates(oracle, F):
    """More facies (wider int8 screen K, raw-code block sums beyond int8 fall
    back to the fp32 screen) and template sizes that are not multiples of 4
    (the byte paste / map paths)."""
    rng = np.random.default_rng(77 + F)
    for J, T, OV in ((1, 14, 4), (1, 22, 6), (2, 20, 8)):
        b = 1 << J
        H, W = b * 60, b * 52
        ti_a = np.repeat(np.repeat(rng.integers(0, F, (H // b, W // b)), b, 0), b, 1).astype(np.uint8)
        ti_a = np.where(rng.random((H, W)) < 0.3, rng.integers(0, F, (H, W)), ti_a).astype(np.uint8)
        ti = cs.CategoricalGrid(H, W, F, ti_a)
        for mode in (0, 1):
            d = dict(sg_height=90, sg_width=77, template_size=T, overlap=OV, dwt_level=J,
                     candidates=int(rng.integers(1, 9)), facies_mode=mode)
            seeds = [int(s) for s in rng.integers(0, 2**63, 3)]
            res = cs.simulate_batch(ti, to_cfg(d), seeds)
            for s_, r in zip(seeds, res):
                o = oracle.simulate_one(ti_a, F, pyoracle.Cfg(**d), None, seed=s_)
                assert np.array_equal(r.realization.cells, o["realization"]), (F, J, T, OV, mode)


def test_provenance_and_replay():
    # test_simulator.cpp:434-460, acceptance.cpp:349-381
    z = load("sim_channel64_base.npz")
    ti = cs.CategoricalGrid(64, 64, 2, z["ti"])
    cfg = cs.SimConfig(52, 64, 16, 4, 2, 6)
    tr = cs.SimTrace()
    res = cs.simulate_one(ti, cfg, 2024, tr)
    replay = np.zeros((res.diagnostics.work_height, res.diagnostics.work_width), np.uint8)
    for ev in tr.events:
        assert ev.ti_row % 4 == 0 and ev.ti_col % 4 == 0
        assert np.array_equal(ev.pasted.cells, z["ti"][ev.ti_row:ev.ti_row + 16, ev.ti_col:ev.ti_col + 16])
        replay[ev.placement.top:ev.placement.top + 16, ev.placement.left:ev.placement.left + 16] = ev.pasted.cells
    assert np.array_equal(replay[:52, :64], res.realization.cells)


def test_constant_ti_and_determinism():
    # test_simulator.cpp:401-432
    ti = cs.CategoricalGrid(32, 32, 2, fill=1)
    cfg = cs.SimConfig(48, 48, 16, 4, 2, 4)
    assert (cs.simulate_one(ti, cfg, 999).realization.cells == 1).all()
    z = load("sim_channel64_base.npz")
    ti = cs.CategoricalGrid(64, 64, 2, z["ti"])
    cfg = cs.SimConfig(64, 64, 16, 4, 2, 4)
    a = cs.simulate_one(ti, cfg, 31337)
    b = cs.simulate_one(ti, cfg, 31337)
    c = cs.simulate_one(ti, cfg, 31338)
    assert a.realization == b.realization and a.realization != c.realization
    assert a.diagnostics.seed == 31337 and a.diagnostics.placement_count > 0


def test_batch_equals_single():
    z = load("sim_channel64_base.npz")
    ti = cs.CategoricalGrid(64, 64, 2, z["ti"])
    cfg = cs.SimConfig(64, 64, 16, 4, 2, 4, min_cut=True)
    seeds = [5, 6, 7, 8, 9]
    batch = cs.simulate_batch(ti, cfg, seeds)
    for s, r in zip(seeds, batch):
        assert r.realization == cs.simulate_one(ti, cfg, s).realization


@pytest.mark.slow
def test_config1_full_size_bit_exact(oracle):
    """BASELINE config 1 geometry (TI 500^2, 3 facies, SG 1000^2, T64, OV16,
    J2, K5): two realizations bit-identical to the oracle."""
    from paper_2404_00441_b200 import synth
    ti_a = synth.config1_ti()
    ti = cs.CategoricalGrid(500, 500, 3, ti_a)
    cfg = cs.SimConfig(1000, 1000, 64, 16, 2, 5)
    seeds = [cs.mix64(0, 1), cs.mix64(0, 2)]
    res = cs.simulate_batch(ti, cfg, seeds)
    for s, r in zip(seeds, res):
        o = oracle.simulate_one(ti_a, 3, pyoracle.Cfg(**cfg_dict(cfg)), None, seed=s)
        assert np.array_equal(r.realization.cells, o["realization"])


@pytest.mark.slow
def test_config2_full_size_bit_exact(oracle):
    """BASELINE config 2 geometry (TI 2000^2, SG 4000^2, T96, OV24, J3, K1,
    1% hard data): one realization bit-identical to the oracle."""
    from paper_2404_00441_b200 import synth
    ti_a = synth.config2_ti()
    hd = synth.config2_hard_data(ti_a)
    ti = cs.CategoricalGrid(2000, 2000, 2, ti_a)
    cfg = cs.SimConfig(4000, 4000, 96, 24, 3, 1)
    cfg.hard_data = hd
    seed = cs.mix64(0, 1)
    r = cs.simulate_one(ti, cfg, seed)
    o = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**cfg_dict(cfg)), hd, seed=seed)
    assert np.array_equal(r.realization.cells, o["realization"])
    assert r.diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]
    assert (r.realization.cells[hd[:, 0], hd[:, 1]] == hd[:, 2]).all()


def cfg_dict(cfg):
    c = cfg.to_c()
    return dict(sg_height=c.sg_height, sg_width=c.sg_width, template_size=c.template_size,
                overlap=c.overlap, dwt_level=c.dwt_level, candidates=c.candidates,
                scoring=c.scoring, facies_mode=c.facies_mode, min_cut=bool(c.min_cut))


def test_uniform_window_groups(oracle):
    """Large background regions: placements whose overlap is all background
    tie hundreds of pure-background windows at the top score.  The fast select
    rescores one representative per uniform facies (their fp64 scores are
    bit-identical) -- the realizations must still equal the oracle's."""
    rng = np.random.default_rng(31)
    ti_a = np.zeros((256, 256), np.uint8)
    for _ in range(40):  # lenses of facies 1-2 on a background of facies 0
        r, c = rng.integers(0, 240, 2)
        h, w = rng.integers(4, 24, 2)
        ti_a[r:r + h, c:c + w] = rng.integers(1, 3)
    ti = cs.CategoricalGrid(256, 256, 3, ti_a)
    for k, mode in ((5, "indicator"), (3, "raw_codes"), (8, "indicator")):
        d = dict(sg_height=200, sg_width=180, template_size=32, overlap=8, dwt_level=2, candidates=k,
                 facies_mode=1 if mode == "raw_codes" else 0)
        cfg = to_cfg(d)
        seeds = [int(s) for s in rng.integers(0, 2**63, 3)]
        for s, r in zip(seeds, cs.simulate_batch(ti, cfg, seeds)):
            o = oracle.simulate_one(ti_a, 3, pyoracle.Cfg(**d), None, seed=s)
            assert np.array_equal(r.realization.cells, o["realization"]), (k, mode, s)
