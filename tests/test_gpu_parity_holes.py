"""Parity of the CUDA path against the COMPILED REFERENCE (oracle/_ref: the
unmodified reference headers, simulator.hpp:418-566) at the BASELINE
configurations' full sizes, plus the history-dependent launch-plan paths of
the library (the per-context bulk_off memory, sim.cu run_simulation) and the
production options forced off.  Every comparison is exact equality."""
import numpy as np
import pytest

import pyoracle
from paper_2404_00441_b200 import ccwsim as cs
from paper_2404_00441_b200 import synth

pytestmark = pytest.mark.gpu


def cfg_dict(cfg):
    c = cfg.to_c()
    return dict(sg_height=c.sg_height, sg_width=c.sg_width, template_size=c.template_size,
                overlap=c.overlap, dwt_level=c.dwt_level, candidates=c.candidates,
                scoring=c.scoring, facies_mode=c.facies_mode, min_cut=bool(c.min_cut))


def config0_adjusted():
    """Config 0': the 250^2 generated TI cropped to its
    top-left 248^2 (250 is not divisible by 2^J = 4, simulator.hpp:78-81),
    OV 12 instead of 10 (simulator.hpp:58-60)."""
    ti_a = np.ascontiguousarray(synth.config0_ti()[:248, :248])
    cfg = cs.SimConfig(250, 250, 40, 12, 2, 1)
    return ti_a, cfg


def test_config0_adjusted_vs_reference(reference):
    """Config 0' (TI 248^2 binary channels, SG 250^2, T40, OV12, J2, K1):
    six realizations bit-identical to the compiled reference, with and
    without hard data, and through simulate_ensemble (seeds mix64(master, r+1))."""
    ti_a, cfg = config0_adjusted()
    ti = cs.CategoricalGrid(248, 248, 2, ti_a)
    seeds = [cs.mix64(20240441, r + 1) for r in range(6)]
    res = cs.simulate_batch(ti, cfg, seeds)
    for s, r in zip(seeds, res):
        o = reference.simulate_one(ti_a, 2, pyoracle.Cfg(**cfg_dict(cfg)), None, seed=s)
        assert np.array_equal(r.realization.cells, o["realization"]), s
        assert r.diagnostics.origin == o["diagnostics"]["origin"]
    # conditional: 1 % hard data drawn from a reference realization
    hd = synth.hard_data_from(res[0].realization.cells, 0.01, 5)
    cfg.hard_data = hd
    for s in seeds[:3]:
        r = cs.simulate_one(ti, cfg, s)
        o = reference.simulate_one(ti_a, 2, pyoracle.Cfg(**cfg_dict(cfg)), hd, seed=s)
        assert np.array_equal(r.realization.cells, o["realization"]), s
        assert r.diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]
    # simulate_ensemble: worker-count invariance (acceptance.cpp:665-702)
    cfg.hard_data = cs.HardDataSet()
    cfg.n_realizations = 4
    cfg.master_seed = 77
    ens = cs.simulate_ensemble(ti, cfg, workers=8)
    ref, _ = reference.simulate_ensemble(ti_a, 2, pyoracle.Cfg(**cfg_dict(cfg), n_realizations=4,
                                                               master_seed=77), None, workers=1)
    assert len(ens) == 4
    for a, b in zip(ens, ref):
        assert np.array_equal(a.realization.cells, b)


@pytest.mark.slow
def test_config1_full_size_vs_reference(reference):
    """BASELINE config 1 (TI 500^2 3 facies, SG 1000^2, T64 OV16 J2 K5): the
    first four of the benchmarked realizations (bench.py: master 20240441,
    seeds mix64(master, r+1)) bit-identical to the compiled reference."""
    ti_a = synth.config1_ti()
    ti = cs.CategoricalGrid(500, 500, 3, ti_a)
    cfg = cs.SimConfig(1000, 1000, 64, 16, 2, 5)
    seeds = [cs.mix64(20240441, r + 1) for r in range(100)]
    res = cs.simulate_batch(ti, cfg, seeds)  # the bench's whole 100-realization call
    for r in range(4):
        o = reference.simulate_one(ti_a, 3, pyoracle.Cfg(**cfg_dict(cfg)), None, seed=seeds[r])
        assert np.array_equal(res[r].realization.cells, o["realization"]), r


@pytest.mark.slow
def test_config2_full_size_vs_reference(reference):
    """BASELINE config 2 (TI 2000^2, SG 4000^2, T96 OV24 J3 K1, 1 % hard data):
    one realization of an 8-realization call bit-identical to the compiled
    reference, hard-data diagnostics included."""
    ti_a = synth.config2_ti()
    hd = synth.config2_hard_data(ti_a)
    ti = cs.CategoricalGrid(2000, 2000, 2, ti_a)
    cfg = cs.SimConfig(4000, 4000, 96, 24, 3, 1)
    cfg.hard_data = hd
    seeds = [cs.mix64(20240441, r + 1) for r in range(8)]
    res = cs.simulate_batch(ti, cfg, seeds)
    o = reference.simulate_one(ti_a, 2, pyoracle.Cfg(**cfg_dict(cfg)), hd, seed=seeds[3])
    assert np.array_equal(res[3].realization.cells, o["realization"])
    assert res[3].diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]


def tie_heavy_case():
    ti_a = synth.channel_ti(640, 640, 77, scale=6.0)
    return ti_a, dict(template_size=96, overlap=24, dwt_level=3, candidates=1)


def test_learned_bulk_off_then_overflow(oracle):
    """sim.cu memoizes, per (TI content, Tc, OVc, K, T) on the context, that a
    call deferred no tie group; the next call then skips the bulk kernel.  A
    later call that overflows the candidate list on the same TI and shape
    must take the in-kernel fallback (select.cu) and stay exact; the call
    after it brings the bulk kernel back."""
    ti_a, geo = tie_heavy_case()
    ti = cs.CategoricalGrid(640, 640, 2, ti_a)
    dev = cs.Device(0)  # a fresh context: no plan memory
    try:
        # call 1: one placement (SG = T), nothing screened -> nothing deferred
        small = dict(sg_height=96, sg_width=96, **geo)
        cs.simulate_batch(ti, to_cfg(small), [3], device=dev)
        assert dev.last_timing()["bulk_jobs"] == 0
        # call 2: the tie-heavy shape, bulk kernel switched off by the memory
        big = dict(sg_height=600, sg_width=700, **geo)
        seeds = [cs.mix64(5, 1), cs.mix64(6, 1)]
        res = cs.simulate_batch(ti, to_cfg(big), seeds, device=dev)
        t2 = dev.last_timing()
        assert t2["bulk_jobs"] == 0 and t2["list_overflows"] > 0
        for s, r in zip(seeds, res):
            o = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**big), None, seed=s)
            assert np.array_equal(r.realization.cells, o["realization"]), s
        # call 3: the overflow re-enabled the bulk kernel
        res3 = cs.simulate_batch(ti, to_cfg(big), seeds, device=dev)
        assert dev.last_timing()["bulk_jobs"] > 0
        for a, b in zip(res, res3):
            assert a.realization == b.realization
    finally:
        dev.close()


@pytest.mark.parametrize("opts", [dict(bulk=0), dict(uniform=0, s16=0), dict(groups=1),
                                  dict(groups=3, stream_out=0), dict(pack=0, stream_bands=2)])
def test_options_forced_paths(oracle, opts):
    """The production options switched off one by one (include/ccwgpu.h
    ccw_ctx_set_option): no bulk kernel (every overflow takes the in-kernel
    fallback), no uniform-class reduction / int32 score rows, other group
    counts, no streamed or no packed host bands.  Bit-exact."""
    ti_a, geo = tie_heavy_case()
    ti = cs.CategoricalGrid(640, 640, 2, ti_a)
    d = dict(sg_height=500, sg_width=520, **geo)
    seeds = [cs.mix64(11, 1), cs.mix64(11, 2), cs.mix64(11, 3)]
    dev = cs.default_device()
    with dev.options(**opts):
        res = cs.simulate_batch(ti, to_cfg(d), seeds)
        if opts.get("bulk") == 0:
            assert dev.last_timing()["bulk_jobs"] == 0
    for s, r in zip(seeds, res):
        o = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**d), None, seed=s)
        assert np.array_equal(r.realization.cells, o["realization"]), (opts, s)


def test_option_names_validated():
    dev = cs.default_device()
    with pytest.raises(cs.ConfigError):
        dev.set_option("no_such_option", 1)
    with pytest.raises(cs.ConfigError):
        dev.set_option("groups", -1)


def test_context_create_destroy_frees_device_memory():
    """ccw_ctx_destroy releases every buffer (DevBuf / HostBuf are RAII): a
    create / simulate / destroy cycle does not grow the device footprint."""
    import torch
    ti_a, cfg = config0_adjusted()
    ti = cs.CategoricalGrid(248, 248, 2, ti_a)

    def cycle():
        dev = cs.Device(0)
        try:
            cs.simulate_batch(ti, cfg, [1, 2, 3, 4], device=dev)
        finally:
            dev.close()

    cycle()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(4):
        cycle()
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 8 << 20, (free0, free1)


def to_cfg(d, hd=None):
    cfg = cs.SimConfig(sg_height=d["sg_height"], sg_width=d["sg_width"],
                       template_size=d["template_size"], overlap=d["overlap"],
                       dwt_level=d["dwt_level"], candidates=d["candidates"])
    if hd:
        cfg.hard_data = cs.HardDataSet([cs.HardDatum(*p) for p in hd])
    return cfg


@pytest.mark.parametrize("cs_", [4, 8, 16])
def test_wave_kernel_paths(oracle, cs_):
    """The fused wave kernel (csrc/wave.cu, option `wave`): OR prep, the
    implicit-im2col tcgen05 screen, the epilogue's top-K' lists, fp64 tie
    ranking, conditional and unconditional picks and the in-kernel tie-storm
    fallback, for every cluster size.  Bit-exact against the restatement."""
    dev = cs.Device(0)  # a fresh context: no tie-storm memory
    try:
        with dev.options(wave=1, wave_cs=cs_):
            # tie-heavy binary channels, J3, K1: list drops and the generic fallback
            ti_a, geo = tie_heavy_case()
            ti = cs.CategoricalGrid(640, 640, 2, ti_a)
            d = dict(sg_height=500, sg_width=520, **geo)
            seeds = [cs.mix64(13, 1), cs.mix64(13, 2)]
            res = cs.simulate_batch(ti, to_cfg(d), seeds, device=dev)
            assert dev.last_timing()["ccf_variant"] == 5  # the wave kernel ran
            for s, r in zip(seeds, res):
                o = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**d), None, seed=s)
                assert np.array_equal(r.realization.cells, o["realization"]), ("ties", cs_, s)
            # three facies, K5 unconditional picks (config-1 shape, smaller grid)
            ti3 = synth.config1_ti()
            g3 = cs.CategoricalGrid(500, 500, 3, ti3)
            d3 = dict(sg_height=400, sg_width=352, template_size=64, overlap=16, dwt_level=2, candidates=5)
            seeds3 = [cs.mix64(17, r + 1) for r in range(3)]
            res3 = cs.simulate_batch(g3, to_cfg(d3), seeds3, device=dev)
            assert dev.last_timing()["ccf_variant"] == 5
            for s, r in zip(seeds3, res3):
                o = oracle.simulate_one(ti3, 3, pyoracle.Cfg(**d3), None, seed=s)
                assert np.array_equal(r.realization.cells, o["realization"]), ("k5", cs_, s)
            # conditional picks: config 0' with 1 % hard data
            ti0, cfg0 = config0_adjusted()
            g0 = cs.CategoricalGrid(248, 248, 2, ti0)
            base = cs.simulate_one(g0, cfg0, 5, device=dev).realization.cells
            hd = synth.hard_data_from(base, 0.01, 5)
            cfg0.hard_data = hd
            for s in [cs.mix64(19, 1), cs.mix64(19, 2)]:
                r = cs.simulate_one(g0, cfg0, s, device=dev)
                o = oracle.simulate_one(ti0, 2, pyoracle.Cfg(**cfg_dict(cfg0)), hd, seed=s)
                assert np.array_equal(r.realization.cells, o["realization"]), ("cond", cs_, s)
                assert r.diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]
    finally:
        dev.close()


def test_flagprep_off_equals_on(oracle):
    """The dependency-flag OR prep (option flagprep, default on: a prep CTA
    waits only on the two previous-wave placements it reads) and the whole-
    launch wait give the same realizations, equal to the restatement."""
    ti_a = synth.config1_ti()
    ti = cs.CategoricalGrid(500, 500, 3, ti_a)
    d = dict(sg_height=520, sg_width=616, template_size=64, overlap=16, dwt_level=2, candidates=5)
    seeds = [cs.mix64(23, r + 1) for r in range(6)]
    dev = cs.default_device()
    cs.simulate_batch(ti, to_cfg(d), seeds[:1])  # (the bulk-off plan memory: flag prep needs it)
    res_on = cs.simulate_batch(ti, to_cfg(d), seeds)
    with dev.options(flagprep=0):
        res_off = cs.simulate_batch(ti, to_cfg(d), seeds)
    for s, a, b in zip(seeds, res_on, res_off):
        assert np.array_equal(a.realization.cells, b.realization.cells), s
    for s, r in zip(seeds[:2], res_on[:2]):
        o = oracle.simulate_one(ti_a, 3, pyoracle.Cfg(**d), None, seed=s)
        assert np.array_equal(r.realization.cells, o["realization"]), s


def test_ti_upload_code_range_checked_on_device():
    """Large training images go through the staged upload and the device
    code-range check (grid.hpp:36-40): the first bad cell and its code are
    reported exactly as the host check did."""
    import ctypes as C
    from paper_2404_00441_b200 import _abi
    dev = cs.default_device()
    lib = _abi.lib()
    a = np.zeros((1500, 1500), np.uint8)
    a[700, 1234] = 7
    a[900, 3] = 5
    h = C.c_void_p()
    with pytest.raises(cs.BoundsError, match=r"cell 1051234 holds code 7 outside \[0, 3\)"):
        dev.check(lib.ccw_ti_create(dev.handle, a.ctypes.data_as(_abi.U8P), 1500, 1500, 3, 2, 0, C.byref(h)))
    b = np.zeros((64, 96, 200), np.uint8)
    b[10, 20, 30] = 9
    with pytest.raises(cs.BoundsError, match=r"cell 196030 holds code 9 outside \[0, 4\)"):
        dev.check(lib.ccw_ti3d_create(dev.handle, b.ctypes.data_as(_abi.U8P), 64, 96, 200, 4, 2, C.byref(h)))
    # a valid large TI through the same path simulates like the small-TI path
    a[:] = (np.arange(1500 * 1500).reshape(1500, 1500) // 37 % 3).astype(np.uint8)
    dev.check(lib.ccw_ti_create(dev.handle, a.ctypes.data_as(_abi.U8P), 1500, 1500, 3, 2, 0, C.byref(h)))
    lib.ccw_ti_destroy(h)


def test_async_device_calls_equal_sync():
    """ccw_simulate_device_async: back-to-back calls (each one's host planning
    overlapping the previous one's device work, alternating staging halves and
    result slots) produce the synchronous call's realizations; the timing and
    the plan memory are settled by ccw_ctx_synchronize."""
    import ctypes as C
    import torch
    from paper_2404_00441_b200 import _abi
    ti_a = synth.config1_ti()
    grid = cs.CategoricalGrid(500, 500, 3, ti_a)
    cfg = cs.SimConfig(440, 392, 64, 16, 2, 5, n_realizations=12, master_seed=31)
    dev = cs.Device(0)
    lib = _abi.lib()
    try:
        tih = cs.TrainingImage(grid, 2, "indicator", dev)
        c = cfg.to_c()
        n = 12
        sg = 440 * 392
        outs = [torch.zeros(n * sg, dtype=torch.uint8, device="cuda:0") for _ in range(5)]
        ref = torch.zeros(n * sg, dtype=torch.uint8, device="cuda:0")
        seed_sets = [np.array([cs.mix64(31 + k % 2, r + 1) for r in range(n)], np.uint64) for k in range(5)]
        diags = (_abi.DiagC * n)()
        for k in range(5):
            dev.check(lib.ccw_simulate_device_async(dev.handle, tih.handle, C.byref(c),
                                                    seed_sets[k].ctypes.data_as(_abi.U64P), n, None, 0,
                                                    C.c_void_p(outs[k].data_ptr())))
        dev.synchronize()
        t = dev.last_timing()
        assert t["total_ms"] > 0 and t["jobs"] > 0
        for k in range(5):
            dev.check(lib.ccw_simulate_device(dev.handle, tih.handle, C.byref(c),
                                              seed_sets[k].ctypes.data_as(_abi.U64P), n, None, 0,
                                              C.c_void_p(ref.data_ptr()), diags))
            torch.cuda.synchronize()
            assert torch.equal(outs[k], ref), k
    finally:
        dev.close()
