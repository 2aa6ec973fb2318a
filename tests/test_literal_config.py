"""Literal-config extension: BASELINE
config 0 as stated (TI 250^2, OV 10 at J 2) and any overlap / TI extent that
2^J does not divide.  The reference rejects these (simulator.hpp:58-60,
78-81); with ``any_support`` the coarse mask keeps every block the fine
overlap touches (replacing coarse_mask_from_fine, simulator.hpp:256-272) and
the TI is used at its top-left whole-block crop.  Oracle: the C restatement
with the flag (oracle/ccw_oracle.h), pinned to the reference where the flag
is a no-op.  GPU tests are marked gpu; the oracle pins run on CPU."""
import numpy as np
import pytest

import pyoracle
from paper_2404_00441_b200 import synth


def cfgd(**kw):
    d = dict(sg_height=64, sg_width=64, template_size=16, overlap=4, dwt_level=2, candidates=3)
    d.update(kw)
    return d


# ----------------------------------------------------------- oracle pins --

def test_flag_is_a_noop_on_aligned_configs(oracle, reference):
    """OV and TI divisible by 2^J: the any-support mask equals the
    reference's block mask, so the flagged restatement equals the reference."""
    rng = np.random.default_rng(4)
    ti = rng.integers(0, 3, (64, 72)).astype(np.uint8)
    for d in (cfgd(), cfgd(min_cut=True, candidates=5), cfgd(scoring=1, facies_mode=1, overlap=8)):
        for s in (1, 2, 3):
            a = oracle.simulate_one(ti, 3, pyoracle.Cfg(**d, any_support=True), None, seed=s)
            b = reference.simulate_one(ti, 3, pyoracle.Cfg(**d), None, seed=s)
            assert np.array_equal(a["realization"], b["realization"]), (d, s)


def test_reference_rejects_the_flag(reference):
    with pytest.raises(pyoracle.OracleError, match="any_support"):
        reference.simulate_one(np.zeros((32, 32), np.uint8), 2, pyoracle.Cfg(any_support=True), None, seed=1)


def test_unflagged_literal_config0_rejected(oracle):
    ti = synth.config0_ti()
    with pytest.raises(pyoracle.OracleError, match="overlap: 10 not divisible"):
        oracle.simulate_one(ti, 2, pyoracle.Cfg(sg_height=250, sg_width=250, template_size=40, overlap=10,
                                                dwt_level=2, candidates=1), None, seed=1)


def test_ti_crop_equivalence(oracle):
    """A TI 2^J does not divide gives the same realizations as its top-left
    whole-block crop (no block-aligned window reaches the trailing cells)."""
    rng = np.random.default_rng(8)
    ti = rng.integers(0, 2, (66, 71)).astype(np.uint8)
    d = cfgd(overlap=6, any_support=True)
    for s in (4, 5):
        a = oracle.simulate_one(ti, 2, pyoracle.Cfg(**d), None, seed=s)
        b = oracle.simulate_one(np.ascontiguousarray(ti[:64, :68]), 2, pyoracle.Cfg(**d), None, seed=s)
        assert np.array_equal(a["realization"], b["realization"])


# --------------------------------------------------------------- GPU --------

def _gpu_cfg(d, hd=None):
    from paper_2404_00441_b200 import ccwsim as cs
    cfg = cs.SimConfig(sg_height=d["sg_height"], sg_width=d["sg_width"], template_size=d["template_size"],
                       overlap=d["overlap"], dwt_level=d["dwt_level"], candidates=d["candidates"],
                       scoring={0: "raw", 1: "normalized"}[d.get("scoring", 0)],
                       facies_mode={0: "indicator", 1: "raw_codes"}[d.get("facies_mode", 0)],
                       min_cut=bool(d.get("min_cut", False)), any_support=bool(d.get("any_support", False)))
    if hd is not None:
        cfg.hard_data = hd
    return cfg


@pytest.mark.gpu
def test_config0_literal(oracle):
    """BASELINE config 0 as stated: TI 250^2 binary channels, SG 250^2, T40,
    OV10, J2, K1 -- bit-identical to the flagged restatement, with and
    without 1 % hard data."""
    from paper_2404_00441_b200 import ccwsim as cs
    ti_a = synth.config0_ti()
    ti = cs.CategoricalGrid(250, 250, 2, ti_a)
    d = dict(sg_height=250, sg_width=250, template_size=40, overlap=10, dwt_level=2, candidates=1,
             any_support=True)
    seeds = [cs.mix64(20240441, r + 1) for r in range(6)]
    res = cs.simulate_batch(ti, _gpu_cfg(d), seeds)
    for s, r in zip(seeds, res):
        o = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**d), None, seed=s)
        assert np.array_equal(r.realization.cells, o["realization"]), s
    hd = synth.hard_data_from(res[0].realization.cells, 0.01, 3)
    for s in seeds[:3]:
        r = cs.simulate_one(ti, _gpu_cfg(d, hd), s)
        o = oracle.simulate_one(ti_a, 2, pyoracle.Cfg(**d), hd, seed=s)
        assert np.array_equal(r.realization.cells, o["realization"]), s
        assert r.diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]


@pytest.mark.gpu
@pytest.mark.parametrize("block", range(3))
def test_literal_corpus(oracle, block):
    """Random overlaps and TI extents 2^J does not divide, K 1-8, both facies
    modes, raw / normalized scoring, min-cut on a third of the cases."""
    from paper_2404_00441_b200 import ccwsim as cs
    rng = np.random.default_rng(500 + block)
    for trial in range(8):
        J = int(rng.integers(1, 4))
        B = 1 << J
        T = B * int(rng.integers(2, 6))
        OV = int(rng.integers(1, T))
        nf = int(rng.integers(2, 5))
        H = T + int(rng.integers(B, 80))
        W = T + int(rng.integers(B, 80))
        ti_a = np.repeat(np.repeat(rng.integers(0, nf, (H // 2 + 1, W // 2 + 1)), 2, 0), 2, 1)[:H, :W]
        ti_a = np.ascontiguousarray(ti_a).astype(np.uint8)
        d = dict(sg_height=int(rng.integers(T, 3 * T)), sg_width=int(rng.integers(T, 3 * T)), template_size=T,
                 overlap=OV, dwt_level=J, candidates=int(rng.integers(1, 9)), any_support=True,
                 facies_mode=int(trial % 2), scoring=int(trial % 4 == 3), min_cut=bool(trial % 3 == 2))
        ti = cs.CategoricalGrid(H, W, nf, ti_a)
        seeds = [int(s) for s in rng.integers(0, 2**63, 3)]
        hd = None
        if trial % 2:
            ref0 = oracle.simulate_one(ti_a, nf, pyoracle.Cfg(**d), None, seed=seeds[0])["realization"]
            hd = synth.hard_data_from(ref0, 0.02, trial)
        res = cs.simulate_batch(ti, _gpu_cfg(d, hd), seeds)
        for s, r in zip(seeds, res):
            o = oracle.simulate_one(ti_a, nf, pyoracle.Cfg(**d), hd, seed=s)
            assert np.array_equal(r.realization.cells, o["realization"]), (block, trial, d)
