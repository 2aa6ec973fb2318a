"""Candidate-position sharding on the GPU: a single realization
whose placements' TI window positions are split into S shards, each screening
and ranking its range, with the shards' top-K lists exchanged and merged per
placement wave.  One GPU is available, so the S shards run as virtual shards
of one rank (exchange through device memory) and, separately, through a real
one-rank NCCL communicator (ncclAllGather in place).  Every result must be
bit-identical to the oracle -- the sharded path is the same computation with
a different decomposition of the window positions."""
import numpy as np
import pytest

import pyoracle
from paper_2404_00441_b200 import ccwsim as cs
from test_gpu_sim_parity import random_case, to_cfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    # a context of its own (released at exit after its TIs, ccwsim._shutdown);
    # sharding is switched off again so no other test sees it
    d = cs.Device(0)
    yield d
    d.set_position_shards(1, 0, None, 1)


def _check(oracle, dev, ti_a, nf, d, hd, seeds, traces=False):
    ti = cs.CategoricalGrid(ti_a.shape[0], ti_a.shape[1], nf, ti_a)
    cfg = to_cfg(d, hd)
    tr = [cs.SimTrace() for _ in seeds] if traces else None
    res = cs.simulate_batch(ti, cfg, seeds, tr, dev)
    for i, (s, r) in enumerate(zip(seeds, res)):
        o = oracle.simulate_one(ti_a, nf, pyoracle.Cfg(**d), hd, seed=s, trace=traces)
        assert np.array_equal(r.realization.cells, o["realization"]), (d, s)
        assert r.diagnostics.pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]
        if traces:
            assert [e.ti_row for e in tr[i].events] == list(o["trace"]["ti_row"])
            assert [e.ti_col for e in tr[i].events] == list(o["trace"]["ti_col"])


@pytest.mark.parametrize("shards", [2, 3, 7])
def test_virtual_shards_corpus_vs_oracle(oracle, dev, shards):
    """Randomized corpus (J 1-3, F 1-5, K 1-11, both scorings and facies
    modes, min-cut, hard data, tie-heavy blocky TIs) with S virtual shards."""
    dev.set_position_shards(1, 0, None, shards)
    rng = np.random.default_rng(4200 + shards)
    for trial in range(10):
        ti_a, nf, d, hd = random_case(rng, trial)
        out_h = (ti_a.shape[0] >> d["dwt_level"]) - (d["template_size"] >> d["dwt_level"]) + 1
        out_w = (ti_a.shape[1] >> d["dwt_level"]) - (d["template_size"] >> d["dwt_level"]) + 1
        if out_h * out_w < shards:
            continue
        seeds = [int(s) for s in rng.integers(0, 2**63, 2)]
        _check(oracle, dev, ti_a, nf, d, hd, seeds)


def test_shards_with_ties_and_traces(oracle, dev):
    """Binary blocky TI at J=3: thousands of exact screen ties cross shard
    boundaries; the merged ranking must still be the reference's."""
    dev.set_position_shards(1, 0, None, 4)
    rng = np.random.default_rng(77)
    ti_a = np.repeat(np.repeat(rng.integers(0, 2, (16, 16)), 8, 0), 8, 1).astype(np.uint8)
    for k in (1, 2, 5):
        d = dict(sg_height=120, sg_width=104, template_size=32, overlap=8, dwt_level=3, candidates=k)
        _check(oracle, dev, ti_a, 2, d, None, [3, 2**40 + 9], traces=True)


def test_more_shards_than_k_and_short_lists(oracle, dev):
    """Shards smaller than K return short lists (empty slots in the exchange)."""
    rng = np.random.default_rng(5)
    ti_a = rng.integers(0, 3, (40, 40)).astype(np.uint8)
    d = dict(sg_height=48, sg_width=48, template_size=16, overlap=4, dwt_level=2, candidates=11)
    npos = (10 - 4 + 1) ** 2  # 49 windows
    dev.set_position_shards(1, 0, None, 12)  # 4-5 windows per shard < K
    _check(oracle, dev, ti_a, 3, d, None, [1, 2, 3])
    dev.set_position_shards(1, 0, None, npos)  # one window per shard
    _check(oracle, dev, ti_a, 3, d, None, [4])
    dev.set_position_shards(1, 0, None, 1)
    _check(oracle, dev, ti_a, 3, d, None, [4])


def test_too_many_shards_rejected(dev):
    ti_a = np.zeros((16, 16), np.uint8)
    ti = cs.CategoricalGrid(16, 16, 2, ti_a)
    cfg = cs.SimConfig(16, 16, 8, 4, 2, 1)
    dev.set_position_shards(1, 0, None, 64)  # 3x3 = 9 windows
    with pytest.raises(cs.ConfigError, match="position shards"):
        cs.simulate_batch(ti, cfg, [1], None, dev)


def test_nccl_one_rank_communicator(oracle, dev):
    """The NCCL exchange itself: a one-rank communicator (ncclAllGather in
    place) with 3 virtual shards, conditional config with hard data."""
    uid = cs.nccl_unique_id()
    assert len(uid) == 128
    dev.set_position_shards(1, 0, uid, 3)
    rng = np.random.default_rng(11)
    ti_a = rng.integers(0, 4, (96, 96)).astype(np.uint8)
    d = dict(sg_height=100, sg_width=90, template_size=24, overlap=8, dwt_level=2, candidates=5)
    cells = rng.choice(100 * 90, size=40, replace=False)
    hd = [(int(c // 90), int(c % 90), int(rng.integers(0, 4))) for c in cells]
    _check(oracle, dev, ti_a, 4, d, hd, [21, 22])


def test_config2_geometry_single_realization_sharded(oracle, dev):
    """BASELINE config 2 geometry (TI 2000^2, SG 4000^2, T96 OV24 J3 K1, 1 %
    hard data) as ONE realization with 8 position shards -- the single-
    realization decomposition 8(e) prescribes for multi-GPU."""
    from paper_2404_00441_b200 import synth
    ti_a = synth.config2_ti()
    hd = [tuple(int(v) for v in row) for row in synth.config2_hard_data(ti_a)]
    d = dict(sg_height=4000, sg_width=4000, template_size=96, overlap=24, dwt_level=3, candidates=1)
    dev.set_position_shards(1, 0, None, 8)
    _check(oracle, dev, ti_a, 2, d, hd, [cs.mix64(2024, 1)])


@pytest.mark.parametrize("shards", [2, 3, 5])
def test_fast_select_shards(oracle, dev, shards):
    """Shards large enough for the fast select (tile-maximum bound, equal-score
    rescoring, merge rescoring of absent keys) -- K 1-8, hard data."""
    dev.set_position_shards(1, 0, None, shards)
    rng = np.random.default_rng(900 + shards)
    ti_a = np.repeat(np.repeat(rng.integers(0, 3, (64, 64)), 4, 0), 4, 1).astype(np.uint8)
    ti_a[rng.random(ti_a.shape) < 0.2] = 1
    for k in (1, 3, 5, 8):
        if 3249 // shards < 256 + 128 * k:
            continue
        d = dict(sg_height=130, sg_width=118, template_size=32, overlap=8, dwt_level=2, candidates=k)
        hd = None
        if k == 3:
            cells = rng.choice(130 * 118, size=60, replace=False)
            hd = [(int(c // 118), int(c % 118), int(rng.integers(0, 3))) for c in cells]
        _check(oracle, dev, ti_a, 3, d, hd, [k, 1000 + k])


def test_fast_select_shards_bulk_ties(oracle, dev):
    """Binary channel TI at J=3 with K=1/2: tie groups large enough to defer
    to the bulk kernel, which then hands its list to the exchange."""
    from paper_2404_00441_b200 import synth
    ti_a = synth.config2_ti()[:512, :512].copy()
    dev.set_position_shards(1, 0, None, 4)
    dev.set_profiling(True)
    bulk = 0
    for k in (1, 2):
        d = dict(sg_height=200, sg_width=176, template_size=32, overlap=8, dwt_level=3, candidates=k)
        _check(oracle, dev, ti_a, 2, d, None, [5, 6])
        bulk += dev.last_timing()["bulk_jobs"]
    dev.set_profiling(False)
    assert bulk > 0
