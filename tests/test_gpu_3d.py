"""3D extension (BASELINE configs 3 and 4): the CUDA path (libccwgpu.so,
ccw_simulate3d) against the exact-integer 3D restatement (oracle/ccw3d_oracle.c,
pinned to the independent loop restatement in tests/test_oracle3d_cpu.py).
Every comparison is exact equality: realizations and hard-data diagnostics."""
import numpy as np
import pytest

import pyoracle3d as P3
from paper_2404_00441_b200 import ccwsim as cs
from paper_2404_00441_b200 import ccwsim3d as c3
from paper_2404_00441_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def o3():
    return P3.oracle3()


def to_o(cfg: c3.SimConfig3D) -> P3.Cfg3:
    return P3.Cfg3(sg=tuple(cfg.sg), template_size=cfg.template_size, overlap=cfg.overlap,
                   dwt_level=cfg.dwt_level, candidates=cfg.candidates,
                   n_realizations=cfg.n_realizations, any_support=cfg.any_support,
                   master_seed=cfg.master_seed)


def blocky(rng, shape, nf, cell=2):
    g = rng.integers(0, nf, tuple(-(-s // cell) for s in shape))
    for a in range(3):
        g = g.repeat(cell, a)
    return np.ascontiguousarray(g[:shape[0], :shape[1], :shape[2]]).astype(np.uint8)


def random_case(rng, trial):
    J = int(rng.integers(1, 4))
    B = 1 << J
    tcb = int(rng.integers(2, 5)) if J < 3 else int(rng.integers(2, 4))
    T = B * tcb
    anys = bool(trial % 3 == 2)
    OV = int(rng.integers(1, T)) if anys else B * int(rng.integers(1, tcb))
    nf = int(rng.integers(1, 6))
    dims = tuple(int(B * rng.integers(tcb + 1, tcb + 5) + (int(rng.integers(0, B)) if anys else 0))
                 for _ in range(3))
    ti = blocky(rng, dims, nf, cell=int(rng.integers(1, 4)))
    sg = tuple(int(v) for v in rng.integers(T, T + 3 * (T - OV) + 5, 3))
    K = int(rng.integers(1, 9))
    cfg = c3.SimConfig3D(sg=sg, template_size=T, overlap=OV, dwt_level=J, candidates=K,
                         any_support=anys)
    return ti, nf, cfg


@pytest.mark.parametrize("tc3d", [1, 0])
@pytest.mark.parametrize("block", range(4))
def test_randomized_corpus_vs_oracle(o3, block, tc3d):
    """J 1-3, F 1-5, K 1-8, overlap shapes of every corner / axis order,
    the literal-config extension on every third case, hard data on half;
    with the tcgen05 screen (int8 block counts at J <= 2, F <= 5; two-digit
    counts otherwise) and without."""
    rng = np.random.default_rng(1000 + block)
    dev = cs.default_device()
    dev.set_option("tc3d", tc3d)
    try:
        _corpus(o3, block, tc3d, rng, dev)
    finally:
        dev.set_option("tc3d", 1)


def _corpus(o3, block, tc3d, rng, dev):
    for trial in range(8):
        ti_a, nf, cfg = random_case(rng, trial)
        seeds = [int(s) for s in rng.integers(0, 2**63, 4)]
        hd = None
        if trial % 2 == 1:
            ref0 = o3.simulate_one(ti_a, nf, to_o(cfg), None, seed=seeds[0])["realization"]
            hd = synth.hard_data3d_from(ref0, 0.02, 7 + trial)
        ti = c3.TrainingImage3D(ti_a, nf, cfg.dwt_level)
        got, diags = c3.simulate3d(ti, cfg, seeds, hd)
        for r, s in enumerate(seeds):
            o = o3.simulate_one(ti_a, nf, to_o(cfg), hd, seed=s)
            assert np.array_equal(got[r], o["realization"]), (block, trial, r, cfg)
            assert diags[r].pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]
            assert diags[r].corner == o["diagnostics"]["corner"]
            assert diags[r].order == o["diagnostics"]["order"]
        int8_counts = cfg.dwt_level <= 2 and nf <= 5
        # 6: tcgen05 GEMM on int8 counts, 7: on 9-bit counts as two digits (three rows per job)
        assert dev.last_timing()["ccf_variant"] == ((6 if int8_counts else 7) if tc3d else 3 if int8_counts else 4)
        ti.close()


def test_all_corners_and_orders(o3):
    """Enough seeds that all 8 corners x 6 axis orders occur, one call."""
    rng = np.random.default_rng(5)
    ti_a = blocky(rng, (40, 36, 44), 3, cell=2)
    cfg = c3.SimConfig3D(sg=(30, 34, 29), template_size=8, overlap=4, dwt_level=1, candidates=3)
    seeds = list(range(1, 320))
    ti = c3.TrainingImage3D(ti_a, 3, 1)
    got, diags = c3.simulate3d(ti, cfg, seeds)
    assert len({(d.corner, d.order) for d in diags}) == 48
    for r in range(0, len(seeds), 7):
        o = o3.simulate_one(ti_a, 3, to_o(cfg), None, seed=seeds[r])
        assert np.array_equal(got[r], o["realization"]), r


@pytest.mark.parametrize("nf", [2, 4, 7])
def test_packed_host_result(o3, nf):
    """Option pack = 2: result codes packed 1 / 2 / 4 bits per cell for the
    device -> host copy and unpacked by host threads; same realizations."""
    rng = np.random.default_rng(40 + nf)
    ti_a = blocky(rng, (40, 36, 44), nf, cell=2)
    cfg = c3.SimConfig3D(sg=(41, 50, 37), template_size=8, overlap=4, dwt_level=1, candidates=2)
    seeds = [3, 4, 5]
    ti = c3.TrainingImage3D(ti_a, nf, 1)
    dev = cs.default_device()
    ref, _ = c3.simulate3d(ti, cfg, seeds)
    with dev.options(pack=2):
        got, _ = c3.simulate3d(ti, cfg, seeds)
        assert dev.last_timing()["d2h_bytes"] < ref.size
    assert np.array_equal(got, ref)
    o = o3.simulate_one(ti_a, nf, to_o(cfg), None, seed=seeds[1])
    assert np.array_equal(got[1], o["realization"])
    with dev.options(tc3d=0):
        alt, _ = c3.simulate3d(ti, cfg, seeds)
    assert np.array_equal(alt, ref)
    ti.close()


@pytest.mark.parametrize("nf,J", [(6, 1), (7, 2), (9, 2), (6, 3), (8, 3)])
def test_many_facies(o3, nf, J):
    """More than 5 facies (more than 4 screen channels: int32 counts at B <= 4,
    two-digit tensor screen at B = 8)."""
    rng = np.random.default_rng(70 + nf + J)
    B = 1 << J
    T = 2 * B if J == 3 else 4 * B
    ti_a = blocky(rng, (5 * T // 2 + B, 3 * T, 2 * T + 2 * B), nf, cell=2)
    cfg = c3.SimConfig3D(sg=(2 * T + 3, 2 * T, 3 * T - 1), template_size=T, overlap=B, dwt_level=J, candidates=3)
    ti = c3.TrainingImage3D(ti_a, nf, J)
    seeds = [11, 12]
    got, _ = c3.simulate3d(ti, cfg, seeds)
    for r, s in enumerate(seeds):
        o = o3.simulate_one(ti_a, nf, to_o(cfg), None, seed=s)
        assert np.array_equal(got[r], o["realization"]), (nf, J, r)
    ti.close()


def test_ensemble_seeds(o3):
    rng = np.random.default_rng(9)
    ti_a = blocky(rng, (24, 32, 28), 2)
    cfg = c3.SimConfig3D(sg=(20, 30, 25), template_size=8, overlap=4, dwt_level=2, candidates=2,
                         n_realizations=5, master_seed=77)
    ti = c3.TrainingImage3D(ti_a, 2, 2)
    got, _ = c3.simulate3d_ensemble(ti, cfg)
    ref, _ = o3.simulate_ensemble(ti_a, 2, to_o(cfg), None, workers=3)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("virtual", [2, 3, 5])
def test_position_shards(o3, virtual):
    """Candidate-position sharding of the screen boxes (virtual shards on one
    GPU, exchange through device memory): identical realizations."""
    rng = np.random.default_rng(40 + virtual)
    ti_a = blocky(rng, (48, 80, 72), 4, cell=2)
    cfg = c3.SimConfig3D(sg=(24, 40, 40), template_size=16, overlap=4, dwt_level=1, candidates=3)
    dev = cs.default_device()
    ti = c3.TrainingImage3D(ti_a, 4, 1, dev)
    seeds = [11, 12]
    base, _ = c3.simulate3d(ti, cfg, seeds)
    dev.set_position_shards(1, 0, None, virtual)
    try:
        got, _ = c3.simulate3d(ti, cfg, seeds)
    finally:
        dev.set_position_shards(1, 0, None, 1)
    assert np.array_equal(got, base)
    o = o3.simulate_one(ti_a, 4, to_o(cfg), None, seed=11)
    assert np.array_equal(got[0], o["realization"])


def test_position_shards_nccl_one_rank():
    """The same through a real one-rank NCCL communicator (ncclAllGather)."""
    rng = np.random.default_rng(3)
    ti_a = blocky(rng, (64, 96, 96), 3, cell=2)
    cfg = c3.SimConfig3D(sg=(24, 32, 32), template_size=16, overlap=8, dwt_level=2, candidates=2)
    dev = cs.default_device()
    ti = c3.TrainingImage3D(ti_a, 3, 2, dev)
    base, _ = c3.simulate3d(ti, cfg, [5, 6])
    dev.set_position_shards(1, 0, cs.nccl_unique_id(), 2)
    try:
        got, _ = c3.simulate3d(ti, cfg, [5, 6])
    finally:
        dev.set_position_shards(1, 0, None, 1)
    assert np.array_equal(got, base)


def test_validation_messages():
    ti = c3.TrainingImage3D(np.zeros((16, 16, 16), np.uint8), 2, 2)
    with pytest.raises(cs.ConfigError, match="overlap"):
        c3.simulate3d(ti, c3.SimConfig3D(sg=(16, 16, 16), template_size=8, overlap=3, dwt_level=2), [1])
    with pytest.raises(cs.ConfigError, match="template"):
        c3.simulate3d(ti, c3.SimConfig3D(sg=(16, 16, 16), template_size=32, overlap=4, dwt_level=2), [1])
    with pytest.raises(cs.BoundsError, match="outside"):
        c3.simulate3d(ti, c3.SimConfig3D(sg=(16, 16, 16), template_size=8, overlap=4, dwt_level=2), [1],
                      [(0, 0, 16, 1)])
    with pytest.raises(cs.ConfigError, match="candidates"):
        c3.simulate3d(ti, c3.SimConfig3D(sg=(16, 16, 16), template_size=8, overlap=4, dwt_level=2,
                                         candidates=17), [1])


def config3_cfg(literal: bool):
    return c3.SimConfig3D(sg=(100, 200, 200), template_size=32, overlap=8, dwt_level=2, candidates=1,
                          n_realizations=16, any_support=literal, master_seed=20240441)


@pytest.mark.slow
@pytest.mark.parametrize("literal", [False, True])
def test_config3_full_size(o3, literal):
    """BASELINE config 3 (4 facies, SG 200x200x100, T32 OV8 J2, 16
    realizations): adjusted TI 180x148x120, or the literal 180x150x120
    through the any_support extension.  Two realizations of the 16-call
    bit-identical to the restatement (host threads split each score map)."""
    ti_a = synth.config3_ti()
    if not literal:
        ti_a = np.ascontiguousarray(ti_a[:, :148, :])
    cfg = config3_cfg(literal)
    ti = c3.TrainingImage3D(ti_a, 4, 2)
    got, diags = c3.simulate3d_ensemble(ti, cfg)
    for r in (0, 9):
        o = o3.simulate_one(ti_a, 4, to_o(cfg), None, seed=cs.mix64(cfg.master_seed, r + 1), threads=16)
        assert np.array_equal(got[r], o["realization"]), r


@pytest.mark.slow
@pytest.mark.parametrize("ov", [16, 12])
def test_config4_full_size(o3, ov):
    """BASELINE config 4 (5 facies, TI 400x400x200, SG 500x500x250, T48, J3,
    20 vertical wells, one realization): OV 16 (aligned) and the literal OV 12
    through the any_support extension; wells read from a seeded
    unconditional realization.  Bit-identical to the restatement."""
    ti_a = synth.config4_ti()
    cfg = c3.SimConfig3D(sg=(250, 500, 500), template_size=48, overlap=ov, dwt_level=3, candidates=1,
                         any_support=ov % 8 != 0, master_seed=20240441)
    ti = c3.TrainingImage3D(ti_a, 5, 3)
    ref_real, _ = c3.simulate3d(ti, cfg, [777])
    wells = synth.wells3d_from(ref_real[0], 20, 404)
    seed = cs.mix64(cfg.master_seed, 1)
    got, diags = c3.simulate3d(ti, cfg, [seed], wells)
    o = o3.simulate_one(ti_a, 5, to_o(cfg), wells, seed=seed, threads=16)
    assert np.array_equal(got[0], o["realization"])
    assert diags[0].pre_overwrite_mismatches == o["diagnostics"]["pre_overwrite_mismatches"]
    assert (got[0][wells[:, 0], wells[:, 1], wells[:, 2]] == wells[:, 3]).all()
