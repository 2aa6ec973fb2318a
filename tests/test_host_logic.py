"""Host-side logic of the framework: the raster plan (simulator.hpp:148-190)
through the C-ABI, and the wavefront schedule invariant the batched device
path relies on (every pair of overlapping placements runs in raster order)."""
import numpy as np
import pytest

from paper_2404_00441_b200 import ccwsim as cs


def base():
    return cs.SimConfig(sg_height=64, sg_width=64, template_size=16, overlap=4, dwt_level=2,
                        candidates=4, master_seed=1234)


def test_plan_matches_oracle(oracle):
    for seed in range(40):
        cfg = base()
        cfg.sg_height, cfg.sg_width = 40 + seed, 52 + 2 * seed
        p = cs.plan_raster_path(cfg, cs.Mt19937_64(seed))
        o = oracle.plan_raster_path(cfg, seed)
        assert (p.origin, p.column_major, p.work_height, p.work_width) == \
            (o["origin"], o["column_major"], o["work_height"], o["work_width"])
        assert [(q.top, q.left, q.or_shape) for q in p.placements] == \
            list(zip(o["tops"].tolist(), o["lefts"].tolist(), o["shapes"].tolist()))


def test_plan_geometry_reference_cases():
    # test_simulator.cpp:73-190
    cfg = base()
    cfg.sg_height = cfg.sg_width = 512
    cfg.template_size, cfg.overlap = 32, 8
    p = cs.plan_raster_path(cfg, cs.Mt19937_64(1))
    assert cfg.stride() == 24 and (p.work_height, p.work_width) == (512, 512)
    assert len(p.placements) == 441
    cfg = base()
    cfg.sg_height = cfg.sg_width = 16
    p = cs.plan_raster_path(cfg, cs.Mt19937_64(2))
    assert len(p.placements) == 1 and p.placements[0].or_shape == cs.OR_NONE
    cfg = base()
    cfg.sg_height = 70
    p = cs.plan_raster_path(cfg, cs.Mt19937_64(3))
    assert (p.work_height, p.work_width) == (76, 64)
    seen = set()
    for seed in range(64):
        p = cs.plan_raster_path(base(), cs.Mt19937_64(seed))
        seen.add((p.origin, p.column_major))
    assert len(seen) == 8


def test_plan_coverage_and_stride_law():
    cfg = base()
    cfg.sg_height, cfg.sg_width = 40, 52
    for seed in range(8):
        p = cs.plan_raster_path(cfg, cs.Mt19937_64(seed))
        cov = np.zeros((p.work_height, p.work_width), bool)
        for q in p.placements:
            cov[q.top:q.top + 16, q.left:q.left + 16] = True
        assert cov.all()
        for a, b in zip(p.placements, p.placements[1:]):
            fast = abs(b.top - a.top) if p.column_major else abs(b.left - a.left)
            slow = abs(b.left - a.left) if p.column_major else abs(b.top - a.top)
            assert (fast == cfg.stride()) if slow == 0 else (slow == cfg.stride())


@pytest.mark.parametrize("T,OV", [(16, 4), (16, 8), (12, 8), (40, 12), (64, 16), (32, 24)])
def test_wavefront_key_orders_overlapping_placements(T, OV):
    """The device scheduler runs placement (o, i) in wave (d+1)*o + i, with
    d = ceil(T/stride) - 1 (sim.cu run_simulation).  Every pair of placements
    whose footprints overlap must be ordered the same way as the raster loop
    (simulator.hpp:447-496), and distinct waves may only contain
    non-overlapping footprints."""
    stride = T - OV
    d = (T + stride - 1) // stride - 1
    cfg = cs.SimConfig(sg_height=5 * T, sg_width=4 * T + 3, template_size=T, overlap=OV,
                       dwt_level=1 if (T % 2 == 0 and OV % 2 == 0) else 1, candidates=1)
    for seed in range(8):
        p = cs.plan_raster_path(cfg, cs.Mt19937_64(seed))
        nin = (p.work_height - T) // stride + 1 if p.column_major else (p.work_width - T) // stride + 1
        keys = [(d + 1) * (k // nin) + (k % nin) for k in range(len(p.placements))]
        for a in range(len(p.placements)):
            pa = p.placements[a]
            for b in range(a + 1, len(p.placements)):
                pb = p.placements[b]
                overlap = (abs(pa.top - pb.top) < T) and (abs(pa.left - pb.left) < T)
                if overlap:
                    assert keys[a] < keys[b], (T, OV, a, b)
