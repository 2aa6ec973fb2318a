"""The C-ABI library loads and exports every symbol include/ccwgpu.h declares;
host-side entry points (validation, plan, mix64) work without a GPU; device
entry points fail loudly (never a silent CPU fallback) when no GPU exists."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2404_00441_b200 import _abi, ccwsim as cs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ccwgpu.h")).read()
    return sorted(set(re.findall(r"CCW_API\s+[\w\s\*]*?\b(ccw_\w+)\s*\(", text)))


def test_header_declares_the_binding_surface():
    decl = declared_symbols()
    assert len(decl) >= 25
    assert sorted(_abi.SIGNATURES) == decl


def test_library_exports_every_declared_symbol():
    lib = _abi.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_library_has_sm100a_code():
    data = open(_abi.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_mix64_matches_mirror_and_oracle(oracle):
    lib = _abi.lib()
    for seed, idx in [(0, 1), (1234, 7), (2**64 - 1, 3), (42, 100)]:
        v = lib.ccw_mix64(seed, idx)
        assert v == cs.mix64(seed, idx) == oracle.mix64(seed, idx)


def test_mt19937_64_mirror_matches_oracle(oracle):
    for seed in (0, 5489, 2**64 - 1):
        g = cs.Mt19937_64(seed)
        assert [g() for _ in range(700)] == [int(x) for x in oracle.mt64_draws(seed, 700)]
    ns = np.array([1, 2, 3, 5, 7, 1000, 2**63 + 5], np.uint64)
    g = cs.Mt19937_64(77)
    assert [cs.bounded(g, int(n)) for n in ns] == [int(x) for x in oracle.bounded_draws(77, ns)]


def test_validation_messages_name_the_key():
    # simulator.hpp:46-84 via ccw_validate_config (host-only)
    base = dict(sg_height=64, sg_width=64, template_size=16, overlap=4, dwt_level=2,
                candidates=4)
    cs.SimConfig(**base).validate()
    for kw, kind, word in [
        (dict(overlap=16), cs.ConfigError, "overlap"),
        (dict(template_size=32, overlap=6), cs.ConfigError, "overlap"),
        (dict(template_size=18, overlap=8), cs.ConfigError, "template"),
        (dict(sg_height=8), cs.ConfigError, "template"),
        (dict(candidates=0), cs.ConfigError, "candidates"),
        (dict(n_realizations=0), cs.ConfigError, "realizations"),
        (dict(dwt_level=0), cs.ConfigError, "dwt_level"),
        (dict(sg_width=0), cs.ConfigError, "sg_size"),
    ]:
        d = dict(base)
        d.update(kw)
        with pytest.raises(kind) as e:
            cs.SimConfig(**d).validate()
        assert word in str(e.value)
    small = cs.CategoricalGrid(8, 8, 2)
    with pytest.raises(cs.ConfigError):
        cs.SimConfig(**base).validate_against(small)
    odd = cs.CategoricalGrid(66, 66, 2)
    with pytest.raises(cs.ConfigError) as e:
        cs.SimConfig(**base).validate_against(odd)
    assert "training image" in str(e.value)


def test_hard_data_validation():
    # grid.hpp:151-170
    ti = cs.CategoricalGrid(64, 64, 2)
    cfg = cs.SimConfig(64, 64, 16, 4, 2, 4)
    cfg.hard_data = cs.HardDataSet([cs.HardDatum(70, 1, 0)])
    with pytest.raises(cs.BoundsError):
        cfg.validate_against(ti)
    cfg.hard_data = cs.HardDataSet([cs.HardDatum(1, 1, 5)])
    with pytest.raises(cs.BoundsError):
        cfg.validate_against(ti)
    cfg.hard_data = cs.HardDataSet([cs.HardDatum(0, 0, 1), cs.HardDatum(0, 0, 0)])
    with pytest.raises(cs.StructureError) as e:
        cfg.validate_against(ti)
    assert "(0, 0)" in str(e.value)


def test_grid_invariants():
    # grid.hpp:16-81
    with pytest.raises(cs.DimensionError):
        cs.CategoricalGrid(0, 3, 2)
    with pytest.raises(cs.BoundsError):
        cs.CategoricalGrid(2, 2, 2, [0, 1, 2, 0])
    with pytest.raises(cs.StructureError):
        cs.CategoricalGrid(2, 2, 2, [0, 1, 1])
    g = cs.CategoricalGrid(2, 3, 3, [0, 1, 2, 2, 1, 0])
    assert g.at(1, 2) == 0
    with pytest.raises(cs.BoundsError) as e:
        g.at(2, 0)
    assert "(2, 0)" in str(e.value)


def test_device_calls_fail_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(cs.DeviceError):
        cs.Device(0)


def test_nccl_unique_id_host_side():
    """The position-sharding rendezvous (ccw_nccl_unique_id: libnccl.so.2 is
    dlopen'ed on first use) works without a GPU: 128 bytes, fresh per call."""
    from paper_2404_00441_b200 import ccwsim as cs
    a, b = cs.nccl_unique_id(), cs.nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b


def test_position_shard_arguments_validated():
    """ccw_ctx_set_position_shards rejects bad ranks before touching a device
    (a null context returns the generic error code, never crashes)."""
    import ctypes as C
    from paper_2404_00441_b200 import _abi
    L = _abi.lib()
    assert L.ccw_ctx_set_position_shards(None, 2, 0, None, 1) == 7
    ms = C.c_double()
    assert L.ccw_measure_ccf_screen(None, None, 64, 1, 1, C.byref(ms)) == 7
