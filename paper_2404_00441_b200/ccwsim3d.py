"""3D extension of the simulate API (BASELINE configs 3 and 4), backed by
libccwgpu.so (include/ccwgpu.h, ccw_*3d).

The reference has no 3D.  This module generalizes
``simulate_one`` / ``simulate_ensemble`` (simulator.hpp:418-566) to 3D grids
as defined in oracle/ccw3d_oracle.h: arrays are numpy uint8 of shape
(d0, d1, d2) with axis 0 vertical; hard data are (i0, i1, i2, facies) rows.
Every call runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from .ccwsim import Device, _raise, default_device, mix64

_M64 = (1 << 64) - 1


@dataclass
class SimConfig3D:
    sg: Tuple[int, int, int] = (64, 64, 64)
    template_size: int = 16
    overlap: int = 4
    dwt_level: int = 2
    candidates: int = 1
    n_realizations: int = 1
    any_support: bool = False   # literal-config extension (overlap not a multiple of 2^J)
    master_seed: int = 0

    def to_c(self) -> _abi.Sim3dConfigC:
        c = _abi.Sim3dConfigC()
        for a in range(3):
            c.sg[a] = int(self.sg[a])
        c.template_size = int(self.template_size)
        c.overlap = int(self.overlap)
        c.dwt_level = int(self.dwt_level)
        c.candidates = int(self.candidates)
        c.n_realizations = int(self.n_realizations)
        c.any_support = int(bool(self.any_support))
        c.master_seed = int(self.master_seed) & _M64
        return c


@dataclass
class Diagnostics3D:
    seed: int
    corner: int
    order: int
    work: Tuple[int, int, int]
    placement_count: int
    hard_data_count: int
    pre_overwrite_mismatches: int
    wall_seconds: float


def _diag(d) -> Diagnostics3D:
    return Diagnostics3D(int(d.seed), d.corner, d.order, tuple(d.work), d.placement_count,
                         d.hard_data_count, d.pre_overwrite_mismatches, d.wall_seconds)


def _hd(hd):
    if hd is None or len(hd) == 0:
        return None, 0
    a = np.ascontiguousarray(np.asarray(hd, np.int32).reshape(-1, 4))
    return a, a.shape[0]


def validate_config3d(cfg: SimConfig3D, ti_shape=None, num_facies: int = 2, hard_data=None) -> None:
    L = _abi.lib()
    dims = np.asarray(ti_shape, np.int32) if ti_shape is not None else None
    a, n = _hd(hard_data)
    msg = C.create_string_buffer(512)
    rc = L.ccw_validate_config3d(C.byref(cfg.to_c()),
                                 dims.ctypes.data_as(_abi.I32P) if dims is not None else None,
                                 int(num_facies), a.ctypes.data_as(_abi.I32P) if a is not None else None,
                                 n, msg, 512)
    if rc:
        _raise(rc, msg.value.decode())


class TrainingImage3D:
    """A 3D TI resident on the device with its level-J block counts (ccw_ti3d)."""

    def __init__(self, cells: np.ndarray, num_facies: int, levels: int, device: Optional[Device] = None):
        self.device = device or default_device()
        self.cells = np.ascontiguousarray(cells, np.uint8)
        if self.cells.ndim != 3:
            raise ValueError("a 3D training image needs a (d0, d1, d2) array")
        self.num_facies = int(num_facies)
        self.levels = int(levels)
        h = C.c_void_p()
        d0, d1, d2 = self.cells.shape
        self.device.check(self.device._lib.ccw_ti3d_create(
            self.device.handle, self.cells.ctypes.data_as(_abi.U8P), d0, d1, d2, self.num_facies,
            self.levels, C.byref(h)))
        self.handle = h

    @property
    def shape(self):
        return self.cells.shape

    def close(self) -> None:
        if self.handle:
            self.device._lib.ccw_ti3d_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def simulate3d(ti: TrainingImage3D, cfg: SimConfig3D, seeds: Sequence[int], hard_data=None,
               trace: bool = False):
    """Realization r uses seeds[r]; returns (n, sg0, sg1, sg2) codes and
    diagnostics, plus with trace=True the (n, placements, 3) TI origins."""
    dev = ti.device
    seeds_a = np.array([int(s) & _M64 for s in seeds], np.uint64)
    n = len(seeds_a)
    out = np.zeros((n,) + tuple(int(v) for v in cfg.sg), np.uint8)
    diags = (_abi.Diag3dC * max(n, 1))()
    a, nh = _hd(hard_data)
    args = (dev.handle, ti.handle, C.byref(cfg.to_c()), seeds_a.ctypes.data_as(_abi.U64P), n,
            a.ctypes.data_as(_abi.I32P) if a is not None else None, nh, out.ctypes.data_as(_abi.U8P), diags)
    if trace:
        t, stride = cfg.template_size, cfg.template_size - cfg.overlap
        cap = 1
        for ax in range(3):
            w = t if cfg.sg[ax] == t else t + -(-(cfg.sg[ax] - t) // stride) * stride
            cap *= (w - t) // stride + 1
        org = np.zeros((n, cap, 3), np.int32)
        dev.check(dev._lib.ccw_simulate3d_trace(*args, org.ctypes.data_as(_abi.I32P), cap))
        return out, [_diag(d) for d in diags[:n]], org
    dev.check(dev._lib.ccw_simulate3d(*args))
    return out, [_diag(d) for d in diags[:n]]


def simulate3d_ensemble(ti: TrainingImage3D, cfg: SimConfig3D, hard_data=None):
    """Seeds mix64(master, r + 1) (simulator.hpp:523-566 in 3D)."""
    return simulate3d(ti, cfg, [mix64(cfg.master_seed, r + 1) for r in range(cfg.n_realizations)],
                      hard_data)
