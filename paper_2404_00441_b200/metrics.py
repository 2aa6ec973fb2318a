"""Python mirror of the reference's validation metrics (metrics.hpp:68-311),
computed on the GPU by libccwgpu.so (csrc/metrics.cu).

Same names and error behaviour as the reference: ``indicator_variogram``,
``connectivity_function``, ``ensemble_average``, ``pattern_histogram``,
``js_divergence``, ``downsample_majority``.  The batched forms
(``indicator_variograms``, ``connectivity_functions``) take a whole ensemble
-- a (n, h, w) numpy array, or a CUDA tensor such as the output buffer of
``ccw_simulate_device`` (read in place, no host round trip).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _abi
from .ccwsim import CategoricalGrid, Device, _raise, default_device

EAST_WEST, NORTH_SOUTH = 0, 1


def _dir(d) -> int:
    if isinstance(d, str):
        return {"east_west": 0, "north_south": 1}[d]
    return int(d)


def _dir_name(d: int) -> str:
    return "east_west" if d == 0 else "north_south"


@dataclass
class VariogramSeries:
    direction: str
    facies: int
    facies_present: bool
    gamma: List[float]


@dataclass
class ConnectivitySeries:
    direction: str
    facies: int
    probability: List[Optional[float]]


def _grids(x):
    """(pointer, on_device, n, h, w, keepalive) of an ensemble."""
    if hasattr(x, "data_ptr") and getattr(x, "is_cuda", False):  # torch CUDA tensor (n, h, w) uint8
        n, h, w = (1,) + tuple(x.shape) if x.dim() == 2 else tuple(x.shape)
        return C.cast(C.c_void_p(x.data_ptr()), _abi.U8P), 1, n, h, w, x
    if isinstance(x, CategoricalGrid):
        a = np.ascontiguousarray(x.cells, np.uint8)[None]
    elif isinstance(x, (list, tuple)):
        shapes = {(g.height, g.width) if isinstance(g, CategoricalGrid) else np.asarray(g).shape for g in x}
        if len(shapes) > 1:
            from .ccwsim import StructureError
            raise StructureError("ensemble realizations differ in size")
        a = np.ascontiguousarray(np.stack([g.cells if isinstance(g, CategoricalGrid) else np.asarray(g, np.uint8)
                                           for g in x]), np.uint8) if x else np.zeros((0, 1, 1), np.uint8)
    else:
        a = np.ascontiguousarray(x, np.uint8)
        if a.ndim == 2:
            a = a[None]
    return a.ctypes.data_as(_abi.U8P), 0, a.shape[0], a.shape[1], a.shape[2], a


def indicator_variograms(grids, facies: int, direction, max_lag: int, device: Optional[Device] = None):
    """gamma of every realization: ((n, max_lag) array, (n,) facies-present flags)."""
    dev = device or default_device()
    p, on, n, h, w, keep = _grids(grids)
    gamma = np.zeros((max(n, 1), max(max_lag, 1)), np.float64)
    present = np.zeros(max(n, 1), np.int32)
    dev.check(dev._lib.ccw_variogram(dev.handle, p, on, n, h, w, int(facies), _dir(direction), int(max_lag),
                                     gamma.ctypes.data_as(_abi.F64P), present.ctypes.data_as(_abi.I32P)))
    return gamma[:n], present[:n].astype(bool)


def indicator_variogram(grid, facies: int, direction, max_lag: int, device=None) -> VariogramSeries:
    """metrics.hpp:68-112."""
    g, pr = indicator_variograms(grid, facies, direction, max_lag, device)
    return VariogramSeries(_dir_name(_dir(direction)), int(facies), bool(pr[0]), g[0].tolist())


def connectivity_functions(grids, facies: int, direction, max_lag: int, device: Optional[Device] = None):
    """(n, max_lag) connection probabilities, NaN where undefined."""
    dev = device or default_device()
    p, on, n, h, w, keep = _grids(grids)
    prob = np.zeros((max(n, 1), max(max_lag, 1)), np.float64)
    dev.check(dev._lib.ccw_connectivity(dev.handle, p, on, n, h, w, int(facies), _dir(direction), int(max_lag),
                                        prob.ctypes.data_as(_abi.F64P)))
    return prob[:n]


def connectivity_function(grid, facies: int, direction, max_lag: int, device=None) -> ConnectivitySeries:
    """metrics.hpp:158-205 (None = the reference's unset optional)."""
    pr = connectivity_functions(grid, facies, direction, max_lag, device)[0]
    return ConnectivitySeries(_dir_name(_dir(direction)), int(facies),
                              [None if np.isnan(v) else float(v) for v in pr])


def ensemble_average(ensemble, facies: int, device: Optional[Device] = None) -> np.ndarray:
    """metrics.hpp:208-227: per-cell fraction of realizations equal to facies."""
    dev = device or default_device()
    p, on, n, h, w, keep = _grids(ensemble)
    out = np.zeros((h, w), np.float64)
    dev.check(dev._lib.ccw_ensemble_average(dev.handle, p, on, n, h, w, int(facies),
                                            out.ctypes.data_as(_abi.F64P)))
    return out


def downsample_majority(grid: CategoricalGrid, factor: int, device: Optional[Device] = None) -> CategoricalGrid:
    """metrics.hpp:288-311: block majority, ties to the lowest code."""
    if factor == 1:
        return grid
    dev = device or default_device()
    p, on, n, h, w, keep = _grids(grid)
    out = np.zeros((max(h // max(factor, 1), 1), max(w // max(factor, 1), 1)), np.uint8)
    dev.check(dev._lib.ccw_downsample_majority(dev.handle, p, on, h, w, grid.num_facies, int(factor),
                                               out.ctypes.data_as(_abi.U8P)))
    return CategoricalGrid(out.shape[0], out.shape[1], grid.num_facies, out)


class PatternHistogram:
    """metrics.hpp:44-49, resident on the device (ccw_phist); ``counts``
    (window bytes -> multiplicity) is fetched on first use."""

    def __init__(self, handle, device: Device):
        self.handle = handle
        self.device = device
        n, t, win = C.c_int64(), C.c_int64(), C.c_int()
        device.check(device._lib.ccw_phist_info(handle, C.byref(n), C.byref(t), C.byref(win)))
        self.distinct, self.total, self.window = n.value, t.value, win.value
        self._counts = None

    @property
    def counts(self) -> Dict[bytes, int]:
        if self._counts is None:
            kw = self.window * self.window
            keys = np.zeros(max(self.distinct, 1) * kw, np.uint8)
            cnt = np.zeros(max(self.distinct, 1), np.uint64)
            self.device.check(self.device._lib.ccw_phist_copy(self.device.handle, self.handle,
                                                              keys.ctypes.data_as(_abi.U8P),
                                                              cnt.ctypes.data_as(_abi.U64P)))
            self._counts = {keys[i * kw:(i + 1) * kw].tobytes(): int(cnt[i]) for i in range(self.distinct)}
        return self._counts

    def close(self):
        if self.handle:
            self.device._lib.ccw_phist_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pattern_histogram(grid, w: int, stride: int = 1, num_facies: Optional[int] = None,
                      device: Optional[Device] = None) -> PatternHistogram:
    """metrics.hpp:230-254.  ``grid``: a CategoricalGrid, (h, w) array or CUDA tensor."""
    dev = device or default_device()
    nf = num_facies if num_facies is not None else (grid.num_facies if isinstance(grid, CategoricalGrid) else 256)
    p, on, n, h, ww, keep = _grids(grid)
    out = C.c_void_p()
    dev.check(dev._lib.ccw_pattern_histogram(dev.handle, p, on, h, ww, int(nf), int(w), int(stride), C.byref(out)))
    return PatternHistogram(out, dev)


def js_divergence(p: PatternHistogram, q: PatternHistogram) -> float:
    """metrics.hpp:258-284 (base-2, clamped to [0, 1])."""
    v = C.c_double()
    p.device.check(p.device._lib.ccw_js_divergence(p.device.handle, p.handle, q.handle, C.byref(v)))
    return v.value


@dataclass
class AnodiLevel:
    between_a: float
    between_b: float
    within_a: float
    within_b: float
    d_between: float
    d_within: float
    ratio: float
    weight: float


@dataclass
class AnodiResult:
    levels: List[AnodiLevel]
    aggregate: float


def anodi(ensemble_a, ensemble_b, ti, levels: int, window: int, weights: Optional[Sequence[float]] = None,
          num_facies: Optional[int] = None, device: Optional[Device] = None) -> AnodiResult:
    """metrics.hpp:318-384 (the MDS step needs Eigen and is not included):
    ensembles as lists of grids, (n, h, w) arrays or CUDA tensors."""
    dev = device or default_device()
    pa, ona, na, h, w, ka = _grids(ensemble_a)
    pb, onb, nb, hb, wb, kb = _grids(ensemble_b)
    if ona != onb:
        raise ValueError("both ensembles must be on the device or both on the host")
    if (hb, wb) != (h, w):
        from .ccwsim import StructureError
        raise StructureError("ensembles differ in grid size")
    t = np.ascontiguousarray(ti.cells if isinstance(ti, CategoricalGrid) else ti, np.uint8)
    nf = num_facies if num_facies is not None else (ti.num_facies if isinstance(ti, CategoricalGrid)
                                                    else int(t.max()) + 1)
    out = np.zeros((max(levels, 1), 8), np.float64)
    agg = C.c_double()
    wts = np.ascontiguousarray(weights, np.float64) if weights is not None else None
    if wts is not None and len(wts) != levels:
        from .ccwsim import StructureError
        raise StructureError("weight count does not match level count")
    dev.check(dev._lib.ccw_anodi(dev.handle, pa, na, pb, nb, ona, h, w, t.ctypes.data_as(_abi.U8P), t.shape[0],
                                 t.shape[1], int(nf), int(levels), int(window),
                                 wts.ctypes.data_as(_abi.F64P) if wts is not None else None,
                                 out.ctypes.data_as(_abi.F64P), C.byref(agg)))
    return AnodiResult([AnodiLevel(*[float(v) for v in row]) for row in out[:levels]], agg.value)
