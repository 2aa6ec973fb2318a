"""Python mirror of the reference's ``namespace ccwsim`` hot-path API.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/ccwsim/{grid,wavelet,matcher,simulator,rng}.hpp,
backed by libccwgpu.so.  Grids are numpy ``uint8`` arrays (row-major, row 0 at
the top); real planes are numpy ``float64`` arrays.

Host-only pieces are host logic by nature (the mt19937_64 generator and
``bounded``, ``mix64``, ``coarse_to_fine``, ``select_unconditional``); every
numeric operator and the simulation itself run on the GPU through the C-ABI.
"""
from __future__ import annotations

import atexit
import contextlib
import ctypes as C
import threading
import weakref
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi

# ----------------------------------------------------------------- errors --


class Error(RuntimeError):
    """ccwsim::Error (errors.hpp:9-12)."""


class BoundsError(Error):
    pass


class DimensionError(Error):
    pass


class StructureError(Error):
    pass


class ConfigError(Error):
    pass


class EmptyInputError(Error):
    pass


class IoError(Error):
    pass


class ParseError(Error):
    """errors.hpp:57-73: a malformed input file; carries the path and the
    1-based line number (0 when unknown)."""

    def __init__(self, path: str, line, msg: Optional[str] = None):
        if msg is None:  # (path, msg)
            line, msg = 0, line
            super().__init__(f"{path}: {msg}")
        else:
            super().__init__(f"{path}:{line}: {msg}")
        self.path = path
        self.line = line


class DegeneracyError(Error):
    """errors.hpp:44-47 (ANODI on degenerate ensembles)."""


class DeviceError(Error):
    """CUDA failure inside libccwgpu.so (status >= 100)."""


_ERRORS = {1: BoundsError, 2: DimensionError, 3: StructureError, 4: ConfigError,
           5: EmptyInputError, 6: IoError, 7: Error, 8: DegeneracyError}


def _raise(code: int, msg: str):
    raise _ERRORS.get(code, DeviceError)(msg)


# -------------------------------------------------------------- rng (host) --

_M64 = (1 << 64) - 1


class Mt19937_64:
    """std::mt19937_64 (sequence pinned by the C++ standard)."""

    def __init__(self, seed: int = 5489):
        self.seed(seed)

    def seed(self, s: int) -> None:
        mt = [0] * 312
        mt[0] = s & _M64
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self.mt = mt
        self.idx = 312

    def __call__(self) -> int:
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64


def mix64(seed: int, index: int) -> int:
    """rng.hpp:11-16."""
    z = (seed + index * 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def bounded(rng: Mt19937_64, n: int) -> int:
    """rng.hpp:21-28: unbiased draw in [0, n) by rejection."""
    threshold = ((1 << 64) - n) % n
    while True:
        r = rng()
        if r >= threshold:
            return r % n


# ------------------------------------------------------------- data types --

class CategoricalGrid:
    """grid.hpp:16-81 over a uint8 numpy array (codes in [0, num_facies))."""

    def __init__(self, height: int, width: int, num_facies: int, cells=None, fill: int = 0):
        if height <= 0 or width <= 0:
            raise DimensionError("grid dimensions must be positive")
        if num_facies <= 0:
            raise DimensionError("num_facies must be positive")
        if num_facies > 255:
            raise DimensionError("num_facies must be <= 255 (uint8 codes)")
        if cells is None:
            if fill < 0 or fill >= num_facies:
                raise BoundsError(f"fill code {fill} outside [0, {num_facies})")
            arr = np.full((height, width), fill, np.uint8)
        else:
            raw = np.asarray(cells)
            if raw.size != height * width:
                raise StructureError(f"cell count {raw.size} does not match {height}x{width}")
            flat = raw.reshape(-1).astype(np.int64)
            bad = np.nonzero((flat < 0) | (flat >= num_facies))[0]
            if bad.size:
                i = int(bad[0])
                raise BoundsError(f"cell {i} holds code {int(flat[i])} outside [0, {num_facies})")
            arr = flat.astype(np.uint8).reshape(height, width)
        arr.setflags(write=False)
        self._cells = arr
        self.num_facies = int(num_facies)

    @classmethod
    def _trusted(cls, cells: np.ndarray, num_facies: int) -> "CategoricalGrid":
        """Wrap device output without re-validating every code."""
        g = cls.__new__(cls)
        cells.setflags(write=False)
        g._cells = cells
        g.num_facies = int(num_facies)
        return g

    @classmethod
    def from_array(cls, cells, num_facies: Optional[int] = None) -> "CategoricalGrid":
        a = np.asarray(cells)
        nf = int(a.max()) + 1 if num_facies is None else num_facies
        return cls(a.shape[0], a.shape[1], nf, a)

    @property
    def height(self) -> int:
        return self._cells.shape[0]

    @property
    def width(self) -> int:
        return self._cells.shape[1]

    @property
    def cells(self) -> np.ndarray:
        return self._cells

    def area(self) -> int:
        return self.height * self.width

    def at(self, r: int, c: int) -> int:
        if r < 0 or r >= self.height or c < 0 or c >= self.width:
            raise BoundsError(f"cell ({r}, {c}) outside {self.height}x{self.width} grid")
        return int(self._cells[r, c])

    def __eq__(self, other) -> bool:
        return (isinstance(other, CategoricalGrid) and self.num_facies == other.num_facies
                and np.array_equal(self._cells, other._cells))

    __hash__ = object.__hash__  # identity: cells are read-only

    def __repr__(self) -> str:
        return f"CategoricalGrid({self.height}x{self.width}, F={self.num_facies})"


@dataclass(frozen=True)
class HardDatum:
    row: int
    col: int
    facies: int


@dataclass
class HardDataSet:
    points: List[HardDatum] = field(default_factory=list)

    def empty(self) -> bool:
        return not self.points

    def size(self) -> int:
        return len(self.points)


def _hd_array(hd) -> Optional[np.ndarray]:
    if hd is None:
        return None
    if isinstance(hd, HardDataSet):
        hd = hd.points
    if isinstance(hd, np.ndarray):
        return np.ascontiguousarray(hd, np.int32).reshape(-1, 3)
    rows = [(p.row, p.col, p.facies) if isinstance(p, HardDatum) else tuple(p) for p in hd]
    return np.ascontiguousarray(np.array(rows, np.int32).reshape(-1, 3))


@dataclass
class SimConfig:
    """simulator.hpp:28-85 (defaults :34-39)."""
    sg_height: int = 0
    sg_width: int = 0
    template_size: int = 0
    overlap: int = 0
    dwt_level: int = 1
    candidates: int = 1
    n_realizations: int = 1
    master_seed: int = 0
    scoring: str = "raw"            # "raw" | "normalized"
    facies_mode: str = "indicator"  # "indicator" | "raw_codes"
    min_cut: bool = False
    hard_data: Optional[HardDataSet] = None
    # literal-config extension (not in the reference; include/ccwgpu.h):
    # overlap / TI extents not divisible by 2^J, any-support coarse mask
    any_support: bool = False

    def block(self) -> int:
        return 1 << self.dwt_level

    def stride(self) -> int:
        return self.template_size - self.overlap

    def to_c(self) -> _abi.SimConfigC:
        sc = {"raw": 0, "normalized": 1}
        fm = {"indicator": 0, "raw_codes": 1, "raw-codes": 1}
        scoring = sc[self.scoring] if isinstance(self.scoring, str) else int(self.scoring)
        mode = fm[self.facies_mode] if isinstance(self.facies_mode, str) else int(self.facies_mode)
        return _abi.SimConfigC(self.sg_height, self.sg_width, self.template_size, self.overlap,
                               self.dwt_level, self.candidates, self.n_realizations, scoring, mode,
                               int(bool(self.min_cut)), int(self.master_seed) & _M64,
                               int(bool(self.any_support)), 0)

    def validate(self) -> None:
        c = self.to_c()
        buf = C.create_string_buffer(512)
        rc = _abi.lib().ccw_validate_config(C.byref(c), 0, 0, 0, None, 0, buf, 512)
        if rc:
            _raise(rc, buf.value.decode())

    def validate_against(self, ti: CategoricalGrid) -> None:
        c = self.to_c()
        hd = _hd_array(self.hard_data)
        buf = C.create_string_buffer(512)
        rc = _abi.lib().ccw_validate_config(
            C.byref(c), ti.height, ti.width, ti.num_facies,
            hd.ctypes.data_as(_abi.I32P) if hd is not None else None,
            0 if hd is None else hd.shape[0], buf, 512)
        if rc:
            _raise(rc, buf.value.decode())


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (ccw_nccl_unique_id), to broadcast to the
    ranks of a position-sharded simulation."""
    L = _abi.lib()
    buf = (C.c_uint8 * 128)()
    rc = L.ccw_nccl_unique_id(C.cast(buf, _abi.U8P))
    if rc:
        _raise(rc, L.ccw_last_error(None).decode())
    return bytes(buf)


# ----------------------------------------------------------------- device --

class Device:
    """One ccw_ctx: a GPU and a CUDA stream (not thread-safe)."""

    def __init__(self, device: int = 0):
        L = _abi.lib()
        h = C.c_void_p()
        rc = L.ccw_ctx_create(int(device), C.byref(h))
        if rc:
            _raise(rc, L.ccw_last_error(None).decode())
        self.handle = h
        self.index = int(device)
        self._lib = L
        _live_devices.add(self)

    def check(self, rc: int) -> None:
        if rc:
            _raise(rc, self._lib.ccw_last_error(self.handle).decode())

    @property
    def stream_ptr(self) -> int:
        return int(self._lib.ccw_ctx_stream(self.handle) or 0)

    def set_profiling(self, on: bool) -> None:
        self.check(self._lib.ccw_ctx_set_profiling(self.handle, int(bool(on))))

    def synchronize(self) -> None:
        """Wait for this context's asynchronous calls (ccw_ctx_synchronize) and raise
        the first error one of them reported."""
        self.check(self._lib.ccw_ctx_synchronize(self.handle))

    def last_timing(self) -> dict:
        t = _abi.TimingC()
        self.check(self._lib.ccw_ctx_last_timing(self.handle, C.byref(t)))
        return {k: getattr(t, k) for k, _ in _abi.TimingC._fields_}

    # production defaults of include/ccwgpu.h ccw_ctx_set_option
    OPTION_DEFAULTS = {"groups": 0, "sched_replay": 0, "norm_screen": 1, "shard_fast": 1,
                       "uniform": 1, "s16": 1, "bulk": 1, "help_min": 32, "stream_out": 1,
                       "pack": 1, "stream_bands": 6, "place_threads": 0,
                       "wave": 0, "wave_cs": 0, "flagprep": 1, "tc3d": 1}

    def set_option(self, name: str, value: int) -> None:
        """Per-context option (include/ccwgpu.h ccw_ctx_set_option)."""
        self.check(self._lib.ccw_ctx_set_option(self.handle, name.encode(), int(value)))

    @contextlib.contextmanager
    def options(self, **kw):
        """Set options for the duration of a with-block, then restore the defaults."""
        try:
            for k, v in kw.items():
                self.set_option(k, v)
            yield self
        finally:
            for k in kw:
                self.set_option(k, self.OPTION_DEFAULTS[k])

    def set_ccf_variant(self, variant: int) -> None:
        """0 auto (tcgen05 int8 when it is exact), 1 fp32 CUDA-core, 2 tcgen05 int8."""
        self.check(self._lib.ccw_ctx_set_ccf_variant(self.handle, int(variant)))

    def set_position_shards(self, nranks: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None,
                            virtual_shards: int = 1) -> None:
        """Candidate-position sharding (include/ccwgpu.h ccw_ctx_set_position_shards):
        this rank screens and ranks its share of the TI window positions and the
        shards' top-K lists are all-gathered (NCCL when nccl_id is given) and
        merged per placement.  nranks = virtual_shards = 1 switches it off."""
        idp = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("an NCCL unique id has 128 bytes")
            buf = (C.c_uint8 * 128).from_buffer_copy(bytes(nccl_id))
            idp = C.cast(buf, _abi.U8P)
        self.check(self._lib.ccw_ctx_set_position_shards(self.handle, int(nranks), int(rank), idp,
                                                         int(virtual_shards)))

    def measure_fp32_peak(self) -> float:
        """FP32 FFMA peak of this GPU in TFLOP/s (in-library microbenchmark)."""
        v = C.c_double(0)
        self.check(self._lib.ccw_measure_fp32_peak(self.handle, C.byref(v)))
        return v.value

    def measure_i8_peak(self) -> float:
        """Dense int8 tcgen05 rate (TOPS) of the screen's MMA shape."""
        v = C.c_double(0)
        self.check(self._lib.ccw_measure_i8_peak(self.handle, C.byref(v)))
        return v.value

    def measure_int_peak(self, kind: int) -> float:
        """CUDA-core integer rate (TOPS): kind 0 IMAD, 1 dp4a (the 3D screen's loops)."""
        v = C.c_double(0)
        self.check(self._lib.ccw_measure_int_peak(self.handle, int(kind), C.byref(v)))
        return v.value

    def close(self) -> None:
        if self.handle:
            # TI handles cached for this context go with it (the cache keys on
            # id(self), which a later Device may reuse)
            for per in list(_ti_cache.values()):
                for k in [k for k in per if k[1] == id(self)]:
                    per.pop(k).close()
            self._lib.ccw_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()
_live_devices: "weakref.WeakSet" = weakref.WeakSet()
_live_tis: "weakref.WeakSet" = weakref.WeakSet()


@atexit.register
def _shutdown() -> None:
    """Release device objects before the CUDA runtime unloads."""
    for t in list(_live_tis):
        t.close()
    for d in list(_live_devices):
        d.close()


def default_device(index: int = 0) -> Device:
    devs = getattr(_tls, "devices", None)
    if devs is None:
        devs = _tls.devices = {}
    if index not in devs:
        devs[index] = Device(index)
    return devs[index]


class TrainingImage:
    """A TI resident on the device with its level-J pyramid (ccw_ti)."""

    def __init__(self, ti: CategoricalGrid, levels: int, facies_mode="indicator",
                 device: Optional[Device] = None):
        self.device = device or default_device()
        self.grid = ti
        self.levels = int(levels)
        self.mode = {"indicator": 0, "raw_codes": 1, "raw-codes": 1}.get(facies_mode, facies_mode)
        h = C.c_void_p()
        cells = np.ascontiguousarray(ti.cells, np.uint8)
        self.device.check(self.device._lib.ccw_ti_create(
            self.device.handle, cells.ctypes.data_as(_abi.U8P), ti.height, ti.width,
            ti.num_facies, self.levels, int(self.mode), C.byref(h)))
        self.handle = h
        _live_tis.add(self)

    def apex(self) -> np.ndarray:
        nch = self.grid.num_facies if self.mode == 0 else 1
        out = np.zeros((nch, self.grid.height >> self.levels, self.grid.width >> self.levels))
        self.device.check(self.device._lib.ccw_ti_apex(self.handle, out.ctypes.data_as(_abi.F64P)))
        return out

    def close(self) -> None:
        if self.handle:
            self.device._lib.ccw_ti_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_ti_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _ti_handle(ti: CategoricalGrid, cfg: SimConfig, device: Optional[Device]) -> TrainingImage:
    dev = device or default_device()
    mode = cfg.to_c().facies_mode
    per = _ti_cache.setdefault(ti, {})
    key = (dev.index, id(dev), cfg.dwt_level, mode)
    h = per.get(key)
    if h is None:
        h = TrainingImage(ti, cfg.dwt_level, mode, dev)
        per[key] = h
    return h


# ---------------------------------------------------------------- wavelet --

@dataclass
class SingleLevelDwt:
    approx: np.ndarray
    detail_h: np.ndarray
    detail_v: np.ndarray
    detail_d: np.ndarray


@dataclass
class SubbandSet:
    detail_h: np.ndarray
    detail_v: np.ndarray
    detail_d: np.ndarray


@dataclass
class WaveletPyramid:
    levels: int
    original_height: int
    original_width: int
    apex: np.ndarray
    details: List[SubbandSet]


def _plane(p) -> np.ndarray:
    a = np.ascontiguousarray(p, np.float64)
    if a.ndim != 2 or a.shape[0] <= 0 or a.shape[1] <= 0:
        raise DimensionError("plane dimensions must be positive")
    if not np.all(np.isfinite(a)):
        raise StructureError("plane values must be finite")
    return a


def _f64(a):
    return a.ctypes.data_as(_abi.F64P)


def dwt2_single(plane, device: Optional[Device] = None) -> SingleLevelDwt:
    """wavelet.hpp:69-106."""
    dev = device or default_device()
    x = _plane(plane)
    h, w = x.shape
    outs = [np.zeros((max(h // 2, 1), max(w // 2, 1))) for _ in range(4)]
    dev.check(dev._lib.ccw_dwt2_single_f64(dev.handle, _f64(x), h, w, *[_f64(o) for o in outs]))
    return SingleLevelDwt(*outs)


def idwt2_single(approx, detail_h, detail_v, detail_d,
                 device: Optional[Device] = None) -> np.ndarray:
    """wavelet.hpp:108-143."""
    dev = device or default_device()
    a, dh, dv, dd = (_plane(p) for p in (approx, detail_h, detail_v, detail_d))
    if not (a.shape == dh.shape == dv.shape == dd.shape):
        raise StructureError("subband sizes disagree")
    out = np.zeros((2 * a.shape[0], 2 * a.shape[1]))
    dev.check(dev._lib.ccw_idwt2_single_f64(dev.handle, _f64(a), _f64(dh), _f64(dv), _f64(dd),
                                            a.shape[0], a.shape[1], _f64(out)))
    return out


def dwt2(plane, levels: int, device: Optional[Device] = None) -> WaveletPyramid:
    """wavelet.hpp:147-171."""
    dev = device or default_device()
    x = _plane(plane)
    h, w = x.shape
    if levels < 1:
        raise DimensionError("decomposition level must be >= 1")
    if levels > 30 or h % (1 << levels) or w % (1 << levels):
        raise DimensionError(f"plane {h}x{w} not divisible by 2^{levels}")
    apex = np.zeros((h >> levels, w >> levels))
    nd = sum(3 * (h >> j) * (w >> j) for j in range(1, levels + 1))
    det = np.zeros(nd)
    dev.check(dev._lib.ccw_dwt2_f64(dev.handle, _f64(x), h, w, levels, _f64(apex), _f64(det)))
    details, off = [], 0
    for j in range(1, levels + 1):
        ph, pw = h >> j, w >> j
        n = ph * pw
        details.append(SubbandSet(*(det[off + i * n: off + (i + 1) * n].reshape(ph, pw).copy()
                                    for i in range(3))))
        off += 3 * n
    return WaveletPyramid(levels, h, w, apex, details)


def idwt2(pyr: WaveletPyramid, device: Optional[Device] = None) -> np.ndarray:
    """wavelet.hpp:174-191."""
    dev = device or default_device()
    L = pyr.levels
    if L < 1 or len(pyr.details) != L:
        raise StructureError("pyramid level count inconsistent")
    h, w = pyr.original_height, pyr.original_width
    if np.shape(pyr.apex) != (h >> L, w >> L):
        raise StructureError("apex size does not match original/2^levels")
    for j in range(L, 0, -1):
        sb = pyr.details[j - 1]
        if np.shape(sb.detail_h) != (h >> j, w >> j):
            raise StructureError(f"level {j} subband size inconsistent")
        if np.shape(sb.detail_v) != (h >> j, w >> j) or np.shape(sb.detail_d) != (h >> j, w >> j):
            raise StructureError("subband sizes disagree")
    packed = np.concatenate([np.ravel(_plane(p)) for sb in pyr.details
                             for p in (sb.detail_h, sb.detail_v, sb.detail_d)])
    apex = _plane(pyr.apex)
    out = np.zeros((h, w))
    dev.check(dev._lib.ccw_idwt2_f64(dev.handle, _f64(apex), _f64(packed), h, w, L, _f64(out)))
    return out


def coarse_to_fine(coord, levels: int):
    """wavelet.hpp:197-199."""
    return (coord[0] << levels, coord[1] << levels)


# ---------------------------------------------------------------- matcher --

@dataclass
class ScoreMap:
    scores: np.ndarray


@dataclass
class Candidate:
    row: int = 0
    col: int = 0
    score: float = 0.0


@dataclass
class CandidateSet:
    entries: List[Candidate] = field(default_factory=list)

    def empty(self) -> bool:
        return not self.entries

    def size(self) -> int:
        return len(self.entries)


@dataclass
class ConditionalPick:
    candidate: Candidate
    mismatches: int = 0


def ccw_score_map_channels(ti_channels: Sequence, or_channels: Sequence, or_mask,
                           mode: str = "raw", device: Optional[Device] = None) -> ScoreMap:
    """matcher.hpp:147-173."""
    dev = device or default_device()
    if len(ti_channels) == 0 or len(ti_channels) != len(or_channels):
        raise StructureError("channel counts disagree")
    tis = [_plane(p) for p in ti_channels]
    ors = [_plane(p) for p in or_channels]
    mask = _plane(or_mask)
    for t, o in zip(tis, ors):
        if mask.shape != o.shape:
            raise StructureError(f"mask size {mask.shape[0]}x{mask.shape[1]} does not match "
                                 f"template {o.shape[0]}x{o.shape[1]}")
        if t.shape != tis[0].shape or o.shape != ors[0].shape:
            raise StructureError("channel plane sizes disagree")
    ti = np.ascontiguousarray(np.stack(tis))
    tm = np.ascontiguousarray(np.stack(ors))
    th, tw = tm.shape[1:]
    if th > ti.shape[1] or tw > ti.shape[2]:
        raise DimensionError(f"template {th}x{tw} larger than TI coefficients "
                             f"{ti.shape[1]}x{ti.shape[2]}")
    out = np.zeros((ti.shape[1] - th + 1, ti.shape[2] - tw + 1))
    scoring = {"raw": 0, "normalized": 1}[mode] if isinstance(mode, str) else int(mode)
    dev.check(dev._lib.ccw_score_map_f64(dev.handle, _f64(ti), _f64(tm), ti.shape[0], ti.shape[1],
                                         ti.shape[2], th, tw, _f64(mask), scoring, _f64(out)))
    return ScoreMap(out)


def ccw_score_map(ti_approx, or_approx, or_mask, device: Optional[Device] = None) -> ScoreMap:
    """matcher.hpp:132-141."""
    return ccw_score_map_channels([ti_approx], [or_approx], or_mask, "raw", device)


def top_k(score_map: ScoreMap, k: int, device: Optional[Device] = None) -> CandidateSet:
    """matcher.hpp:177-204."""
    dev = device or default_device()
    s = score_map.scores
    if s is None or np.size(s) == 0:
        raise EmptyInputError("top_k on empty score map")
    if k < 1:
        raise ConfigError("candidate count must be >= 1")
    s = np.ascontiguousarray(s, np.float64)
    kk = min(int(k), s.size)
    rows = np.zeros(kk, np.int32)
    cols = np.zeros(kk, np.int32)
    vals = np.zeros(kk)
    n = C.c_int(0)
    dev.check(dev._lib.ccw_top_k_f64(dev.handle, _f64(s), s.shape[0], s.shape[1], int(k),
                                     rows.ctypes.data_as(_abi.I32P), cols.ctypes.data_as(_abi.I32P),
                                     _f64(vals), C.byref(n)))
    return CandidateSet([Candidate(int(r), int(c), float(v))
                         for r, c, v in zip(rows[:n.value], cols[:n.value], vals[:n.value])])


def select_unconditional(cands: CandidateSet, rng: Mt19937_64) -> Candidate:
    """matcher.hpp:207-211 (host: an index draw)."""
    if cands.empty():
        raise EmptyInputError("select_unconditional on empty candidate set")
    return cands.entries[bounded(rng, len(cands.entries))]


def select_conditional(cands: CandidateSet, hd_in_footprint, ti: CategoricalGrid, levels: int,
                       device: Optional[Device] = None) -> ConditionalPick:
    """matcher.hpp:222-241."""
    dev = device or default_device()
    if cands.empty():
        raise EmptyInputError("select_conditional on empty candidate set")
    rows = np.array([c.row for c in cands.entries], np.int32)
    cols = np.array([c.col for c in cands.entries], np.int32)
    hd = _hd_array(hd_in_footprint)
    if hd is None or hd.size == 0:
        hd = np.zeros((0, 3), np.int32)
    cells = np.ascontiguousarray(ti.cells, np.uint8)
    pick, mis = C.c_int(0), C.c_int(0)
    dev.check(dev._lib.ccw_select_conditional(
        dev.handle, rows.ctypes.data_as(_abi.I32P), cols.ctypes.data_as(_abi.I32P), len(rows),
        hd.ctypes.data_as(_abi.I32P) if hd.size else None, hd.shape[0],
        cells.ctypes.data_as(_abi.U8P), ti.height, ti.width, int(levels), C.byref(pick),
        C.byref(mis)))
    return ConditionalPick(cands.entries[pick.value], mis.value)


# -------------------------------------------------------------- simulator --

OR_NONE, OR_VERTICAL, OR_HORIZONTAL, OR_L = 0, 1, 2, 3
TOP_LEFT, TOP_RIGHT, BOTTOM_LEFT, BOTTOM_RIGHT = 0, 1, 2, 3
CORNER_NAMES = ["top_left", "top_right", "bottom_left", "bottom_right"]


@dataclass
class Placement:
    top: int = 0
    left: int = 0
    or_shape: int = OR_NONE


@dataclass
class PlacementPlan:
    origin: int = TOP_LEFT
    column_major: bool = False
    work_height: int = 0
    work_width: int = 0
    placements: List[Placement] = field(default_factory=list)

    def vertical_on_left(self) -> bool:
        return self.origin in (TOP_LEFT, BOTTOM_LEFT)

    def horizontal_on_top(self) -> bool:
        return self.origin in (TOP_LEFT, TOP_RIGHT)


def plan_raster_path(cfg: SimConfig, rng: Mt19937_64) -> PlacementPlan:
    """simulator.hpp:148-190 (consumes exactly two draws from rng)."""
    cfg.validate()
    origin = bounded(rng, 4)
    column_major = bounded(rng, 2) == 1
    c = cfg.to_c()
    t, s = cfg.template_size, cfg.stride()
    cap = ((cfg.sg_height + s) // s + 2) * ((cfg.sg_width + s) // s + 2)
    tops = np.zeros(cap, np.int32)
    lefts = np.zeros(cap, np.int32)
    shapes = np.zeros(cap, np.int32)
    wh, ww, n = C.c_int(0), C.c_int(0), C.c_int(0)
    buf = C.create_string_buffer(512)
    rc = _abi.lib().ccw_plan_raster_path(C.byref(c), origin, int(column_major), C.byref(wh),
                                         C.byref(ww), tops.ctypes.data_as(_abi.I32P),
                                         lefts.ctypes.data_as(_abi.I32P),
                                         shapes.ctypes.data_as(_abi.I32P), cap, C.byref(n), buf, 512)
    if rc:
        _raise(rc, buf.value.decode())
    del t
    return PlacementPlan(origin, column_major, wh.value, ww.value,
                         [Placement(int(a), int(b), int(sh))
                          for a, b, sh in zip(tops[:n.value], lefts[:n.value], shapes[:n.value])])


@dataclass
class OrGeometry:
    shape: int = OR_NONE
    vertical_on_left: bool = True
    horizontal_on_top: bool = True
    overlap: int = 0


def min_cut_stitch(existing: CategoricalGrid, incoming: CategoricalGrid, geom: OrGeometry,
                   device: Optional[Device] = None) -> CategoricalGrid:
    """simulator.hpp:328-374."""
    dev = device or default_device()
    if existing.height != incoming.height or existing.width != incoming.width:
        raise StructureError("existing and incoming patch sizes disagree")
    if geom.shape == OR_NONE:
        return incoming
    t = incoming.height
    if incoming.width != t:
        raise StructureError("stitching needs square patches")
    if geom.overlap < 1 or geom.overlap >= t:
        raise StructureError("overlap band width out of range")
    e = np.ascontiguousarray(existing.cells, np.uint8)
    i = np.ascontiguousarray(incoming.cells, np.uint8)
    out = np.zeros_like(i)
    dev.check(dev._lib.ccw_min_cut_stitch(dev.handle, e.ctypes.data_as(_abi.U8P),
                                          i.ctypes.data_as(_abi.U8P), t, int(geom.shape),
                                          int(bool(geom.vertical_on_left)),
                                          int(bool(geom.horizontal_on_top)), int(geom.overlap),
                                          out.ctypes.data_as(_abi.U8P)))
    return CategoricalGrid(t, t, incoming.num_facies, out)


@dataclass
class SimDiagnostics:
    seed: int = 0
    origin: int = TOP_LEFT
    column_major: bool = False
    work_height: int = 0
    work_width: int = 0
    placement_count: int = 0
    hard_data_count: int = 0
    pre_overwrite_mismatches: int = 0
    wall_seconds: float = 0.0

    def pre_overwrite_mismatch_rate(self) -> float:
        return (self.pre_overwrite_mismatches / self.hard_data_count
                if self.hard_data_count > 0 else 0.0)


@dataclass
class PasteEvent:
    placement: Placement
    ti_row: int
    ti_col: int
    pasted: CategoricalGrid


@dataclass
class SimTrace:
    events: List[PasteEvent] = field(default_factory=list)


@dataclass
class SimResult:
    realization: CategoricalGrid
    diagnostics: SimDiagnostics


def _diag(d: _abi.DiagC) -> SimDiagnostics:
    return SimDiagnostics(int(d.seed), int(d.origin), bool(d.column_major), d.work_height,
                          d.work_width, d.placement_count, d.hard_data_count,
                          d.pre_overwrite_mismatches, d.wall_seconds)


def simulate_batch(ti: CategoricalGrid, cfg: SimConfig, seeds: Sequence[int],
                   traces: Optional[List[SimTrace]] = None,
                   device: Optional[Device] = None) -> List[SimResult]:
    """Batched simulate_one: realization r uses seeds[r]; one device call."""
    cfg.validate_against(ti)
    h = _ti_handle(ti, cfg, device)
    dev = h.device
    n = len(seeds)
    if n < 1:
        raise ConfigError("realizations: must be >= 1")
    c = cfg.to_c()
    hd = _hd_array(cfg.hard_data)
    seeds_a = np.array([int(s) & _M64 for s in seeds], np.uint64)
    out = np.zeros((n, cfg.sg_height, cfg.sg_width), np.uint8)
    diags = (_abi.DiagC * n)()
    tr_c = None
    keep = []
    if traces is not None:
        t = cfg.template_size
        cap = ((cfg.sg_height + cfg.stride()) // cfg.stride() + 2) * \
              ((cfg.sg_width + cfg.stride()) // cfg.stride() + 2)
        tr_c = (_abi.TraceC * n)()
        for r in range(n):
            arrs = [np.zeros(cap, np.int32) for _ in range(5)] + [np.zeros(cap * t * t, np.uint8)]
            keep.append(arrs)
            tr_c[r] = _abi.TraceC(cap, 0, *[a.ctypes.data_as(_abi.I32P) for a in arrs[:5]],
                                  arrs[5].ctypes.data_as(_abi.U8P))
    dev.check(dev._lib.ccw_simulate(
        dev.handle, h.handle, C.byref(c), seeds_a.ctypes.data_as(_abi.U64P), n,
        hd.ctypes.data_as(_abi.I32P) if hd is not None else None, 0 if hd is None else hd.shape[0],
        out.ctypes.data_as(_abi.U8P), diags, tr_c))
    results = [SimResult(CategoricalGrid._trusted(out[r], ti.num_facies), _diag(diags[r]))
               for r in range(n)]
    if traces is not None:
        t = cfg.template_size
        for r in range(n):
            arrs = keep[r]
            cnt = tr_c[r].count
            traces[r].events = [
                PasteEvent(Placement(int(arrs[0][e]), int(arrs[1][e]), int(arrs[2][e])),
                           int(arrs[3][e]), int(arrs[4][e]),
                           CategoricalGrid(t, t, ti.num_facies,
                                           arrs[5][e * t * t:(e + 1) * t * t].reshape(t, t)))
                for e in range(cnt)]
    return results


def simulate_one(ti: CategoricalGrid, cfg: SimConfig, seed: int,
                 trace: Optional[SimTrace] = None, device: Optional[Device] = None) -> SimResult:
    """simulator.hpp:418-519."""
    traces = [trace] if trace is not None else None
    return simulate_batch(ti, cfg, [seed], traces, device)[0]


def simulate_ensemble(ti: CategoricalGrid, cfg: SimConfig, workers: int = 1,
                      device: Optional[Device] = None) -> List[SimResult]:
    """simulator.hpp:523-566: realization r uses mix64(master, r + 1); results
    ordered by r.  All realizations run in one batched device call, so
    ``workers`` has no effect (the reference guarantees worker-count-invariant
    output, so this is observably identical)."""
    seeds = [mix64(cfg.master_seed, r + 1) for r in range(cfg.n_realizations)]
    return simulate_batch(ti, cfg, seeds, None, device)  # (validates)
