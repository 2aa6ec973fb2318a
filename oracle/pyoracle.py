"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

- ``restatement()``: oracle/_build/libccworacle.so, the C restatement
  (ccw_oracle.c) of the reference hot path;
- ``reference()``:   oracle/_ref/libccwref.so, the unmodified reference
  headers behind ref_driver.cpp.

Both expose the same Python surface so tests can run one against the other.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "_build", "libccworacle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libccwref.so")

ERROR_NAMES = {1: "BoundsError", 2: "DimensionError", 3: "StructureError",
               4: "ConfigError", 5: "EmptyInputError", 6: "IoError", 7: "Error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERROR_NAMES.get(code, "Error")
        self.msg = msg


class SimConfigC(C.Structure):
    _fields_ = [("sg_height", C.c_int32), ("sg_width", C.c_int32),
                ("template_size", C.c_int32), ("overlap", C.c_int32),
                ("dwt_level", C.c_int32), ("candidates", C.c_int32),
                ("n_realizations", C.c_int32), ("scoring", C.c_int32),
                ("facies_mode", C.c_int32), ("min_cut", C.c_int32),
                ("master_seed", C.c_uint64), ("any_support", C.c_int32), ("_pad", C.c_int32)]


class DiagC(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("origin", C.c_int32), ("column_major", C.c_int32),
                ("work_height", C.c_int32), ("work_width", C.c_int32),
                ("placement_count", C.c_int32), ("hard_data_count", C.c_int32),
                ("pre_overwrite_mismatches", C.c_int32), ("_pad", C.c_int32),
                ("wall_seconds", C.c_double)]


class TraceC(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("count", C.c_int32),
                ("top", C.POINTER(C.c_int32)), ("left", C.POINTER(C.c_int32)),
                ("shape", C.POINTER(C.c_int32)), ("ti_row", C.POINTER(C.c_int32)),
                ("ti_col", C.POINTER(C.c_int32)), ("pasted", C.POINTER(C.c_uint8))]


def config_struct(cfg) -> SimConfigC:
    def mode(v, names):
        if isinstance(v, str):
            return names.index(v)
        return int(v)
    return SimConfigC(int(cfg.sg_height), int(cfg.sg_width), int(cfg.template_size),
                      int(cfg.overlap), int(cfg.dwt_level), int(cfg.candidates),
                      int(cfg.n_realizations), mode(cfg.scoring, ["raw", "normalized"]),
                      mode(cfg.facies_mode, ["indicator", "raw_codes"]), int(bool(cfg.min_cut)),
                      int(cfg.master_seed) & 0xFFFFFFFFFFFFFFFF,
                      int(bool(getattr(cfg, "any_support", False))), 0)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _hd_array(hd):
    if hd is None:
        return None, 0
    arr = np.ascontiguousarray(np.asarray(hd, dtype=np.int32).reshape(-1, 3))
    return arr, int(arr.shape[0])


def diag_dict(d: DiagC) -> dict:
    return {k: getattr(d, k) for k, _ in DiagC._fields_ if k != "_pad"}


def build(quiet: bool = True) -> None:
    """Compile both checkers (``make -C oracle``)."""
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class CpuImpl:
    """One CPU implementation (restatement or reference) behind a common API."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.path = path
        self.lib = C.CDLL(path)
        self.prefix = prefix
        getattr(self.lib, prefix + "last_error").restype = C.c_char_p
        getattr(self.lib, prefix + "mix64").restype = C.c_uint64
        getattr(self.lib, prefix + "mix64").argtypes = [C.c_uint64, C.c_uint64]

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._fn("last_error")().decode())

    # -- rng ---------------------------------------------------------------
    def mix64(self, seed, index):
        return int(self._fn("mix64")(C.c_uint64(seed & (2**64 - 1)), C.c_uint64(index)))

    def mt64_draws(self, seed, n):
        out = np.zeros(n, np.uint64)
        self._fn("mt64_draws")(C.c_uint64(seed), _p(out, C.c_uint64), C.c_int(n))
        return out

    def bounded_draws(self, seed, ns):
        ns = np.ascontiguousarray(ns, np.uint64)
        out = np.zeros(len(ns), np.uint64)
        self._fn("bounded_draws")(C.c_uint64(seed), _p(ns, C.c_uint64), _p(out, C.c_uint64),
                                  C.c_int(len(ns)))
        return out

    # -- wavelet -----------------------------------------------------------
    def dwt2_single(self, plane):
        x = np.ascontiguousarray(plane, np.float64)
        h, w = x.shape
        outs = [np.zeros((max(h // 2, 1), max(w // 2, 1))) for _ in range(4)]
        self._check(self._fn("dwt2_single")(_p(x, C.c_double), h, w,
                                            *[_p(o, C.c_double) for o in outs]))
        return tuple(outs)

    def idwt2_single(self, a, dh, dv, dd):
        a, dh, dv, dd = (np.ascontiguousarray(v, np.float64) for v in (a, dh, dv, dd))
        hh, hw = a.shape
        out = np.zeros((2 * hh, 2 * hw))
        self._check(self._fn("idwt2_single")(_p(a, C.c_double), _p(dh, C.c_double),
                                             _p(dv, C.c_double), _p(dd, C.c_double), hh, hw,
                                             _p(out, C.c_double)))
        return out

    def dwt2(self, plane, levels):
        """Returns (apex, details) with details[j-1] = (H, V, D) of level j."""
        x = np.ascontiguousarray(plane, np.float64)
        h, w = x.shape
        levels = int(levels)
        ah, aw = (h >> levels, w >> levels) if 0 < levels < 31 else (1, 1)
        apex = np.zeros((max(ah, 1), max(aw, 1)))
        nd = sum(3 * (h >> j) * (w >> j) for j in range(1, levels + 1)) if 0 < levels < 31 else 0
        det = np.zeros(max(nd, 1))
        self._check(self._fn("dwt2")(_p(x, C.c_double), h, w, levels, _p(apex, C.c_double),
                                     _p(det, C.c_double)))
        details, off = [], 0
        for j in range(1, levels + 1):
            ph, pw = h >> j, w >> j
            n = ph * pw
            details.append(tuple(det[off + i * n: off + (i + 1) * n].reshape(ph, pw)
                                 for i in range(3)))
            off += 3 * n
        return apex, details

    def idwt2(self, apex, details, h, w, levels):
        packed = np.concatenate([np.ravel(p) for lvl in details for p in lvl]).astype(np.float64)
        apex = np.ascontiguousarray(apex, np.float64)
        out = np.zeros((h, w))
        self._check(self._fn("idwt2")(_p(apex, C.c_double), _p(packed, C.c_double), h, w, levels,
                                      _p(out, C.c_double)))
        return out

    # -- matcher -----------------------------------------------------------
    def score_map_channels(self, ti, tmpl, mask, scoring=0):
        ti = np.ascontiguousarray(ti, np.float64)
        tmpl = np.ascontiguousarray(tmpl, np.float64)
        if ti.ndim == 2:
            ti, tmpl = ti[None], tmpl[None]
        mask = np.ascontiguousarray(mask, np.float64)
        nch, th_, tw_ = ti.shape[0], tmpl.shape[1], tmpl.shape[2]
        oh, ow = ti.shape[1] - th_ + 1, ti.shape[2] - tw_ + 1
        out = np.zeros((max(oh, 1), max(ow, 1)))
        self._check(self._fn("score_map_channels")(
            _p(ti, C.c_double), _p(tmpl, C.c_double), nch, ti.shape[1], ti.shape[2], th_, tw_,
            _p(mask, C.c_double), int(scoring), _p(out, C.c_double)))
        return out

    def top_k(self, scores, k):
        s = np.ascontiguousarray(scores, np.float64)
        h, w = s.shape if s.ndim == 2 else (0, 0)
        cap = max(int(k), 1)
        rows = np.zeros(cap, np.int32)
        cols = np.zeros(cap, np.int32)
        vals = np.zeros(cap)
        n = C.c_int(0)
        self._check(self._fn("top_k")(_p(s, C.c_double) if s.size else None, h, w, int(k),
                                      _p(rows, C.c_int32), _p(cols, C.c_int32),
                                      _p(vals, C.c_double), C.byref(n)))
        m = n.value
        return list(zip(rows[:m].tolist(), cols[:m].tolist(), vals[:m].tolist()))

    def select_conditional(self, cands, hd_local, ti, levels):
        rows = np.array([c[0] for c in cands], np.int32)
        cols = np.array([c[1] for c in cands], np.int32)
        vals = np.array([c[2] for c in cands], np.float64)
        hd, n_hd = _hd_array(hd_local)
        if hd is None:
            hd = np.zeros((1, 3), np.int32)
        ti = np.ascontiguousarray(ti, np.uint8)
        pick, mis = C.c_int(0), C.c_int(0)
        self._check(self._fn("select_conditional")(
            _p(rows, C.c_int32), _p(cols, C.c_int32), _p(vals, C.c_double), len(cands),
            _p(hd, C.c_int32), n_hd, _p(ti, C.c_uint8), ti.shape[0], ti.shape[1], int(levels),
            C.byref(pick), C.byref(mis)))
        return pick.value, mis.value

    # -- simulator ---------------------------------------------------------
    def plan_raster_path(self, cfg, seed):
        cs = config_struct(cfg)
        cap = 1 << 20
        tops = np.zeros(cap, np.int32)
        lefts = np.zeros(cap, np.int32)
        shapes = np.zeros(cap, np.int32)
        o, cm, wh, ww, n = (C.c_int(0) for _ in range(5))
        self._check(self._fn("plan_raster_path")(
            C.byref(cs), C.c_uint64(seed), C.byref(o), C.byref(cm), C.byref(wh), C.byref(ww),
            _p(tops, C.c_int32), _p(lefts, C.c_int32), _p(shapes, C.c_int32), cap, C.byref(n)))
        m = n.value
        return {"origin": o.value, "column_major": bool(cm.value), "work_height": wh.value,
                "work_width": ww.value, "tops": tops[:m].copy(), "lefts": lefts[:m].copy(),
                "shapes": shapes[:m].copy()}

    def min_cost_seam(self, cost):
        c = np.ascontiguousarray(cost, np.int32)
        seam = np.zeros(c.shape[0], np.int32)
        self._check(self._fn("min_cost_seam")(_p(c, C.c_int32), c.shape[0], c.shape[1],
                                              _p(seam, C.c_int32)))
        return seam

    def min_cut_stitch(self, existing, incoming, shape, vertical_on_left, horizontal_on_top,
                       overlap):
        e = np.ascontiguousarray(existing, np.uint8)
        i = np.ascontiguousarray(incoming, np.uint8)
        out = np.zeros_like(i)
        self._check(self._fn("min_cut_stitch")(
            _p(e, C.c_uint8), _p(i, C.c_uint8), i.shape[0], int(shape), int(vertical_on_left),
            int(horizontal_on_top), int(overlap), _p(out, C.c_uint8)))
        return out

    def simulate_one(self, ti, num_facies, cfg, hard_data=None, seed=0, trace=False):
        ti = np.ascontiguousarray(ti, np.uint8)
        cs = config_struct(cfg)
        hd, n_hd = _hd_array(hard_data)
        out = np.zeros((cfg.sg_height, cfg.sg_width), np.uint8)
        diag = DiagC()
        tr = None
        arrays = None
        if trace:
            t = cfg.template_size
            cap = 1 << 16
            arrays = [np.zeros(cap, np.int32) for _ in range(5)] + [np.zeros(cap * t * t, np.uint8)]
            tr = TraceC(cap, 0, *[_p(a, C.c_int32) for a in arrays[:5]], _p(arrays[5], C.c_uint8))
        self._check(self._fn("simulate_one")(
            _p(ti, C.c_uint8), ti.shape[0], ti.shape[1], int(num_facies), C.byref(cs),
            _p(hd, C.c_int32) if hd is not None else None, n_hd, C.c_uint64(seed),
            _p(out, C.c_uint8), C.byref(diag), C.byref(tr) if tr is not None else None))
        res = {"realization": out, "diagnostics": diag_dict(diag)}
        if trace:
            n = tr.count
            t = cfg.template_size
            res["trace"] = {"top": arrays[0][:n].copy(), "left": arrays[1][:n].copy(),
                            "shape": arrays[2][:n].copy(), "ti_row": arrays[3][:n].copy(),
                            "ti_col": arrays[4][:n].copy(),
                            "pasted": arrays[5][: n * t * t].reshape(n, t, t).copy()}
        return res

    def simulate_ensemble(self, ti, num_facies, cfg, hard_data=None, workers=1):
        ti = np.ascontiguousarray(ti, np.uint8)
        cs = config_struct(cfg)
        hd, n_hd = _hd_array(hard_data)
        n = int(cfg.n_realizations)
        out = np.zeros((max(n, 1), cfg.sg_height, cfg.sg_width), np.uint8)
        diags = (DiagC * max(n, 1))()
        self._check(self._fn("simulate_ensemble")(
            _p(ti, C.c_uint8), ti.shape[0], ti.shape[1], int(num_facies), C.byref(cs),
            _p(hd, C.c_int32) if hd is not None else None, n_hd, int(workers),
            _p(out, C.c_uint8), diags))
        return out[:n], [diag_dict(d) for d in diags[:n]]


class RefImpl(CpuImpl):
    """The compiled reference, plus its test-support fixture generators."""

    def make_channel_ti(self, h, w, seed):
        out = np.zeros((h, w), np.uint8)
        self.lib.ccwr_make_channel_ti(h, w, C.c_uint64(seed), _p(out, C.c_uint8))
        return out

    def random_grid(self, h, w, nf, seed):
        out = np.zeros((h, w), np.uint8)
        self.lib.ccwr_random_grid(h, w, nf, C.c_uint64(seed), _p(out, C.c_uint8))
        return out

    def random_plane(self, h, w, seed):
        out = np.zeros((h, w))
        self.lib.ccwr_random_plane(h, w, C.c_uint64(seed), _p(out, C.c_double))
        return out


_cache: dict = {}


def restatement() -> CpuImpl:
    if "o" not in _cache:
        _cache["o"] = CpuImpl(RESTATEMENT_SO, "ccwo_")
    return _cache["o"]


def reference() -> RefImpl:
    if "r" not in _cache:
        _cache["r"] = RefImpl(REFERENCE_SO, "ccwr_")
    return _cache["r"]


def reference_available() -> bool:
    return os.path.exists(REFERENCE_SO)


@dataclass
class Cfg:
    """Minimal SimConfig stand-in for oracle-only callers."""
    sg_height: int = 64
    sg_width: int = 64
    template_size: int = 16
    overlap: int = 4
    dwt_level: int = 2
    candidates: int = 4
    n_realizations: int = 1
    scoring: int = 0
    facies_mode: int = 0
    min_cut: bool = False
    master_seed: int = 1234
    any_support: bool = False  # literal-config extension (ccw_oracle.h)
