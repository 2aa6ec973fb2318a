"""ctypes binding of the metrics restatement (oracle/ccw_metrics_oracle.c in
_build/libccworacle.so).  TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libccworacle.so")
_L = None


def _lib():
    global _L
    if _L is None:
        _L = C.CDLL(SO)
        _L.ccwm_js_divergence.restype = C.c_double
    return _L


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def variogram(g, facies, direction, max_lag):
    g = np.ascontiguousarray(g, np.uint8)
    out = np.zeros(max_lag, np.float64)
    present = _lib().ccwm_variogram(_p(g, C.c_uint8), g.shape[0], g.shape[1], int(facies), int(direction),
                                    int(max_lag), _p(out, C.c_double))
    return out, bool(present)


def connectivity(g, facies, direction, max_lag):
    g = np.ascontiguousarray(g, np.uint8)
    out = np.zeros(max_lag, np.float64)
    _lib().ccwm_connectivity(_p(g, C.c_uint8), g.shape[0], g.shape[1], int(facies), int(direction), int(max_lag),
                             _p(out, C.c_double))
    return out


def ensemble_average(grids, facies):
    a = np.ascontiguousarray(grids, np.uint8)
    out = np.zeros(a.shape[1:], np.float64)
    _lib().ccwm_ensemble_average(_p(a, C.c_uint8), a.shape[0], a.shape[1], a.shape[2], int(facies),
                                 _p(out, C.c_double))
    return out


def pattern_histogram(g, win, stride=1):
    """(sorted list of (key bytes, count), total)."""
    g = np.ascontiguousarray(g, np.uint8)
    nwin = ((g.shape[0] - win) // stride + 1) * ((g.shape[1] - win) // stride + 1)
    keys = np.zeros(max(nwin, 1) * win * win, np.uint8)
    counts = np.zeros(max(nwin, 1), np.uint64)
    total = C.c_uint64()
    nd = _lib().ccwm_pattern_histogram(_p(g, C.c_uint8), g.shape[0], g.shape[1], int(win), int(stride),
                                       _p(keys, C.c_uint8), _p(counts, C.c_uint64), C.byref(total))
    kw = win * win
    return [(keys[i * kw:(i + 1) * kw].tobytes(), int(counts[i])) for i in range(nd)], total.value


def js_divergence(ph, qh, win):
    """ph / qh: (sorted list of (key, count), total) from pattern_histogram."""
    (pl, pt), (ql, qt) = ph, qh
    kw = win * win
    pk = np.frombuffer(b"".join(k for k, _ in pl), np.uint8) if pl else np.zeros(kw, np.uint8)
    qk = np.frombuffer(b"".join(k for k, _ in ql), np.uint8) if ql else np.zeros(kw, np.uint8)
    pk, qk = np.ascontiguousarray(pk), np.ascontiguousarray(qk)
    pc = np.array([c for _, c in pl] or [0], np.uint64)
    qc = np.array([c for _, c in ql] or [0], np.uint64)
    return _lib().ccwm_js_divergence(_p(pk, C.c_uint8), _p(pc, C.c_uint64), len(pl), C.c_uint64(pt),
                                     _p(qk, C.c_uint8), _p(qc, C.c_uint64), len(ql), C.c_uint64(qt), kw)


def downsample_majority(g, nf, factor):
    g = np.ascontiguousarray(g, np.uint8)
    out = np.zeros((g.shape[0] // factor, g.shape[1] // factor), np.uint8)
    _lib().ccwm_downsample_majority(_p(g, C.c_uint8), g.shape[0], g.shape[1], int(nf), int(factor),
                                    _p(out, C.c_uint8))
    return out


def anodi(ens_a, ens_b, ti, nf, levels, window, weights=None):
    """metrics.hpp:318-384 (no MDS): (levels x 8 array, aggregate); raises
    RuntimeError with the reference's error class name on failure."""
    a = np.ascontiguousarray(ens_a, np.uint8)
    b = np.ascontiguousarray(ens_b, np.uint8)
    t = np.ascontiguousarray(ti, np.uint8)
    out = np.zeros((max(levels, 1), 8), np.float64)
    agg = C.c_double()
    w = np.ascontiguousarray(weights, np.float64) if weights is not None else None
    rc = _lib().ccwm_anodi(_p(a, C.c_uint8), a.shape[0], _p(b, C.c_uint8), b.shape[0], a.shape[1], a.shape[2],
                           _p(t, C.c_uint8), t.shape[0], t.shape[1], int(nf), int(levels), int(window),
                           _p(w, C.c_double) if w is not None else None, _p(out, C.c_double), C.byref(agg))
    if rc:
        raise RuntimeError({5: "EmptyInputError", 2: "DimensionError", 8: "DegeneracyError"}.get(rc, str(rc)))
    return out[:levels], agg.value
