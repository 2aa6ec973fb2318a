"""ctypes binding of the 3D restatement (oracle/ccw3d_oracle.c, inside
_build/libccworacle.so) plus a pure-Python loop restatement of the same
definition for small cases.  TEST INFRASTRUCTURE ONLY: tests/ and bench.py's
CPU legs may use it; the product never does.

The reference has no 3D; ccw3d_oracle.h is the normative
definition of the extension.  Parity for 3D is "restatement-pinned": the C
restatement is checked against the independent Python loops below and, for
degenerate extents (one axis equal to the template), against the 2D
reference through the embedding described in tests/test_oracle3d_cpu.py.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libccworacle.so")

ORDERS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


class Config3C(C.Structure):
    _fields_ = [("sg", C.c_int32 * 3), ("template_size", C.c_int32), ("overlap", C.c_int32),
                ("dwt_level", C.c_int32), ("candidates", C.c_int32),
                ("n_realizations", C.c_int32), ("any_support", C.c_int32), ("_pad", C.c_int32),
                ("master_seed", C.c_uint64)]


class Diag3C(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("corner", C.c_int32), ("order", C.c_int32),
                ("work", C.c_int32 * 3), ("placement_count", C.c_int32),
                ("hard_data_count", C.c_int32), ("pre_overwrite_mismatches", C.c_int32)]


@dataclass
class Cfg3:
    sg: tuple = (32, 32, 32)
    template_size: int = 16
    overlap: int = 4
    dwt_level: int = 2
    candidates: int = 1
    n_realizations: int = 1
    any_support: bool = False
    master_seed: int = 1234

    def c(self) -> Config3C:
        s = Config3C()
        for a in range(3):
            s.sg[a] = int(self.sg[a])
        s.template_size = self.template_size
        s.overlap = self.overlap
        s.dwt_level = self.dwt_level
        s.candidates = self.candidates
        s.n_realizations = self.n_realizations
        s.any_support = int(bool(self.any_support))
        s.master_seed = int(self.master_seed) & ((1 << 64) - 1)
        return s


class Oracle3Error(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _hd(hd):
    if hd is None or len(hd) == 0:
        return None, 0
    a = np.ascontiguousarray(np.asarray(hd, np.int32).reshape(-1, 4))
    return a, a.shape[0]


class Oracle3:
    def __init__(self):
        self.lib = C.CDLL(SO)
        self.lib.ccwo3_last_error.restype = C.c_char_p

    def _check(self, rc):
        if rc:
            raise Oracle3Error(rc, self.lib.ccwo3_last_error().decode())

    def validate(self, cfg: Cfg3, ti_dims=None, nf=2, hd=None):
        a, n = _hd(hd)
        dims = np.asarray(ti_dims, np.int32) if ti_dims is not None else None
        self._check(self.lib.ccwo3_validate(C.byref(cfg.c()), _p(dims, C.c_int32) if dims is not None else None,
                                            int(nf), _p(a, C.c_int32) if a is not None else None, n))

    def block_counts(self, ti, nf, levels):
        ti = np.ascontiguousarray(ti, np.uint8)
        dims = np.array(ti.shape, np.int32)
        b = 1 << levels
        out = np.zeros((nf,) + tuple(d // b for d in ti.shape), np.int32)
        self._check(self.lib.ccwo3_block_counts(_p(ti, C.c_uint8), _p(dims, C.c_int32), int(nf),
                                                int(levels), _p(out, C.c_int32)))
        return out

    def score_map(self, counts, or_counts, mask):
        counts = np.ascontiguousarray(counts, np.int32)
        nf = counts.shape[0]
        tc = mask.shape[0]
        cd = np.array(counts.shape[1:], np.int32)
        n = np.ascontiguousarray(or_counts, np.int32)
        m = np.ascontiguousarray(mask, np.uint8)
        out = np.zeros(tuple(int(d) - tc + 1 for d in cd), np.int64)
        self._check(self.lib.ccwo3_score_map(_p(counts, C.c_int32), _p(cd, C.c_int32), nf, _p(n, C.c_int32),
                                             _p(m, C.c_uint8), tc, _p(out, C.c_int64)))
        return out

    def plan(self, cfg: Cfg3, seed):
        cap = 1 << 16
        corner, order, cnt = C.c_int(), C.c_int(), C.c_int()
        work = np.zeros(3, np.int32)
        origins = np.zeros((cap, 3), np.int32)
        shapes = np.zeros(cap, np.int32)
        self._check(self.lib.ccwo3_plan(C.byref(cfg.c()), C.c_uint64(seed), C.byref(corner), C.byref(order),
                                        _p(work, C.c_int32), _p(origins, C.c_int32), _p(shapes, C.c_int32), cap,
                                        C.byref(cnt)))
        n = cnt.value
        return dict(corner=corner.value, order=order.value, work=tuple(work.tolist()),
                    origins=origins[:n].copy(), shapes=shapes[:n].copy())

    def simulate_one(self, ti, nf, cfg: Cfg3, hd=None, seed=0, threads=1, chosen=False):
        ti = np.ascontiguousarray(ti, np.uint8)
        dims = np.array(ti.shape, np.int32)
        a, n = _hd(hd)
        out = np.zeros(tuple(cfg.sg), np.uint8)
        d = Diag3C()
        ch = None
        if chosen:
            pl = self.plan(cfg, seed)
            ch = np.zeros((len(pl["shapes"]), 3), np.int32)
        self._check(self.lib.ccwo3_simulate_one(
            _p(ti, C.c_uint8), _p(dims, C.c_int32), int(nf), C.byref(cfg.c()),
            _p(a, C.c_int32) if a is not None else None, n, C.c_uint64(seed), int(threads),
            _p(out, C.c_uint8), C.byref(d), _p(ch, C.c_int32) if ch is not None else None))
        res = {"realization": out, "diagnostics": diag_dict(d)}
        if chosen:
            res["chosen"] = ch
        return res

    def simulate_ensemble(self, ti, nf, cfg: Cfg3, hd=None, workers=1):
        ti = np.ascontiguousarray(ti, np.uint8)
        dims = np.array(ti.shape, np.int32)
        a, n = _hd(hd)
        nr = cfg.n_realizations
        out = np.zeros((nr,) + tuple(cfg.sg), np.uint8)
        diags = (Diag3C * nr)()
        self._check(self.lib.ccwo3_simulate_ensemble(
            _p(ti, C.c_uint8), _p(dims, C.c_int32), int(nf), C.byref(cfg.c()),
            _p(a, C.c_int32) if a is not None else None, n, int(workers), _p(out, C.c_uint8), diags))
        return out, [diag_dict(x) for x in diags]


def diag_dict(d) -> dict:
    return dict(seed=d.seed, corner=d.corner, order=d.order, work=tuple(d.work),
                placement_count=d.placement_count, hard_data_count=d.hard_data_count,
                pre_overwrite_mismatches=d.pre_overwrite_mismatches)


def oracle3() -> Oracle3:
    return Oracle3()


# ------------------------------------------- pure-Python loop restatement --
# Independent of the C file: written from ccw3d_oracle.h's definition, used
# only on small cases to pin the C restatement.

_M64 = (1 << 64) - 1


class _MT:
    def __init__(self, s):
        mt = [0] * 312
        mt[0] = s & _M64
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self.mt, self.i = mt, 312

    def __call__(self):
        if self.i >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64

    def bounded(self, n):
        thr = ((1 << 64) - n) % n
        while True:
            r = self()
            if r >= thr:
                return r % n


def py_simulate_one(ti, nf, cfg: Cfg3, hd=None, seed=0):
    """Loop restatement of ccw3d_oracle.h (small cases only)."""
    ti = np.asarray(ti, np.uint8)
    J, T, OV = cfg.dwt_level, cfg.template_size, cfg.overlap
    B = 1 << J
    tc = T >> J
    used = [d // B * B for d in ti.shape]
    c = [u // B for u in used]
    counts = np.zeros((nf,) + tuple(c), np.int64)
    for f in range(nf):
        ind = (ti[:used[0], :used[1], :used[2]] == f).astype(np.int64)
        counts[f] = ind.reshape(c[0], B, c[1], B, c[2], B).sum(axis=(1, 3, 5))
    o = [ci - tc + 1 for ci in c]
    rng = _MT(seed)
    corner = rng.bounded(8)
    order = ORDERS[rng.bounded(6)]
    stride = T - OV
    work, pos = [], []
    for a in range(3):
        sg = cfg.sg[a]
        w = T if sg == T else T + -(-(sg - T) // stride) * stride
        work.append(w)
        ps = list(range(0, w - T + 1, stride))
        if (corner >> a) & 1:
            ps.reverse()
        pos.append(ps)
    g = np.zeros(work, np.uint8)
    sim = np.zeros(work, bool)
    K = min(cfg.candidates, int(np.prod(o)))
    hd = [] if hd is None else [tuple(int(v) for v in row) for row in hd]
    for io in range(len(pos[order[0]])):
        for im in range(len(pos[order[1]])):
            for ii in range(len(pos[order[2]])):
                idx = [0, 0, 0]
                idx[order[0]], idx[order[1]], idx[order[2]] = io, im, ii
                P = [pos[a][idx[a]] for a in range(3)]
                sh = [idx[a] > 0 for a in range(3)]
                if not any(sh):
                    fr = [rng.bounded((used[a] - T) // B + 1) * B for a in range(3)]
                else:
                    sup = np.zeros((T, T, T), bool)
                    for a in range(3):
                        if sh[a]:
                            sl = [slice(None)] * 3
                            sl[a] = slice(0, OV) if not (corner >> a) & 1 else slice(T - OV, T)
                            sup[tuple(sl)] = True
                    win = g[P[0]:P[0] + T, P[1]:P[1] + T, P[2]:P[2] + T]
                    assert sim[P[0]:P[0] + T, P[1]:P[1] + T, P[2]:P[2] + T][sup].all()
                    n = np.zeros((nf, tc, tc, tc), np.int64)
                    for f in range(nf):
                        ind = ((win == f) & sup).astype(np.int64)
                        n[f] = ind.reshape(tc, B, tc, B, tc, B).sum(axis=(1, 3, 5))
                    mask = sup.reshape(tc, B, tc, B, tc, B).any(axis=(1, 3, 5))
                    n[:, ~mask] = 0
                    S = np.zeros(o, np.int64)
                    for m0, m1, m2 in zip(*np.nonzero(mask)):
                        for f in range(nf):
                            if n[f, m0, m1, m2]:
                                S += n[f, m0, m1, m2] * counts[f, m0:m0 + o[0], m1:m1 + o[1], m2:m2 + o[2]]
                    flat = S.ravel()
                    order_idx = sorted(range(flat.size), key=lambda q: (-flat[q], q))[:K]
                    local = [(d[0] - P[0], d[1] - P[1], d[2] - P[2], d[3]) for d in hd
                             if all(P[a] <= d[a] < P[a] + T for a in range(3))]
                    if local:
                        best, best_m = 0, len(local) + 1
                        for ci, q in enumerate(order_idx):
                            q0, q1, q2 = np.unravel_index(q, o)
                            mm = sum(int(ti[q0 * B + l0, q1 * B + l1, q2 * B + l2]) != f
                                     for l0, l1, l2, f in local)
                            if mm == 0:
                                best = ci
                                break
                            if mm < best_m:
                                best, best_m = ci, mm
                        q = order_idx[best]
                    else:
                        q = order_idx[rng.bounded(len(order_idx))]
                    fr = [int(v) * B for v in np.unravel_index(q, o)]
                g[P[0]:P[0] + T, P[1]:P[1] + T, P[2]:P[2] + T] = \
                    ti[fr[0]:fr[0] + T, fr[1]:fr[1] + T, fr[2]:fr[2] + T]
                sim[P[0]:P[0] + T, P[1]:P[1] + T, P[2]:P[2] + T] = True
    mism = 0
    for d in hd:
        if g[d[0], d[1], d[2]] != d[3]:
            mism += 1
        g[d[0], d[1], d[2]] = d[3]
    return g[:cfg.sg[0], :cfg.sg[1], :cfg.sg[2]].copy(), mism
