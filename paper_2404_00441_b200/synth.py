"""Seeded synthetic training images and hard data for the BASELINE.json configs.

The paper's Channel / Stonewall / Ganges TIs are not available here, so the
benchmark and the full-size tests use these generators, which follow the
shapes, facies counts and proportions BASELINE.json states.  All randomness is
mt19937_64 + bounded (the reference's own RNG discipline, rng.hpp:21-28); the
geometry is vectorised numpy.  Inputs are generated once per process and the
same bytes feed the GPU path and every CPU baseline.
"""
from __future__ import annotations

import numpy as np

from .ccwsim import Mt19937_64, bounded


def _uniform(rng: Mt19937_64, lo: float, hi: float, steps: int = 1 << 20) -> float:
    return lo + (hi - lo) * bounded(rng, steps) / steps


def channel_ti(h: int, w: int, seed: int, amp=(5.0, 25.0), wavelength=(60.0, 200.0),
               width=(4.0, 10.0), target: float = 0.28, scale: float = 1.0) -> np.ndarray:
    """Binary TI of sinuous east-west sine-curve channels (code 1) on code 0,
    added until the facies-1 proportion reaches ``target`` (config 0; config 2
    uses scale=8)."""
    rng = Mt19937_64(seed)
    ti = np.zeros((h, w), np.uint8)
    rows = np.arange(h, dtype=np.float64)[:, None]
    cols = np.arange(w, dtype=np.float64)[None, :]
    for _ in range(10000):
        if ti.mean() >= target:
            break
        base = _uniform(rng, 0, h)
        a = _uniform(rng, *amp) * scale
        lam = _uniform(rng, *wavelength) * scale
        wd = _uniform(rng, *width) * scale
        phase = _uniform(rng, 0, 2 * np.pi)
        center = base + a * np.sin(2 * np.pi * cols / lam + phase)
        ti[np.abs(rows - center) < wd / 2] = 1
    return ti


def channel_levee_ti(h: int, w: int, seed: int, props=(0.55, 0.30, 0.15)) -> np.ndarray:
    """3-facies TI: channels (code 1) plus elliptical levee lenses (code 2)
    hugging the channels, on a background (code 0) (config 1)."""
    rng = Mt19937_64(seed)
    ti = np.zeros((h, w), np.uint8)
    rows = np.arange(h, dtype=np.float64)[:, None]
    cols = np.arange(w, dtype=np.float64)[None, :]
    centers = []
    for _ in range(10000):
        if (ti == 1).mean() >= props[1]:
            break
        base = _uniform(rng, 0, h)
        a = _uniform(rng, 5, 25)
        lam = _uniform(rng, 60, 200)
        wd = _uniform(rng, 4, 10)
        phase = _uniform(rng, 0, 2 * np.pi)
        center = base + a * np.sin(2 * np.pi * cols / lam + phase)
        ti[np.abs(rows - center) < wd / 2] = 1
        centers.append((center, wd))
    for _ in range(100000):
        if (ti == 2).mean() >= props[2]:
            break
        center, wd = centers[bounded(rng, len(centers))]
        x0 = float(bounded(rng, w))
        side = 1.0 if bounded(rng, 2) else -1.0
        y0 = float(center[0, int(x0)]) + side * (wd / 2 + _uniform(rng, 1, 6))
        ax = _uniform(rng, 6, 30)
        ay = _uniform(rng, 2, 6)
        theta = _uniform(rng, -0.4, 0.4)
        dx, dy = cols - x0, rows - y0
        u = dx * np.cos(theta) + dy * np.sin(theta)
        v = -dx * np.sin(theta) + dy * np.cos(theta)
        lens = (u / ax) ** 2 + (v / ay) ** 2 <= 1.0
        ti[lens & (ti == 0)] = 2
    return ti


def config0_ti() -> np.ndarray:
    """Config 0: 250x250 binary channels.  The reference rejects 250 at J=2
    (simulator.hpp:78-81), so parity runs use the top-left 248x248 crop."""
    return channel_ti(250, 250, seed=20240400)


def config1_ti() -> np.ndarray:
    """Config 1 (the headline bench workload): 500x500, 3 facies."""
    return channel_levee_ti(500, 500, seed=20240401)


def config2_ti() -> np.ndarray:
    """Config 2: 2000x2000 binary channels, config 0's generator scaled x8."""
    return channel_ti(2000, 2000, seed=20240402, scale=8.0)


def hard_data_from(realization: np.ndarray, fraction: float, seed: int) -> np.ndarray:
    """(n, 3) int32 (row, col, facies) triples: a seeded partial Fisher-Yates
    draw of cells (procedure of acceptance.cpp:392-410, with mt19937_64 +
    bounded instead of std::shuffle) read from ``realization``."""
    h, w = realization.shape
    n = int(round(fraction * h * w))
    rng = Mt19937_64(seed)
    perm = np.arange(h * w, dtype=np.int64)
    for i in range(n):
        j = i + bounded(rng, h * w - i)
        perm[i], perm[j] = perm[j], perm[i]
    cells = perm[:n]
    r, c = cells // w, cells % w
    return np.stack([r, c, realization[r, c]], axis=1).astype(np.int32)


def config2_hard_data(ti: np.ndarray, realization: np.ndarray | None = None) -> np.ndarray:
    """1% of the 4000x4000 grid from a seeded realization of the config-2
    simulation (seed 777, K=1, unconditional)."""
    if realization is None:
        from . import ccwsim as cs
        grid = cs.CategoricalGrid(ti.shape[0], ti.shape[1], 2, ti)
        cfg = cs.SimConfig(4000, 4000, 96, 24, 3, 1)
        realization = cs.simulate_one(grid, cfg, 777).realization.cells
    return hard_data_from(realization, 0.01, seed=606)


# --------------------------------------------------------------- 3D (c3, c4) --
# Arrays are (d0, d1, d2) = (z, y, x): axis 0 is vertical, so BASELINE's
# "X x Y x Z" extents appear reversed.

def _ellipsoid(vol: np.ndarray, rng: Mt19937_64, code: int, axes=(5.0, 40.0), flat: float = 0.35,
               only_on=None) -> None:
    """One ellipsoidal lens of ``code``: horizontal semi-axes drawn in
    ``axes``, vertical semi-axis ``flat`` times the smaller one, random
    azimuth and a small dip; written over ``only_on`` cells (None = any)."""
    d0, d1, d2 = vol.shape
    a = _uniform(rng, *axes)
    b = _uniform(rng, axes[0], a)
    c = max(1.5, flat * b)
    z0, y0, x0 = _uniform(rng, 0, d0), _uniform(rng, 0, d1), _uniform(rng, 0, d2)
    az = _uniform(rng, 0, np.pi)
    dip = _uniform(rng, -0.15, 0.15)
    r = int(np.ceil(a)) + 1
    zs = slice(max(0, int(z0 - c - 2 - r * abs(dip))), min(d0, int(z0 + c + 2 + r * abs(dip)) + 1))
    ys = slice(max(0, int(y0) - r), min(d1, int(y0) + r + 1))
    xs = slice(max(0, int(x0) - r), min(d2, int(x0) + r + 1))
    if zs.start >= zs.stop or ys.start >= ys.stop or xs.start >= xs.stop:
        return
    zz, yy, xx = np.meshgrid(np.arange(zs.start, zs.stop, dtype=np.float64) - z0,
                             np.arange(ys.start, ys.stop, dtype=np.float64) - y0,
                             np.arange(xs.start, xs.stop, dtype=np.float64) - x0, indexing="ij")
    u = xx * np.cos(az) + yy * np.sin(az)
    v = -xx * np.sin(az) + yy * np.cos(az)
    w = zz - dip * u
    inside = (u / a) ** 2 + (v / b) ** 2 + (w / c) ** 2 <= 1.0
    sub = vol[zs, ys, xs]
    if only_on is not None:
        inside &= sub == only_on
    sub[inside] = code


def lens_ti3d(shape, seed: int, props=(0.50, 0.25, 0.15, 0.10)) -> np.ndarray:
    """Config 3: ellipsoidal lenses of facies 1..F-1 (axes 5-40 cells,
    random orientation) in a background facies 0, added until each facies
    reaches its proportion."""
    rng = Mt19937_64(seed)
    vol = np.zeros(shape, np.uint8)
    n = vol.size
    for code in range(1, len(props)):
        for _ in range(100000):
            if np.count_nonzero(vol == code) >= props[code] * n:
                break
            _ellipsoid(vol, rng, code, only_on=0)
    return vol


def config3_ti() -> np.ndarray:
    """Config 3: 180 x 150 x 120 (x, y, z) 4-facies lens TI, as a (120, 150, 180)
    array.  150 is not divisible by 2^J = 4: the adjusted runs use the
    148-wide crop, the literal runs the any_support extension (same windows)."""
    return lens_ti3d((120, 150, 180), seed=20240403)


def channel_belt_ti3d(shape, seed: int, props=(0.42, 0.26, 0.12, 0.12, 0.08)) -> np.ndarray:
    """Config 4: sinuous 3D channel belts (facies 1) with levee wings (facies
    2) along their tops, then ellipsoidal lenses of facies 3 and 4, on a
    background facies 0."""
    rng = Mt19937_64(seed)
    vol = np.zeros(shape, np.uint8)
    d0, d1, d2 = shape
    n = vol.size
    ys = np.arange(d1, dtype=np.float64)[:, None]
    xs = np.arange(d2, dtype=np.float64)[None, :]
    for _ in range(100000):
        if np.count_nonzero(vol == 1) >= props[1] * n:
            break
        z0 = _uniform(rng, 0, d0)
        th = _uniform(rng, 3.0, 10.0)
        wd = _uniform(rng, 8.0, 30.0)
        amp = _uniform(rng, 10.0, 60.0)
        lam = _uniform(rng, 120.0, 400.0)
        ph = _uniform(rng, 0, 2 * np.pi)
        base = _uniform(rng, 0, d1)
        along_x = bounded(rng, 2) == 0
        if along_x:
            dist = np.abs(ys - (base + amp * np.sin(2 * np.pi * xs / lam + ph)))
        else:
            dist = np.abs(xs - (base * d2 / d1 + amp * np.sin(2 * np.pi * ys / lam + ph)))
        chan = dist < wd / 2
        lev = (dist >= wd / 2) & (dist < wd / 2 + _uniform(rng, 3.0, 10.0))
        for z in range(max(0, int(z0 - th / 2)), min(d0, int(z0 + th / 2) + 1)):
            sl = vol[z]
            sl[chan] = 1
            if z >= z0:  # levees drape the upper half of the belt
                sl[lev & (sl == 0)] = 2
    for code in (3, 4):
        for _ in range(100000):
            if np.count_nonzero(vol == code) >= props[code] * n:
                break
            _ellipsoid(vol, rng, code, axes=(8.0, 40.0), only_on=0)
    return vol


def config4_ti() -> np.ndarray:
    """Config 4: 400 x 400 x 200 (x, y, z) 5-facies channel-belt TI, as a
    (200, 400, 400) array."""
    return channel_belt_ti3d((200, 400, 400), seed=20240404)


def hard_data3d_from(realization: np.ndarray, fraction: float, seed: int) -> np.ndarray:
    """(n, 4) int32 (i0, i1, i2, facies) rows: a seeded partial Fisher-Yates
    draw of cells read from ``realization``."""
    shape = realization.shape
    tot = int(np.prod(shape))
    n = int(round(fraction * tot))
    rng = Mt19937_64(seed)
    chosen = {}
    out = np.zeros((n, 4), np.int32)
    for i in range(n):  # sparse partial Fisher-Yates over [0, tot)
        j = i + bounded(rng, tot - i)
        vi, vj = chosen.get(i, i), chosen.get(j, j)
        chosen[i], chosen[j] = vj, vi
        c = np.unravel_index(vj, shape)
        out[i] = (c[0], c[1], c[2], realization[c])
    return out


def wells3d_from(realization: np.ndarray, n_wells: int, seed: int) -> np.ndarray:
    """Vertical wells: ``n_wells`` full columns along axis 0 at seeded
    distinct (i1, i2) positions, values read from ``realization``."""
    d0, d1, d2 = realization.shape
    rng = Mt19937_64(seed)
    picked = []
    while len(picked) < n_wells:
        p = (bounded(rng, d1), bounded(rng, d2))
        if p not in picked:
            picked.append(p)
    rows = []
    for i1, i2 in picked:
        for i0 in range(d0):
            rows.append((i0, i1, i2, int(realization[i0, i1, i2])))
    return np.array(rows, np.int32)
