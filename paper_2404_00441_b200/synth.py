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
