"""File formats of the reference's `simulate` path, restated for this package
(`/root/reference/proj/include/ccwsim/io.hpp`).

Host-side text formats only -- nothing here touches the GPU:

* grid files      ``ccwsim-grid v1`` / ``<ncols> <nrows> <ncats>`` / rows
  (io.hpp:92-170): ``read_grid``, ``write_grid``;
* hard data files  ``row,col,facies`` per line, ``#`` comments (io.hpp:172-219):
  ``read_hard_data``, ``write_hard_data``;
* PGM previews     P2, codes spread evenly over 0..255 (io.hpp:221-256):
  ``write_pgm``;
* config files     ``key = value`` lines (io.hpp:408-536): ``read_key_values``,
  ``apply_config_entry``, ``parse_config``.

Parsing follows the reference's rules character for character (the trim set,
integer syntax, line numbering, error precedence and message texts), and the
writers produce the same bytes, so files round-trip between the two
implementations.  Errors are the ``ccwsim`` exception classes with the
reference's messages (``ParseError`` carries ``path`` and 1-based ``line``).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from .ccwsim import (CategoricalGrid, ConfigError, HardDataSet, HardDatum, IoError, ParseError,
                     SimConfig)

GRID_MAGIC = "ccwsim-grid v1"  # io.hpp:22

_TRIM = " \t\r"  # io.hpp:26-33: the only characters trimmed (getline drops '\n')
_INT_MAX = 2**31 - 1
_INT_MIN = -(2**31)
_U64_MAX = 2**64 - 1


def _trim(s: str) -> str:
    return s.strip(_TRIM)


def _parse_int(s: str, lo: int = _INT_MIN, hi: int = _INT_MAX) -> Optional[int]:
    """std::from_chars into an integer type (io.hpp:35-41): optional '-' (for
    signed types) then decimal digits, the whole trimmed token, in range."""
    s = _trim(s)
    if not s:
        return None
    body = s[1:] if s[0] == "-" and lo < 0 else s
    if not body or not all("0" <= ch <= "9" for ch in body):
        return None
    v = int(s)
    return v if lo <= v <= hi else None


def _split_ws(s: str) -> List[str]:
    """io.hpp:43-57: tokens separated by runs of ' ', '\\t', '\\r'."""
    out, i, n = [], 0, len(s)
    while i < n:
        while i < n and s[i] in _TRIM:
            i += 1
        j = i
        while j < n and s[j] not in _TRIM:
            j += 1
        if j > i:
            out.append(s[i:j])
        i = j
    return out


def _lines(path: str) -> List[str]:
    """std::getline over a binary stream: split on '\\n'; a final '\\n' does not
    start another line."""
    try:
        with open(path, "rb") as f:
            data = f.read().decode("latin-1")
    except OSError:
        raise IoError(f"cannot open {path}") from None
    if not data:
        return []
    parts = data.split("\n")
    if parts[-1] == "":
        parts.pop()
    return parts


def _write(path: str, text: str) -> None:
    try:
        with open(path, "wb") as f:
            f.write(text.encode("latin-1"))
    except OSError:
        raise IoError(f"cannot open {path} for writing") from None


# ------------------------------------------------------------------ grids --

def read_grid(path: str) -> CategoricalGrid:
    """io.hpp:99-155."""
    lines = _lines(path)
    if not lines:
        raise ParseError(path, 1, f'empty file, expected magic "{GRID_MAGIC}"')
    if _trim(lines[0]) != GRID_MAGIC:
        raise ParseError(path, 1, f'bad magic, expected "{GRID_MAGIC}"')
    if len(lines) < 2:
        raise ParseError(path, 2, "missing dimension line")
    dims = _split_ws(lines[1])
    vals = [_parse_int(d) for d in dims] if len(dims) == 3 else []
    if len(dims) != 3 or any(v is None for v in vals):
        raise ParseError(path, 2, 'expected "<ncols> <nrows> <ncats>"')
    ncols, nrows, ncats = vals
    if ncols < 1 or nrows < 1 or ncats < 1:
        raise ParseError(path, 2, "dimensions and category count must be positive")
    cells = _fast_rows(lines, nrows, ncols, ncats)
    if cells is not None:
        if any(_trim(l) for l in lines[2 + nrows:]):  # (slow path names the line)
            cells = None
    if cells is not None:
        return CategoricalGrid(nrows, ncols, ncats,
                               cells.astype(np.uint8 if ncats <= 255 else np.int32))
    cells = np.empty((nrows, ncols), np.int64)
    lineno = 2
    for r in range(nrows):
        if lineno >= len(lines):
            raise ParseError(path, lineno + 1,
                             f"unexpected end of file, expected row {r + 1} of {nrows}")
        line = lines[lineno]
        lineno += 1
        toks = _split_ws(line)
        if len(toks) != ncols:
            raise ParseError(path, lineno, f"expected {ncols} values, got {len(toks)}")
        for c, tok in enumerate(toks):
            code = _parse_int(tok)
            if code is None:
                raise ParseError(path, lineno, f'invalid code "{tok}"')
            if code < 0 or code >= ncats:
                raise ParseError(path, lineno, f"code {code} outside [0, {ncats})")
            cells[r, c] = code
    while lineno < len(lines):
        lineno += 1
        if _trim(lines[lineno - 1]):
            raise ParseError(path, lineno, "trailing content after last row")
    if ncats > 255:  # this package stores codes as uint8
        return CategoricalGrid(nrows, ncols, ncats, cells.astype(np.int32))
    return CategoricalGrid(nrows, ncols, ncats, cells.astype(np.uint8))


_FAST_OK = frozenset("0123456789 \t\r")


def _fast_rows(lines: List[str], nrows: int, ncols: int, ncats: int) -> Optional[np.ndarray]:
    """Vectorized parse of well-formed rows (non-negative codes, separators
    from the reference's set only); None sends the caller to the exact
    per-token path, which produces the reference's diagnostics."""
    rows = lines[2:2 + nrows]
    if len(rows) != nrows:
        return None
    for row in rows:
        if not _FAST_OK.issuperset(row):
            return None
    toks = [row.split() for row in rows]  # == _split_ws on this alphabet
    if any(len(t) != ncols for t in toks):
        return None
    flat = [t for row in toks for t in row]
    if any(len(t) > 9 for t in flat):  # (may overflow int32: exact path)
        return None
    cells = np.array(flat, dtype=np.int64).reshape(nrows, ncols) if flat else \
        np.zeros((nrows, ncols), np.int64)
    if cells.size and int(cells.max()) >= ncats:
        return None
    return cells


def _grid_rows(cells: np.ndarray) -> str:
    """Rows of space-separated decimal integers, '\n'-terminated."""
    cells = np.asarray(cells)
    if cells.size == 0:
        return "\n" * cells.shape[0]
    lo, hi = int(cells.min()), int(cells.max())
    h, w = cells.shape
    if lo >= 0 and hi < 10:  # one digit per value: build the bytes directly
        out = np.full((h, 2 * w), ord(" "), np.uint8)
        out[:, 0::2] = cells.astype(np.uint8) + ord("0")
        out[:, -1] = ord("\n")
        return out.tobytes().decode("latin-1")
    toks = np.array([str(v) for v in range(lo, hi + 1)], dtype=object)
    return "".join(" ".join(toks[row - lo]) + "\n" for row in cells.astype(np.int64))


def write_grid(grid: CategoricalGrid, path: str) -> None:
    """io.hpp:157-170."""
    cells = np.asarray(grid.cells)
    _write(path, f"{GRID_MAGIC}\n{grid.width} {grid.height} {grid.num_facies}\n" + _grid_rows(cells))


# -------------------------------------------------------------- hard data --

def read_hard_data(path: str, sg_height: int, sg_width: int) -> HardDataSet:
    """io.hpp:176-212."""
    hd = HardDataSet()
    seen: Dict[Tuple[int, int], int] = {}
    for lineno, line in enumerate(_lines(path), start=1):
        body = _trim(line)
        if not body or body[0] == "#":
            continue
        fields = body.split(",")
        vals = [_parse_int(f) for f in fields] if len(fields) == 3 else []
        if len(fields) != 3 or any(v is None for v in vals):
            raise ParseError(path, lineno, 'expected "row,col,facies"')
        row, col, fac = vals
        if row < 0 or row >= sg_height or col < 0 or col >= sg_width:
            raise ParseError(path, lineno,
                             f"coordinate ({row}, {col}) outside {sg_height}x{sg_width} grid")
        if fac < 0:
            raise ParseError(path, lineno, "facies code must be non-negative")
        first = seen.setdefault((row, col), lineno)
        if first != lineno:
            raise ParseError(path, lineno,
                             f"duplicate coordinate ({row}, {col}), first seen on line {first}")
        hd.points.append(HardDatum(row, col, fac))
    return hd


def write_hard_data(hd, path: str) -> None:
    """io.hpp:214-219."""
    pts = hd.points if isinstance(hd, HardDataSet) else hd
    rows = [(p.row, p.col, p.facies) if isinstance(p, HardDatum) else tuple(int(v) for v in p)
            for p in pts]
    _write(path, "".join(f"{r},{c},{f}\n" for r, c, f in rows))


# -------------------------------------------------------------------- PGM --

def _lround(x: float) -> int:
    """std::lround: nearest, halves away from zero."""
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def write_pgm(grid, path: str) -> None:
    """io.hpp:224-240 (CategoricalGrid: codes over 0..255) and io.hpp:243-256
    (a [0,1]-valued plane, clamped)."""
    if isinstance(grid, CategoricalGrid):
        cells = np.asarray(grid.cells).astype(np.int64)
        n = grid.num_facies
        lut = np.array([_lround(c * 255.0 / (n - 1)) if n > 1 else 0 for c in range(max(n, 1))],
                       np.int64)
        gray = lut[cells]
        h, w = grid.height, grid.width
    else:
        plane = np.asarray(grid, np.float64)
        h, w = plane.shape
        gray = np.vectorize(lambda v: _lround(min(1.0, max(0.0, v)) * 255.0))(plane) \
            if plane.size else plane.astype(np.int64)
    _write(path, f"P2\n{w} {h}\n255\n" + _grid_rows(np.asarray(gray)))


# ---------------------------------------------------------------- configs --

@dataclass
class ConfigFile:
    """io.hpp:415-420."""
    sim: SimConfig = field(default_factory=SimConfig)
    ti_path: str = ""
    hard_data_path: Optional[str] = None
    out_dir: Optional[str] = None


def read_key_values(path: str) -> Dict[str, str]:
    """io.hpp:424-447: key/value pairs (key order is the reference's std::map
    order, i.e. sorted -- callers iterate ``sorted(kv.items())``)."""
    kv: Dict[str, str] = {}
    for lineno, line in enumerate(_lines(path), start=1):
        body = _trim(line)
        if not body or body[0] == "#":
            continue
        eq = body.find("=")
        if eq < 0:
            raise ParseError(path, lineno, 'expected "key = value"')
        key, value = _trim(body[:eq]), _trim(body[eq + 1:])
        if not key:
            raise ParseError(path, lineno, "empty key")
        if key in kv:
            raise ParseError(path, lineno, f'duplicate key "{key}"')
        kv[key] = value
    return kv


def _map_order(kv: Dict[str, str]):
    """std::map<std::string> iteration order: bytewise lexicographic."""
    return sorted(kv.items(), key=lambda it: it[0].encode("latin-1"))


def apply_config_entry(cfg: ConfigFile, key: str, value: str) -> None:
    """io.hpp:453-518."""
    def integer(v: str, name: str) -> int:
        out = _parse_int(v)
        if out is None:
            raise ConfigError(f'{name}: expected an integer, got "{v}"')
        return out

    s = cfg.sim
    if key == "ti":
        cfg.ti_path = value
    elif key == "sg_size":
        parts = value.split("x")
        if len(parts) == 1:
            s.sg_height = s.sg_width = integer(parts[0], "sg_size")
        elif len(parts) == 2:
            s.sg_height = integer(_trim(parts[0]), "sg_size")
            s.sg_width = integer(_trim(parts[1]), "sg_size")
        else:
            raise ConfigError('sg_size: expected "<height>x<width>" or a single size')
    elif key == "template":
        s.template_size = integer(value, "template")
    elif key == "overlap":
        s.overlap = integer(value, "overlap")
    elif key == "dwt_level":
        s.dwt_level = integer(value, "dwt_level")
    elif key == "candidates":
        s.candidates = integer(value, "candidates")
    elif key == "realizations":
        s.n_realizations = integer(value, "realizations")
    elif key == "seed":
        seed = _parse_int(value, 0, _U64_MAX)
        if seed is None:
            raise ConfigError(f'seed: expected a 64-bit unsigned integer, got "{value}"')
        s.master_seed = seed
    elif key == "scoring":
        if value not in ("raw", "normalized"):
            raise ConfigError(f'scoring: expected "raw" or "normalized", got "{value}"')
        s.scoring = value
    elif key == "facies_mode":
        if value == "indicator":
            s.facies_mode = "indicator"
        elif value == "raw-codes":
            s.facies_mode = "raw_codes"
        else:
            raise ConfigError(
                f'facies_mode: expected "indicator" or "raw-codes", got "{value}"')
    elif key == "min_cut":
        if value in ("on", "true", "1"):
            s.min_cut = True
        elif value in ("off", "false", "0"):
            s.min_cut = False
        else:
            raise ConfigError(f'min_cut: expected on/off, got "{value}"')
    elif key == "hard_data":
        cfg.hard_data_path = value
    elif key == "out_dir":
        cfg.out_dir = value
    else:
        raise ConfigError(f'unknown key "{key}"')


REQUIRED_KEYS = ("ti", "sg_size", "template", "overlap", "dwt_level", "candidates",
                 "realizations", "seed")


def parse_config(path: str) -> ConfigFile:
    """io.hpp:522-536: required keys (in this order), every entry in map order,
    then SimConfig::validate."""
    kv = read_key_values(path)
    for key in REQUIRED_KEYS:
        if key not in kv:
            raise ConfigError(f'{path}: missing required key "{key}"')
    cfg = ConfigFile()
    for key, value in _map_order(kv):
        apply_config_entry(cfg, key, value)
    cfg.sim.validate()
    return cfg


__all__ = ["GRID_MAGIC", "ConfigFile", "apply_config_entry", "parse_config", "read_grid",
           "read_hard_data", "read_key_values", "write_grid", "write_hard_data", "write_pgm"]
