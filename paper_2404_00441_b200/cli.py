"""``ccwsim simulate`` on the B200 path (`/root/reference/proj/tools/ccwsim_main.cpp`,
SURVEY §8(f) rank 1).

    python -m paper_2404_00441_b200.cli simulate --config run.cfg [flag twins] \\
        [--workers N] [--entropy]

Same semantics as the reference command: the config file (io.parse rules) and
its flag twins (flag values win and are echoed, ccwsim_main.cpp:26-94), the
seed rules (``--entropy`` draws one only when no seed is given anywhere), the
output directory (config / flag, else ``$CCWSIM_OUT_DIR``, else "."), and the
outputs ``real_<r>.grid``, ``real_<r>.pgm`` and ``manifest.json``
(ccwsim_main.cpp:132-199).  All realizations run in one batched GPU call;
``--workers`` is accepted and recorded but has no effect (the reference's
results are worker-count invariant).  Errors print ``error: <message>`` and
exit 1.  ``validate``, ``anodi`` and ``bench`` need the validation metrics
(metrics.hpp), which are out of this package's scope.
"""
from __future__ import annotations

import argparse
import json
import os
import random
import sys
from typing import Dict, List, Optional

from . import fileio as cio
from .ccwsim import ConfigError, Error, simulate_ensemble

CORNERS = {0: "top_left", 1: "top_right", 2: "bottom_left", 3: "bottom_right"}  # simulator.hpp:97-104

# config key -> flag twin (ccwsim_main.cpp:29-43)
FLAG_TWINS = [("ti", "--ti"), ("sg_size", "--sg-size"), ("template", "--template"),
              ("overlap", "--overlap"), ("dwt_level", "--dwt-level"),
              ("candidates", "--candidates"), ("realizations", "--realizations"),
              ("seed", "--seed"), ("hard_data", "--hard-data"), ("scoring", "--scoring"),
              ("facies_mode", "--facies-mode"), ("min_cut", "--min-cut"),
              ("out_dir", "--out-dir")]


def build_config(config_path: str, flags: Dict[str, str], entropy: bool) -> cio.ConfigFile:
    """ccwsim_main.cpp:57-94."""
    kv = cio.read_key_values(config_path)
    for key in ("ti", "sg_size", "template", "overlap", "dwt_level", "candidates", "realizations"):
        if key not in kv and key not in flags:
            raise ConfigError(f'{config_path}: missing required key "{key}"')
    seed_given = "seed" in kv or "seed" in flags
    if not seed_given and not entropy:
        raise ConfigError(f'{config_path}: missing required key "seed"')
    cfg = cio.ConfigFile()
    for key, value in cio._map_order(kv):
        cio.apply_config_entry(cfg, key, value)
    for key, value in cio._map_order(flags):
        if key in kv and kv[key] != value:
            print(f"override: {key} = {value} (config had {kv[key]})")
        elif key not in kv:
            print(f"override: {key} = {value}")
        cio.apply_config_entry(cfg, key, value)
    if not seed_given:
        cfg.sim.master_seed = random.SystemRandom().getrandbits(64)
        print(f"entropy seed: {cfg.sim.master_seed}")
    cfg.sim.validate()
    return cfg


def resolve_out_dir(configured: Optional[str]) -> str:
    """ccwsim_main.cpp:96-102."""
    if configured:
        return configured
    env = os.environ.get("CCWSIM_OUT_DIR")
    return env if env else "."


def run_simulate(config_path: str, flags: Dict[str, str], entropy: bool, workers: int) -> int:
    """ccwsim_main.cpp:132-199."""
    cfg = build_config(config_path, flags, entropy)
    ti = cio.read_grid(cfg.ti_path)
    if cfg.hard_data_path is not None:
        cfg.sim.hard_data = cio.read_hard_data(cfg.hard_data_path, cfg.sim.sg_height,
                                               cfg.sim.sg_width)
    cfg.sim.validate_against(ti)
    out_dir = resolve_out_dir(cfg.out_dir)
    try:
        os.makedirs(out_dir, exist_ok=True)
    except OSError as e:
        raise cio.IoError(f"cannot create {out_dir}: {e}") from None

    results = simulate_ensemble(ti, cfg.sim, workers)

    s = cfg.sim
    params = {
        "ti": cfg.ti_path, "sg_height": s.sg_height, "sg_width": s.sg_width,
        "template": s.template_size, "overlap": s.overlap, "dwt_level": s.dwt_level,
        "candidates": s.candidates, "realizations": s.n_realizations, "seed": s.master_seed,
        "scoring": s.scoring, "facies_mode": "raw-codes" if s.facies_mode == "raw_codes" else "indicator",
        "min_cut": bool(s.min_cut), "hard_data": cfg.hard_data_path, "out_dir": out_dir,
        "workers": workers,
    }
    reals: List[dict] = []
    for i, res in enumerate(results):
        r = i + 1
        stem = f"real_{r}"
        cio.write_grid(res.realization, os.path.join(out_dir, stem + ".grid"))
        cio.write_pgm(res.realization, os.path.join(out_dir, stem + ".pgm"))
        d = res.diagnostics
        reals.append({
            "index": r, "file": stem + ".grid", "seed": d.seed, "wall_seconds": d.wall_seconds,
            "origin": CORNERS[int(d.origin)], "column_major": bool(d.column_major),
            "hard_data_count": d.hard_data_count,
            "pre_overwrite_mismatches": d.pre_overwrite_mismatches,
            "pre_overwrite_mismatch_rate": d.pre_overwrite_mismatch_rate(),
        })
    manifest = {"subcommand": "simulate", "parameters": params, "realizations": reals}
    path = os.path.join(out_dir, "manifest.json")
    try:
        with open(path, "w", encoding="utf-8", newline="\n") as f:
            # nlohmann::json dump(2): std::map key order, 2-space indent
            f.write(json.dumps(manifest, indent=2, sort_keys=True, ensure_ascii=False) + "\n")
    except OSError:
        raise cio.IoError(f"cannot open {path} for writing") from None
    print(f"wrote {len(results)} realizations to {out_dir}")
    return 0


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="ccwsim",
                                 description="ccwsim: wavelet-space patch simulation (B200 path)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sim = sub.add_parser("simulate", help="run an ensemble of realizations")
    sim.add_argument("--config", required=True, help="config file (key = value lines)")
    for key, flag in FLAG_TWINS:
        sim.add_argument(flag, dest="twin_" + key, default=None)
    sim.add_argument("--workers", type=int, default=1, help="accepted; results do not depend on it")
    sim.add_argument("--entropy", action="store_true",
                     help="allow seeding from system entropy when no seed is given")
    for name in ("validate", "anodi", "bench"):
        p = sub.add_parser(name, help="needs metrics.hpp (out of scope)")
        p.add_argument("rest", nargs=argparse.REMAINDER)
    return ap


def main(argv: Optional[List[str]] = None) -> int:
    args = _parser().parse_args(argv)
    if args.cmd != "simulate":
        print(f"error: {args.cmd} needs the validation metrics (metrics.hpp), which this "
              "package does not implement", file=sys.stderr)
        return 1
    if not os.path.isfile(args.config):
        print(f"error: --config: File does not exist: {args.config}", file=sys.stderr)
        return 1
    if args.workers < 1:
        print("error: --workers: Value must be a positive number", file=sys.stderr)
        return 1
    flags = {key: getattr(args, "twin_" + key) for key, _ in FLAG_TWINS
             if getattr(args, "twin_" + key) is not None}
    try:
        return run_simulate(args.config, flags, args.entropy, args.workers)
    except Error as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
