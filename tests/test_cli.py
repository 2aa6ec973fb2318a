"""`ccwsim simulate` (paper_2404_00441_b200/cli.py) against the reference CLI's
known answers (test_cli.cpp:102-240 restated).  Error paths run on CPU; the
end-to-end runs are GPU tests whose realization files must be byte-identical
to the oracle's realizations written in the reference format."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import pyoracle
from paper_2404_00441_b200 import ccwsim as cs
from paper_2404_00441_b200 import fileio as cio
from paper_2404_00441_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, cwd, env_extra=None):
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, "-m", "paper_2404_00441_b200.cli"] + args, cwd=cwd,
                       capture_output=True, text=True, env=env, timeout=600)
    return r.returncode, r.stdout, r.stderr


@pytest.fixture(scope="module")
def fx(tmp_path_factory):
    root = tmp_path_factory.mktemp("cli")
    ti = synth.channel_ti(128, 128, 7)
    ti_path = root / "ti.grid"
    cio.write_grid(cs.CategoricalGrid(128, 128, 2, ti), str(ti_path))
    cfg = root / "run.cfg"
    cfg.write_text(f"ti = {ti_path}\nsg_size = 96x96\ntemplate = 16\noverlap = 4\n"
                   "dwt_level = 2\ncandidates = 5\nrealizations = 3\nseed = 42\n")
    noseed = root / "noseed.cfg"
    noseed.write_text(f"ti = {ti_path}\nsg_size = 64\ntemplate = 16\noverlap = 4\n"
                      "dwt_level = 2\ncandidates = 4\nrealizations = 1\n")
    return {"root": root, "ti": ti, "ti_path": ti_path, "cfg": cfg, "noseed": noseed}


def test_help_and_subcommands(fx):
    # test_cli.cpp:102-106
    assert run(["--help"], fx["root"])[0] == 0
    assert run([], fx["root"])[0] != 0
    assert run(["frobnicate"], fx["root"])[0] != 0
    assert run(["validate", "--dir", "x"], fx["root"])[0] != 0


def test_config_errors_name_the_key(fx):
    # test_cli.cpp:229-240
    bad = fx["root"] / "bad.cfg"
    bad.write_text(f"ti = {fx['ti_path']}\nsg_size = 64\ntemplate = 16\noverlap = 6\n"
                   "dwt_level = 2\ncandidates = 4\nrealizations = 1\nseed = 1\n")
    rc, out, err = run(["simulate", "--config", str(bad)], fx["root"])
    assert rc != 0 and "overlap" in err and err.startswith("error: ")


def test_missing_seed_names_the_key(fx):
    # test_cli.cpp:209-215
    rc, out, err = run(["simulate", "--config", str(fx["noseed"]), "--out-dir",
                        str(fx["root"] / "noseed_out")], fx["root"])
    assert rc != 0 and "seed" in err


def test_missing_config_file(fx):
    rc, out, err = run(["simulate", "--config", str(fx["root"] / "absent.cfg")], fx["root"])
    assert rc != 0 and "absent.cfg" in err


def test_override_echo_before_simulation(fx):
    # the echo happens while the config is built (ccwsim_main.cpp:76-84), so an
    # invalid override is reported with the echo and the key
    rc, out, err = run(["simulate", "--config", str(fx["cfg"]), "--overlap", "6"], fx["root"])
    assert rc != 0 and "override: overlap = 6 (config had 4)" in out and "overlap" in err


def oracle_grid_bytes(tmp_path, ti, nf, d, hd, seed):
    o = pyoracle.restatement().simulate_one(ti, nf, pyoracle.Cfg(**d), hd, seed=seed)["realization"]
    p = str(tmp_path / "oracle.grid")
    cio.write_grid(cs.CategoricalGrid(o.shape[0], o.shape[1], nf, o.astype(np.uint8)), p)
    with open(p, "rb") as f:
        return f.read()


@pytest.mark.gpu
def test_simulate_writes_realizations_and_manifest(fx, tmp_path):
    # test_cli.cpp:108-133, plus byte parity with the oracle
    out = fx["root"] / "sim_basic"
    rc, stdout, err = run(["simulate", "--config", str(fx["cfg"]), "--out-dir", str(out)], fx["root"])
    assert rc == 0, err
    assert f"wrote 3 realizations to {out}" in stdout
    m = json.loads((out / "manifest.json").read_text())
    assert m["subcommand"] == "simulate"
    p = m["parameters"]
    assert (p["template"], p["seed"], p["realizations"], p["overlap"]) == (16, 42, 3, 4)
    assert p["scoring"] == "raw" and p["facies_mode"] == "indicator" and p["hard_data"] is None
    assert len(m["realizations"]) == 3
    assert "wall_seconds" in m["realizations"][0]
    assert "pre_overwrite_mismatch_rate" in m["realizations"][0]
    assert m["realizations"][0]["seed"] != m["realizations"][1]["seed"]
    d = dict(sg_height=96, sg_width=96, template_size=16, overlap=4, dwt_level=2, candidates=5)
    for r in range(1, 4):
        assert (out / f"real_{r}.pgm").exists()
        g = cio.read_grid(str(out / f"real_{r}.grid"))
        assert (g.height, g.width) == (96, 96)
        seed = cs.mix64(42, r)
        assert m["realizations"][r - 1]["seed"] == seed
        want = oracle_grid_bytes(tmp_path, fx["ti"], 2, d, None, seed)
        assert (out / f"real_{r}.grid").read_bytes() == want
    # the manifest is nlohmann::json dump(2): sorted keys, 2-space indent
    text = (out / "manifest.json").read_text()
    assert text == json.dumps(m, indent=2, sort_keys=True, ensure_ascii=False) + "\n"


@pytest.mark.gpu
def test_simulate_deterministic_across_reruns_and_workers(fx):
    # test_cli.cpp:135-157
    dirs = []
    for name, extra in (("det_a", []), ("det_b", []), ("det_c", ["--workers", "4"])):
        out = fx["root"] / name
        assert run(["simulate", "--config", str(fx["cfg"]), "--out-dir", str(out)] + extra,
                   fx["root"])[0] == 0
        dirs.append(out)
    for r in range(1, 4):
        for ext in ("grid", "pgm"):
            a = (dirs[0] / f"real_{r}.{ext}").read_bytes()
            assert a == (dirs[1] / f"real_{r}.{ext}").read_bytes()
            assert a == (dirs[2] / f"real_{r}.{ext}").read_bytes()


@pytest.mark.gpu
def test_flag_twins_override_and_echo(fx):
    # test_cli.cpp:159-168
    out = fx["root"] / "sim_override"
    rc, stdout, err = run(["simulate", "--config", str(fx["cfg"]), "--overlap", "8",
                           "--out-dir", str(out)], fx["root"])
    assert rc == 0, err
    assert "override: overlap = 8" in stdout
    assert json.loads((out / "manifest.json").read_text())["parameters"]["overlap"] == 8


@pytest.mark.gpu
def test_hard_data_mismatch_rate_and_honoured(fx, tmp_path):
    # test_cli.cpp:170-190, plus byte parity with the oracle
    hd = fx["root"] / "hd.csv"
    hd.write_text("0,0,1\n50,50,0\n10,70,1\n")
    out = fx["root"] / "sim_cond"
    rc, stdout, err = run(["simulate", "--config", str(fx["cfg"]), "--hard-data", str(hd),
                           "--out-dir", str(out)], fx["root"])
    assert rc == 0, err
    m = json.loads((out / "manifest.json").read_text())
    for e in m["realizations"]:
        assert e["hard_data_count"] == 3
        assert isinstance(e["pre_overwrite_mismatch_rate"], float)
    g = cio.read_grid(str(out / "real_1.grid"))
    assert g.at(0, 0) == 1 and g.at(50, 50) == 0 and g.at(10, 70) == 1
    d = dict(sg_height=96, sg_width=96, template_size=16, overlap=4, dwt_level=2, candidates=5)
    pts = [(0, 0, 1), (50, 50, 0), (10, 70, 1)]
    for r in range(1, 4):
        assert (out / f"real_{r}.grid").read_bytes() == \
            oracle_grid_bytes(tmp_path, fx["ti"], 2, d, pts, cs.mix64(42, r))


@pytest.mark.gpu
def test_out_dir_env_fallback(fx):
    # test_cli.cpp:192-199
    out = fx["root"] / "sim_env"
    rc, _, err = run(["simulate", "--config", str(fx["cfg"])], fx["root"],
                     {"CCWSIM_OUT_DIR": str(out)})
    assert rc == 0, err
    assert (out / "real_1.grid").exists()


@pytest.mark.gpu
def test_seed_flag_and_entropy(fx):
    # test_cli.cpp:216-227
    assert run(["simulate", "--config", str(fx["noseed"]), "--seed", "5", "--out-dir",
                str(fx["root"] / "flagseed_out")], fx["root"])[0] == 0
    rc, out, err = run(["simulate", "--config", str(fx["noseed"]), "--entropy", "--out-dir",
                        str(fx["root"] / "entropy_out")], fx["root"])
    assert rc == 0, err
    assert "entropy seed:" in out
