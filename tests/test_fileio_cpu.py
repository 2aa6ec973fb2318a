"""File formats (paper_2404_00441_b200/fileio.py) against the reference's own
known answers: test_io.cpp:46-370 restated (grid round trip, documented
layout, diagnostics with line numbers, hard-data rules, PGM bytes,
parse_config keys / errors)."""
import numpy as np
import pytest

from paper_2404_00441_b200 import ccwsim as cs
from paper_2404_00441_b200 import fileio as cio


def spit(path, text):
    with open(path, "wb") as f:
        f.write(text.encode())


def slurp(path):
    with open(path, "rb") as f:
        return f.read().decode()


def test_grid_roundtrip_byte_identity(tmp_path):
    # test_io.cpp:46-58
    rng = cs.Mt19937_64(61)
    cells = np.array([cs.bounded(rng, 3) for _ in range(32 * 32)], np.uint8).reshape(32, 32)
    g = cs.CategoricalGrid(32, 32, 3, cells)
    p1, p2 = str(tmp_path / "a.grid"), str(tmp_path / "b.grid")
    cio.write_grid(g, p1)
    back = cio.read_grid(p1)
    assert back == g
    cio.write_grid(back, p2)
    assert slurp(p1) == slurp(p2)


def test_read_grid_documented_layout(tmp_path):
    # test_io.cpp:60-71
    p = str(tmp_path / "g.grid")
    spit(p, "ccwsim-grid v1\n3 2 4\n0 1 2\n3 0 1\n")
    g = cio.read_grid(p)
    assert (g.height, g.width, g.num_facies) == (2, 3, 4)
    assert g.at(0, 0) == 0 and g.at(1, 0) == 3 and g.at(1, 2) == 1
    assert slurp(p) == (cio.write_grid(g, str(tmp_path / "h.grid")) or slurp(str(tmp_path / "h.grid")))


@pytest.mark.parametrize("text,line,needle", [
    ("ccwsim-grid v9\n2 2 2\n0 0\n0 0\n", 1, "magic"),
    ("ccwsim-grid v1\n4 2 2\n0 0 0 0\n0 0 0 0 0\n", 4, "expected 4 values, got 5"),
    ("ccwsim-grid v1\n2 2 2\n0 1\n0 2\n", 4, "code 2"),
    ("ccwsim-grid v1\n2 3 2\n0 1\n", 4, "unexpected end of file"),
    ("ccwsim-grid v1\n2 2 2\n0 1\n0 1\n1\n", 5, "trailing content"),
    ("ccwsim-grid v1\n2 x 2\n0 1\n0 1\n", 2, "<ncols> <nrows> <ncats>"),
    ("", 1, "empty file"),
    ("ccwsim-grid v1\n", 2, "missing dimension line"),
    ("ccwsim-grid v1\n0 2 2\n", 2, "must be positive"),
    ("ccwsim-grid v1\n2 1 2\n0 +1\n", 3, 'invalid code "+1"'),
    ("ccwsim-grid v1\n2 1 2\n0 -1\n", 3, "code -1 outside [0, 2)"),
])
def test_read_grid_diagnostics(tmp_path, text, line, needle):
    # test_io.cpp:73-127
    p = str(tmp_path / "bad.grid")
    spit(p, text)
    with pytest.raises(cs.ParseError) as e:
        cio.read_grid(p)
    assert e.value.line == line
    assert needle in str(e.value)
    assert str(e.value).startswith(f"{p}:{line}: ")


def test_read_grid_missing_file(tmp_path):
    with pytest.raises(cs.IoError):
        cio.read_grid(str(tmp_path / "absent.grid"))


def test_read_grid_tolerates_cr_and_tabs(tmp_path):
    p = str(tmp_path / "crlf.grid")
    spit(p, "ccwsim-grid v1\r\n2\t2 3\r\n0 1\r\n2\t\t0  \r\n\r\n")
    g = cio.read_grid(p)
    assert np.array_equal(g.cells, [[0, 1], [2, 0]])


def test_hard_data_files(tmp_path):
    # test_io.cpp:129-189
    p = str(tmp_path / "hd.csv")
    spit(p, "")
    assert cio.read_hard_data(p, 8, 8).points == []
    spit(p, "# header comment\n1,2,0\n\n3,4,1\n  # indented comment\n5,6,1\n")
    hd = cio.read_hard_data(p, 8, 8)
    assert [(d.row, d.col, d.facies) for d in hd.points] == [(1, 2, 0), (3, 4, 1), (5, 6, 1)]
    spit(p, "0,0,1\n1,1,0\n0,0,1\n")
    with pytest.raises(cs.ParseError) as e:
        cio.read_hard_data(p, 8, 8)
    assert e.value.line == 3 and "duplicate" in str(e.value) and "line 1" in str(e.value)
    for bad in ("8,0,1\n", "0,-1,1\n", "1,2\n", "1,2,a\n", "1,2,-1\n", "1, 2 ,x\n"):
        spit(p, bad)
        with pytest.raises(cs.ParseError):
            cio.read_hard_data(p, 8, 8)
    spit(p, " 1 , 2 , 0 \n")  # fields are trimmed (parse_int)
    assert cio.read_hard_data(p, 8, 8).points[0] == cs.HardDatum(1, 2, 0)


def test_hard_data_roundtrip_1000(tmp_path):
    # test_io.cpp:170-188
    rng = cs.Mt19937_64(62)
    seen, pts = set(), []
    while len(pts) < 1000:
        r, c = cs.bounded(rng, 64), cs.bounded(rng, 64)
        if (r, c) not in seen:
            seen.add((r, c))
            pts.append(cs.HardDatum(r, c, cs.bounded(rng, 3)))
    p = str(tmp_path / "hd.csv")
    cio.write_hard_data(cs.HardDataSet(pts), p)
    assert cio.read_hard_data(p, 64, 64).points == pts


def test_write_pgm_bytes(tmp_path):
    # test_io.cpp:191-208
    cio.write_pgm(cs.CategoricalGrid(1, 2, 2, np.array([[0, 1]], np.uint8)), str(tmp_path / "b.pgm"))
    assert slurp(str(tmp_path / "b.pgm")) == "P2\n2 1\n255\n0 255\n"
    cio.write_pgm(cs.CategoricalGrid(1, 3, 3, np.array([[0, 1, 2]], np.uint8)), str(tmp_path / "t.pgm"))
    assert slurp(str(tmp_path / "t.pgm")) == "P2\n3 1\n255\n0 128 255\n"
    cio.write_pgm(np.array([[0.0, 0.5, 1.0]]), str(tmp_path / "r.pgm"))
    assert slurp(str(tmp_path / "r.pgm")) == "P2\n3 1\n255\n0 128 255\n"
    cio.write_pgm(cs.CategoricalGrid(1, 2, 1, np.array([[0, 0]], np.uint8)), str(tmp_path / "o.pgm"))
    assert slurp(str(tmp_path / "o.pgm")) == "P2\n2 1\n255\n0 0\n"


BASE = ("ti = ti.grid\nsg_size = 128x96\ntemplate = 32\noverlap = 8\ndwt_level = 3\n"
        "candidates = 5\nrealizations = 2\nseed = 77\n")


def test_parse_config_full_key_set(tmp_path):
    # test_io.cpp:284-305
    p = str(tmp_path / "run.cfg")
    spit(p, BASE + "scoring = normalized\nfacies_mode = raw-codes\nmin_cut = on\n"
                   "hard_data = hd.csv\nout_dir = out\n# comment\n")
    cfg = cio.parse_config(p)
    s = cfg.sim
    assert cfg.ti_path == "ti.grid"
    assert (s.sg_height, s.sg_width, s.template_size, s.overlap, s.dwt_level) == (128, 96, 32, 8, 3)
    assert (s.candidates, s.n_realizations, s.master_seed) == (5, 2, 77)
    assert s.scoring == "normalized" and s.facies_mode == "raw_codes" and s.min_cut
    assert cfg.hard_data_path == "hd.csv" and cfg.out_dir == "out"


def test_parse_config_square_and_seed_range(tmp_path):
    # test_io.cpp:307-315
    p = str(tmp_path / "run.cfg")
    spit(p, BASE)
    assert cio.parse_config(p).sim.sg_width == 96
    spit(p, "sg_size = 64\n" + BASE[BASE.find("template"):] + "ti = t.grid\n")
    cfg = cio.parse_config(p)
    assert (cfg.sim.sg_height, cfg.sim.sg_width) == (64, 64)
    spit(p, BASE.replace("seed = 77", "seed = 18446744073709551615"))
    assert cio.parse_config(p).sim.master_seed == 2**64 - 1
    spit(p, BASE.replace("seed = 77", "seed = 18446744073709551616"))
    with pytest.raises(cs.ConfigError, match="seed"):
        cio.parse_config(p)


@pytest.mark.parametrize("text,exc,needle", [
    ("ti = ti.grid\nsg_size = 128\ntemplate = 32\noverlap = 6\ndwt_level = 2\n"
     "candidates = 5\nrealizations = 1\nseed = 1\n", cs.ConfigError, "overlap"),
    (BASE[:BASE.find("seed")], cs.ConfigError, "seed"),
    (BASE + "wavelets = 3\n", cs.ConfigError, "wavelets"),
    (BASE + "min_cut = maybe\n", cs.ConfigError, "min_cut"),
    (BASE.replace("template = 32", "template = xx"), cs.ConfigError, "template"),
    (BASE + "scoring = fancy\n", cs.ConfigError, "scoring"),
    (BASE + "facies_mode = raw_codes\n", cs.ConfigError, "facies_mode"),
    (BASE.replace("sg_size = 128x96", "sg_size = 1x2x3"), cs.ConfigError, "sg_size"),
])
def test_parse_config_errors_name_the_key(tmp_path, text, exc, needle):
    # test_io.cpp:317-370
    p = str(tmp_path / "run.cfg")
    spit(p, text)
    with pytest.raises(exc) as e:
        cio.parse_config(p)
    assert needle in str(e.value)


def test_parse_config_line_numbers(tmp_path):
    # test_io.cpp:372-380
    p = str(tmp_path / "run.cfg")
    spit(p, BASE + "seed = 99\n")
    with pytest.raises(cs.ParseError) as e:
        cio.parse_config(p)
    assert e.value.line == 9 and 'duplicate key "seed"' in str(e.value)
    spit(p, "ti ti.grid\n")
    with pytest.raises(cs.ParseError):
        cio.parse_config(p)
    spit(p, " = 3\n")
    with pytest.raises(cs.ParseError, match="empty key"):
        cio.parse_config(p)


def test_parse_config_errors_follow_map_order(tmp_path):
    # apply_config_entry runs in std::map key order: "candidates" < "min_cut"
    p = str(tmp_path / "run.cfg")
    spit(p, BASE.replace("candidates = 5", "candidates = q") + "min_cut = maybe\n")
    with pytest.raises(cs.ConfigError, match="candidates"):
        cio.parse_config(p)
