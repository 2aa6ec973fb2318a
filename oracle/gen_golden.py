"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

TEST INFRASTRUCTURE.  Run here (where /root/reference exists):

    make -C oracle && python oracle/gen_golden.py

The reference ships no stored golden files, so these fixtures are
outputs of the reference's own code on seeded inputs built with the
reference's own test-support generators (tests/support/synthetic.hpp).  They
pin the C restatement (tests/test_oracle_pins.py) and the CUDA path
(tests/test_gpu_*.py) without needing /root/reference at test time.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import pyoracle  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def sim_cases():
    """(name, ti-spec, nf, cfg dict, hard data, seeds)."""
    base = dict(sg_height=64, sg_width=64, template_size=16, overlap=4, dwt_level=2,
                candidates=4, n_realizations=1, scoring=0, facies_mode=0, min_cut=0,
                master_seed=1234)

    def c(**kw):
        d = dict(base)
        d.update(kw)
        return d
    hd3 = [(3, 3, 1), (40, 51, 0), (17, 28, 1)]
    hd_rand = [(5, 7, 2), (33, 12, 0), (60, 10, 1), (21, 44, 2), (47, 47, 1), (2, 50, 0)]
    return [
        ("channel64_base", ("channel", 64, 64, 3), 2, c(), None, [31337, 5, 77]),
        ("channel64_pad", ("channel", 64, 64, 11), 2, c(sg_height=52, sg_width=70), None, [2024]),
        ("channel64_k1", ("channel", 64, 64, 13), 2, c(candidates=1), None, [9, 10]),
        ("channel64_mincut", ("channel", 64, 64, 17), 2, c(min_cut=1), None, [1, 2]),
        ("channel64_rawcodes", ("channel", 64, 64, 19), 2, c(facies_mode=1), None, [3]),
        ("channel64_normalized", ("channel", 64, 64, 23), 2, c(scoring=1), None, [4]),
        ("channel64_hd", ("channel", 64, 64, 19), 2, c(candidates=8), hd3, [4242]),
        ("random3_hd_mincut", ("random", 64, 64, 3, 7), 3,
         c(sg_height=70, sg_width=52, candidates=3, min_cut=1), hd_rand, [99, 100]),
        ("random4_rawcodes_norm", ("random", 48, 48, 4, 8), 4,
         c(sg_height=40, sg_width=56, template_size=8, overlap=2, dwt_level=1, candidates=5,
           facies_mode=1, scoring=1), None, [7]),
        ("channel128_J3", ("channel", 128, 128, 1313), 2,
         c(sg_height=96, sg_width=96, template_size=32, overlap=8, dwt_level=3, candidates=5),
         None, [9001, 9002]),
        ("channel128_J1_T2OV", ("channel", 128, 128, 1414), 2,
         c(sg_height=60, sg_width=60, template_size=12, overlap=8, dwt_level=1, candidates=2),
         None, [55]),
        ("const_ti", ("const", 32, 32, 1), 2, c(sg_height=48, sg_width=48), None, [999]),
    ]


def make_ti(ref, spec):
    kind = spec[0]
    if kind == "channel":
        return ref.make_channel_ti(spec[1], spec[2], spec[3])
    if kind == "random":
        return ref.random_grid(spec[1], spec[2], spec[3], spec[4])
    if kind == "const":
        return np.full((spec[1], spec[2]), spec[3], np.uint8)
    raise ValueError(kind)


def main() -> None:
    ref = pyoracle.reference()
    os.makedirs(OUT, exist_ok=True)

    # -- simulations ------------------------------------------------------
    for name, spec, nf, cfgd, hd, seeds in sim_cases():
        ti = make_ti(ref, spec)
        cfg = pyoracle.Cfg(**cfgd)
        blobs = {"ti": ti, "nf": np.int32(nf), "seeds": np.array(seeds, np.uint64),
                 "cfg_keys": np.array(list(cfgd.keys())),
                 "cfg_vals": np.array([int(v) for v in cfgd.values()], np.uint64),
                 "hd": np.array(hd if hd else np.zeros((0, 3)), np.int32).reshape(-1, 3)}
        for i, s in enumerate(seeds):
            r = ref.simulate_one(ti, nf, cfg, hd, seed=s, trace=True)
            blobs[f"real_{i}"] = r["realization"]
            blobs[f"mism_{i}"] = np.int32(r["diagnostics"]["pre_overwrite_mismatches"])
            blobs[f"origin_{i}"] = np.int32(r["diagnostics"]["origin"])
            blobs[f"colmajor_{i}"] = np.int32(r["diagnostics"]["column_major"])
            blobs[f"ti_row_{i}"] = r["trace"]["ti_row"]
            blobs[f"ti_col_{i}"] = r["trace"]["ti_col"]
        np.savez_compressed(os.path.join(OUT, f"sim_{name}.npz"), **blobs)

    # ensemble (simulate_ensemble seeds mix64(master, r+1), workers 1 vs 4)
    ti = ref.make_channel_ti(64, 64, 23)
    cfg = pyoracle.Cfg(n_realizations=6)
    e1, _ = ref.simulate_ensemble(ti, 2, cfg, None, workers=1)
    e4, _ = ref.simulate_ensemble(ti, 2, cfg, None, workers=4)
    assert np.array_equal(e1, e4)
    np.savez_compressed(os.path.join(OUT, "ensemble_channel64.npz"), ti=ti, real=e1,
                        master=np.uint64(cfg.master_seed))

    # -- wavelet ----------------------------------------------------------
    wav = {}
    for i, (h, w, lv, seed) in enumerate([(8, 8, 1, 22), (16, 16, 2, 23), (16, 16, 3, 23),
                                          (24, 40, 3, 101), (64, 64, 3, 26), (6, 4, 1, 5)]):
        x = ref.random_plane(h, w, seed)
        apex, det = ref.dwt2(x, lv)
        wav[f"x_{i}"] = x
        wav[f"lv_{i}"] = np.int32(lv)
        wav[f"apex_{i}"] = apex
        wav[f"det_{i}"] = np.concatenate([np.ravel(p) for lvl in det for p in lvl])
        wav[f"back_{i}"] = ref.idwt2(apex, det, h, w, lv)
        a, dh, dv, dd = ref.dwt2_single(x)
        wav[f"single_{i}"] = np.stack([a, dh, dv, dd])
    # binary planes (the simulator's indicator inputs)
    g = ref.random_grid(32, 32, 2, 77).astype(np.float64)
    for lv in (1, 2, 3):
        wav[f"bin_apex_{lv}"] = ref.dwt2(g, lv)[0]
    wav["bin"] = g
    np.savez_compressed(os.path.join(OUT, "wavelet.npz"), **wav)

    # -- matcher ----------------------------------------------------------
    mat = {}
    rng = np.random.default_rng(33)
    for i in range(12):
        th, tw = int(rng.integers(2, 6)), int(rng.integers(2, 6))
        ih, iw = th + 4 + int(rng.integers(0, 9)), tw + 4 + int(rng.integers(0, 9))
        nch = int(rng.integers(1, 4))
        ti = np.stack([ref.random_plane(ih, iw, 1000 + 10 * i + f) for f in range(nch)])
        mask = (rng.integers(0, 2, (th, tw)) == 1).astype(np.float64)
        mask[0, 0] = 1.0
        tm = np.stack([ref.random_plane(th, tw, 2000 + 10 * i + f) for f in range(nch)]) * mask
        scoring = i % 2
        mat[f"ti_{i}"] = ti
        mat[f"tm_{i}"] = tm
        mat[f"mask_{i}"] = mask
        mat[f"scoring_{i}"] = np.int32(scoring)
        mat[f"out_{i}"] = ref.score_map_channels(ti, tm, mask, scoring)
    for i in range(6):
        s = rng.integers(0, 50, (20, 20)).astype(np.float64)
        k = int(rng.integers(1, 12))
        mat[f"topk_s_{i}"] = s
        mat[f"topk_k_{i}"] = np.int32(k)
        mat[f"topk_{i}"] = np.array(ref.top_k(s, k), np.float64)
    np.savez_compressed(os.path.join(OUT, "matcher.npz"), **mat)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
