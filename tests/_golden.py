"""Loaders for tests/golden/*.npz (written by oracle/gen_golden.py from the
compiled reference)."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sim_cases():
    out = []
    for path in sorted(glob.glob(os.path.join(GOLDEN, "sim_*.npz"))):
        z = np.load(path)
        cfg = dict(zip([str(k) for k in z["cfg_keys"]], [int(v) for v in z["cfg_vals"]]))
        seeds = [int(s) for s in z["seeds"]]
        hd = z["hd"].reshape(-1, 3)
        case = {"name": os.path.basename(path)[4:-4], "ti": z["ti"], "nf": int(z["nf"]),
                "cfg": cfg, "hd": [tuple(int(x) for x in row) for row in hd] if len(hd) else None,
                "seeds": seeds, "real": [z[f"real_{i}"] for i in range(len(seeds))],
                "mism": [int(z[f"mism_{i}"]) for i in range(len(seeds))],
                "origin": [int(z[f"origin_{i}"]) for i in range(len(seeds))],
                "colmajor": [int(z[f"colmajor_{i}"]) for i in range(len(seeds))],
                "ti_row": [z[f"ti_row_{i}"] for i in range(len(seeds))],
                "ti_col": [z[f"ti_col_{i}"] for i in range(len(seeds))]}
        out.append(case)
    return out


def load(name):
    return np.load(os.path.join(GOLDEN, name))
