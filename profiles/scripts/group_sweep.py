# Config-1 device time per call for several realization-group counts (option `groups`)
# and, with a debug build (CCW_LIB_VARIANT), CCF grid caps (CCW_TC_GRID).
import os, sys, ctypes as C, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_00441_b200 import _abi, ccwsim as cs, synth
import torch
lib = _abi.lib(); dev = cs.Device(0)
ti_a = synth.config1_ti(); grid = cs.CategoricalGrid(500, 500, 3, ti_a)
cfg = cs.SimConfig(1000, 1000, 64, 16, 2, 5, n_realizations=100, master_seed=20240441)
tih = cs.TrainingImage(grid, 2, "indicator", dev)
seeds = np.array([cs.mix64(20240441, r + 1) for r in range(100)], np.uint64)
c = cfg.to_c(); d_out = torch.empty(100 * 10**6, dtype=torch.uint8, device="cuda:0")
diags = (_abi.DiagC * 100)()
ref = None
if os.environ.get("HELP_MIN"): dev.set_option("help_min", int(os.environ["HELP_MIN"]))
if os.environ.get("FLAGPREP"): dev.set_option("flagprep", int(os.environ["FLAGPREP"]))
for G in [int(g) for g in os.environ.get("GROUPS", "1,2,3,4").split(",")]:
    dev.set_option("groups", G)
    ts = []
    for i in range(int(os.environ.get("REPS", "6"))):
        dev.check(lib.ccw_simulate_device(dev.handle, tih.handle, C.byref(c), seeds.ctypes.data_as(_abi.U64P), 100, None, 0, C.c_void_p(d_out.data_ptr()), diags))
        torch.cuda.synchronize()
        ts.append(dev.last_timing()["total_ms"])
    h = d_out[:4 * 10**6].cpu().numpy()
    if ref is None: ref = h
    print("groups", G, "grid", os.environ.get("CCW_TC_GRID", "-"), "ms", " ".join("%.3f" % t for t in ts), "min %.3f" % min(ts[1:]), "same", bool((h == ref).all()), flush=True)
