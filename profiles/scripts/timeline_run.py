# Config-1 simulate calls on the device (REPS of them) for CCW_TIMELINE / CCW_TAIL / CCW_GROUPS experiments.
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
if os.environ.get("GROUPS"): dev.set_option("groups", int(os.environ["GROUPS"]))
for _k in ("wave", "wave_cs"):
    if os.environ.get(_k.upper()): dev.set_option(_k, int(os.environ[_k.upper()]))
for i in range(int(os.environ.get("REPS", "4"))):
    dev.check(lib.ccw_simulate_device(dev.handle, tih.handle, C.byref(c), seeds.ctypes.data_as(_abi.U64P), 100, None, 0, C.c_void_p(d_out.data_ptr()), diags))
    torch.cuda.synchronize()
    print("total_ms", dev.last_timing()["total_ms"], file=sys.stderr)
