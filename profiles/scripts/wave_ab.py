# Config-1 device calls with the fused wave kernel on and off: timing and equality.
import os, sys, ctypes as C, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_00441_b200 import _abi, ccwsim as cs, synth
import torch
lib = _abi.lib(); dev = cs.Device(0)
ti_a = synth.config1_ti(); grid = cs.CategoricalGrid(500, 500, 3, ti_a)
NR = int(os.environ.get("NR", "100"))
cfg = cs.SimConfig(1000, 1000, 64, 16, 2, 5, n_realizations=NR, master_seed=20240441)
tih = cs.TrainingImage(grid, 2, "indicator", dev)
seeds = np.array([cs.mix64(20240441, r + 1) for r in range(NR)], np.uint64)
c = cfg.to_c(); d_out = torch.empty(NR * 10**6, dtype=torch.uint8, device="cuda:0")
diags = (_abi.DiagC * NR)()
outs = {}
for wave in [0, 1]:
    dev.set_option("wave", wave)
    for cs_ in ([0] if wave == 0 else [int(x) for x in os.environ.get("CS", "0").split(",")]):
        dev.set_option("wave_cs", cs_)
        ts = []
        for i in range(int(os.environ.get("REPS", "5"))):
            dev.check(lib.ccw_simulate_device(dev.handle, tih.handle, C.byref(c), seeds.ctypes.data_as(_abi.U64P), NR, None, 0, C.c_void_p(d_out.data_ptr()), diags))
            torch.cuda.synchronize()
            ts.append(dev.last_timing()["total_ms"])
        h = d_out.cpu().numpy().copy()
        t = dev.last_timing()
        outs[(wave, cs_)] = h
        same = bool((h == outs[(0, 0)]).all())
        nbad = int((h.reshape(NR, -1) != outs[(0, 0)].reshape(NR, -1)).any(axis=1).sum())
        print("wave", wave, "cs", cs_, "ms", " ".join("%.3f" % x for x in ts), "same", same, "bad_real", nbad,
              "fallbacks", t.get("list_overflows"), "rescored", t.get("rescored"), "screened", t.get("screened_jobs"), flush=True)
