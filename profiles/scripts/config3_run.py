# BASELINE configs 3 / 4 (3D) on the device: REPS calls (WHICH=3 or 4), for ncu captures of screen3d_kernel (TC3D=0) or the tcgen05 3D screen (TC3D=1, default).
import os, sys, ctypes as C, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_00441_b200 import ccwsim as cs, ccwsim3d as c3, synth
which = int(os.environ.get("WHICH", "3"))
if which == 3:
    ti_a = np.ascontiguousarray(synth.config3_ti()[:, :148, :])
    cfg = c3.SimConfig3D(sg=(100, 200, 200), template_size=32, overlap=8, dwt_level=2, candidates=1,
                         n_realizations=16, master_seed=20240441)
    nf = 4
else:
    ti_a = synth.config4_ti()
    cfg = c3.SimConfig3D(sg=(250, 500, 500), template_size=48, overlap=16, dwt_level=3, candidates=1,
                         n_realizations=1, master_seed=20240441)
    nf = 5
dev = cs.default_device()
ti = c3.TrainingImage3D(ti_a, nf, cfg.dwt_level, dev)
dev.set_option("tc3d", int(os.environ.get("TC3D", "1")))
dev.set_profiling(os.environ.get("PROF", "1") == "1")
for i in range(int(os.environ.get("REPS", "2"))):
    c3.simulate3d_ensemble(ti, cfg)
    t = dev.last_timing()
    print("total_ms %.2f screen_ms %.2f launches %d" % (t["total_ms"], t["ccf_ms"], t["launches"]))
