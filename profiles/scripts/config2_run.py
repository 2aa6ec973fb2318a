# Config 2 (TI 2000^2, SG 4000^2, T96 OV24 J3 K1, 1 % hard data) on the device: REPS calls of N realizations.
import os, sys, ctypes as C, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_00441_b200 import _abi, ccwsim as cs, synth
import torch
lib = _abi.lib(); dev = cs.Device(0)
ti_a = synth.config2_ti(); hd = np.ascontiguousarray(synth.config2_hard_data(ti_a), np.int32)
tih = cs.TrainingImage(cs.CategoricalGrid(2000, 2000, 2, ti_a), 3, "indicator", dev)
n = int(os.environ.get("NREAL", "8"))
cfg = cs.SimConfig(4000, 4000, 96, 24, 3, 1, n_realizations=n, master_seed=20240441)
seeds = np.array([cs.mix64(20240441, r + 1) for r in range(n)], np.uint64)
c = cfg.to_c(); d_out = torch.empty(n * 16 * 10**6, dtype=torch.uint8, device="cuda:0")
diags = (_abi.DiagC * n)()
for _k in ("groups", "wave", "wave_cs", "help_min"):
    if os.environ.get(_k.upper()): dev.set_option(_k, int(os.environ[_k.upper()]))
dev.set_profiling(os.environ.get("PROF", "1") == "1")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
stream = torch.cuda.ExternalStream(dev.stream_ptr, device=torch.device("cuda", 0))
for i in range(int(os.environ.get("REPS", "3"))):
    if os.environ.get("FLUSH"):
        with torch.cuda.stream(stream):
            flush.zero_()
    dev.check(lib.ccw_simulate_device(dev.handle, tih.handle, C.byref(c), seeds.ctypes.data_as(_abi.U64P), n,
                                      hd.ctypes.data_as(_abi.I32P), hd.shape[0], C.c_void_p(d_out.data_ptr()), diags))
    torch.cuda.synchronize()
    t = dev.last_timing()
    print("total_ms %.2f rescored %d bulk_jobs %d ccf_ms %.2f select_ms %.2f launches %d" % (t["total_ms"], t["rescored"], t["bulk_jobs"], t["ccf_ms"], t["select_ms"], t["launches"]))
