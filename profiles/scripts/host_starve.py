# Is the per-call spread host-side? Config-1 device calls with and without a GPU-side
# head start (a spin kernel queued first, so every launch of the call is enqueued before
# the GPU reaches the call); per-call device time from the library's own events.
import os, sys, ctypes as C, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_00441_b200 import _abi, ccwsim as cs, synth
import torch
lib = _abi.lib(); dev = cs.Device(0)
grid = cs.CategoricalGrid(500, 500, 3, synth.config1_ti())
cfg = cs.SimConfig(1000, 1000, 64, 16, 2, 5, n_realizations=100, master_seed=20240441)
tih = cs.TrainingImage(grid, 2, "indicator", dev)
seeds = np.array([cs.mix64(20240441, r + 1) for r in range(100)], np.uint64)
c = cfg.to_c(); d_out = torch.empty(100 * 10**6, dtype=torch.uint8, device="cuda:0")
diags = (_abi.DiagC * 100)()
stream = torch.cuda.ExternalStream(dev.stream_ptr, device=torch.device("cuda", 0))
for head in [0, 1, 0, 1]:
    ts = []
    for i in range(12):
        if head:
            with torch.cuda.stream(stream):
                torch.cuda._sleep(20_000_000)  # ~10 ms of GPU spin ahead of the call
        dev.check(lib.ccw_simulate_device(dev.handle, tih.handle, C.byref(c), seeds.ctypes.data_as(_abi.U64P), 100, None, 0, C.c_void_p(d_out.data_ptr()), diags))
        torch.cuda.synchronize()
        ts.append(dev.last_timing()["total_ms"])
    print("head start" if head else "no head  ", " ".join("%.3f" % t for t in ts), "| mean %.3f" % (sum(ts[2:]) / len(ts[2:])), flush=True)
