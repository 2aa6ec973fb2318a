# Where the config-1 e2e step (bench.py step_e2e) spends its wall time: ti_create, simulate with
# host output (the streamed bands), ti_destroy; and the same simulate on a kept TI handle.
import os, sys, time, ctypes as C, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_00441_b200 import _abi, ccwsim as cs, synth
import torch
lib = _abi.lib(); dev = cs.Device(0)
ti_a = np.ascontiguousarray(synth.config1_ti())
cfg = cs.SimConfig(1000, 1000, 64, 16, 2, 5, n_realizations=100, master_seed=20240441)
c = cfg.to_c()
seeds = np.array([cs.mix64(20240441, r + 1) for r in range(100)], np.uint64)
h_out = torch.empty(100 * 10**6, dtype=torch.uint8).pin_memory()
diags = (_abi.DiagC * 100)()
for _k in ("stream_bands", "place_threads", "groups", "pack"):
    if os.environ.get(_k.upper()): dev.set_option(_k, int(os.environ[_k.upper()]))
def sim(h):
    dev.check(lib.ccw_simulate(dev.handle, h, C.byref(c), seeds.ctypes.data_as(_abi.U64P), 100, None, 0,
                               C.cast(C.c_void_p(h_out.data_ptr()), _abi.U8P), diags, None))
res_t = []
for rep in range(int(os.environ.get("REPS", "4"))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = C.c_void_p()
    dev.check(lib.ccw_ti_create(dev.handle, ti_a.ctypes.data_as(_abi.U8P), 500, 500, 3, 2, 0, C.byref(h)))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    sim(h)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    t = dev.last_timing()
    sim(h)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    t_b = dev.last_timing()
    lib.ccw_ti_destroy(h)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    res_t.append((t4 - t0) * 1e3)
    if os.environ.get("QUIET"): continue
    print("ti_create %.3f ms | simulate(first on handle) %.3f ms (device %.3f, host_prep %.3f) | simulate(kept handle) %.3f ms (device %.3f) | destroy %.3f ms | d2h %d B" % (
        (t1 - t0) * 1e3, (t2 - t1) * 1e3, t["total_ms"], t["host_prep_ms"], (t3 - t2) * 1e3, t_b["total_ms"], (t4 - t3) * 1e3, t["d2h_bytes"]), flush=True)
print("e2e step ms: median %.3f min %.3f (%s)" % (sorted(res_t)[len(res_t) // 2], min(res_t), " ".join(f"{k}={os.environ[k]}" for k in ("STREAM_BANDS", "PLACE_THREADS", "CCW_STREAM_TAIL") if k in os.environ)))
