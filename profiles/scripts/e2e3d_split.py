# Where the 3D e2e step (bench.py measure_3d step_e2e) spends its wall time: ccw_ti3d_create,
# ccw_simulate3d into a pinned host buffer, ccw_ti3d_destroy; and the device-output call beside it.
import os, sys, time, ctypes as C, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_00441_b200 import _abi, ccwsim as cs, ccwsim3d as c3, synth
import torch
which = int(os.environ.get("WHICH", "4"))
dev = cs.default_device(); lib = _abi.lib()
if which == 3:
    ti_a = np.ascontiguousarray(synth.config3_ti()[:, :148, :]); nf = 4
    cfg = c3.SimConfig3D(sg=(100, 200, 200), template_size=32, overlap=8, dwt_level=2, candidates=1, n_realizations=16, master_seed=20240441)
    hd_a = None
else:
    ti_a = np.ascontiguousarray(synth.config4_ti()); nf = 5
    cfg = c3.SimConfig3D(sg=(250, 500, 500), template_size=48, overlap=16, dwt_level=3, candidates=1, n_realizations=1, master_seed=20240441)
    ti0 = c3.TrainingImage3D(ti_a, nf, cfg.dwt_level, dev)
    ref_real, _ = c3.simulate3d(ti0, cfg, [777])
    hd_a = np.ascontiguousarray(synth.wells3d_from(ref_real[0], 20, 404), np.int32)
n_real = cfg.n_realizations
c = cfg.to_c()
seeds = np.array([cs.mix64(20240441, r + 1) for r in range(n_real)], np.uint64)
sgv = int(np.prod(cfg.sg))
h_pin = torch.empty(n_real * sgv, dtype=torch.uint8).pin_memory()
d_out = torch.empty(n_real * sgv, dtype=torch.uint8, device="cuda:0")
diags = (_abi.Diag3dC * n_real)()
hdp = hd_a.ctypes.data_as(_abi.I32P) if hd_a is not None and len(hd_a) else None
nhd = int(len(hd_a)) if hd_a is not None else 0
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = C.c_void_p(); d0, d1, d2 = ti_a.shape
    dev.check(lib.ccw_ti3d_create(dev.handle, ti_a.ctypes.data_as(_abi.U8P), d0, d1, d2, nf, cfg.dwt_level, C.byref(h)))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    dev.check(lib.ccw_simulate3d(dev.handle, h, C.byref(c), seeds.ctypes.data_as(_abi.U64P), n_real, hdp, nhd,
                                 C.cast(C.c_void_p(h_pin.data_ptr()), _abi.U8P), diags))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    t_dev_host = dev.last_timing()["total_ms"]
    dev.check(lib.ccw_simulate3d_device(dev.handle, h, C.byref(c), seeds.ctypes.data_as(_abi.U64P), n_real, hdp, nhd,
                                        C.c_void_p(d_out.data_ptr()), diags))
    torch.cuda.synchronize(); t3 = time.perf_counter()
    lib.ccw_ti3d_destroy(h)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print("ti3d_create %.3f ms | simulate3d(host out) %.3f ms (device %.3f) | simulate3d(device out) %.3f ms (device %.3f) | destroy %.3f" % (
        (t1 - t0) * 1e3, (t2 - t1) * 1e3, t_dev_host, (t3 - t2) * 1e3, dev.last_timing()["total_ms"], (t4 - t3) * 1e3), flush=True)
