# Standalone CCF screen throughput (ccw_measure_ccf_screen) at several placement counts, config 1 TI.
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2404_00441_b200 import _abi, ccwsim as cs, synth
lib = _abi.lib(); dev = cs.Device(0)
tih = cs.TrainingImage(cs.CategoricalGrid(500, 500, 3, synth.config1_ti()), 2, "indicator", dev)
peak = dev.measure_i8_peak()
npos = 110 * 110; kpad = 512
for nj in (175, 350, 700, 1400, 2800):
    ms = C.c_double()
    dev.check(lib.ccw_measure_ccf_screen(dev.handle, tih.handle, 64, nj, 30, C.byref(ms)))
    issued = 2.0 * kpad * npos * nj / (ms.value * 1e-3) / 1e12
    algo = 2.0 * 2 * 112 * npos * nj / (ms.value * 1e-3) / 1e12
    out_bytes = 4.0 * npos * nj
    print(f"njobs {nj:5d}: {ms.value*1e3:8.2f} us/launch  issued {issued:7.1f} TOPS ({issued/peak:.3f} of {peak:.0f})  algorithmic {algo:6.1f} TOPS  score bytes {out_bytes/1e6:.1f} MB -> {out_bytes/(ms.value*1e-3)/1e9:.0f} GB/s")
