#!/usr/bin/env python
"""Benchmark: simulated cells/s on BASELINE config 1 (the headline workload).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload config1|single] [--virtual-shards V]

Workload (BASELINE.json configs[1]): TI 500x500 3-facies (channels + levee
lenses, synth.config1_ti), SG 1000x1000, T=64, OV=16, J=2, K=5 top-k random
pick, unconditional, 100 realizations per GPU (weak scaling: rank r simulates
realizations r*100 .. r*100+99 with seeds mix64(master, index + 1)).

A step = one batched simulation of those 100 realizations.
  value : cells/s with the TI pyramid resident in HBM and realizations left in
          HBM (ccw_simulate_device); per-step CUDA events on the library's
          stream, L2 flushed (256 MiB write) before every timed step.
  e2e   : the same metric through the public C-ABI call with host buffers:
          ccw_ti_create from host bytes (H2D + pyramid) + ccw_simulate into
          pinned host memory (D2H of every realization), wall clock per step.
  parity: after the timed region, the first 8 realizations of the last timed
          call are checked bit for bit against the compiled reference
          (oracle/_ref, the unmodified reference headers) with the same seeds.
  config2: at N=1 the same measurements on BASELINE config 2 (TI 2000^2,
          SG 4000^2, T96 OV24 J3 K1, 1 % hard data, 8 realizations), the
          largest single-GPU configuration, nested in the same line.
Rank 0 prints one JSON line.  --impl reference times the reference's own CPU
implementation (oracle/_ref: the unmodified reference headers) on the host
cores on a bounded sample of the same workload.

--gpus N without torchrun: bench.py spawns the N ranks itself (one process
per GPU, NCCL over 127.0.0.1), so `python bench.py --gpus N` and
`torchrun --nproc-per-node N bench.py --gpus N` measure the same thing.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated cells/s"
UNIT = "cells/s"
REAL_PER_GPU = 100
MASTER = 20240441
WORKLOAD = ("config1: TI 500x500 3-facies, SG 1000x1000, T64 OV16 J2 K5 random top-k pick, "
            f"{REAL_PER_GPU} realizations per GPU")


def cfg1():
    from paper_2404_00441_b200 import ccwsim as cs
    return cs.SimConfig(sg_height=1000, sg_width=1000, template_size=64, overlap=16, dwt_level=2,
                        candidates=5, n_realizations=REAL_PER_GPU, master_seed=MASTER)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_traffic():
    path = os.path.join(ROOT, "profiles", "ccf_traffic.json")
    if os.path.exists(path):
        try:
            return json.load(open(path))
        except Exception:
            return None
    return None


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_impl():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    if pyoracle.reference_available():
        return pyoracle, pyoracle.reference(), "reference"
    return pyoracle, pyoracle.restatement(), "port"


def check_parity(got, ti, nf, cfg, seeds, hd=None, n_check=8):
    """Bit-exact check of benchmarked realizations against the compiled
    reference (oracle/_ref), same seeds, host threads in parallel."""
    from concurrent.futures import ThreadPoolExecutor
    pyoracle, impl, kind = reference_impl()
    c = pyoracle.Cfg(sg_height=cfg.sg_height, sg_width=cfg.sg_width,
                     template_size=cfg.template_size, overlap=cfg.overlap,
                     dwt_level=cfg.dwt_level, candidates=cfg.candidates)
    idx = list(range(min(n_check, len(seeds))))

    def one(r):
        o = impl.simulate_one(ti, nf, c, hd, seed=int(seeds[r]))
        return bool(np.array_equal(got[r], o["realization"]))

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=min(len(idx), os.cpu_count() or 1)) as ex:
        ok = list(ex.map(one, idx))
    return {"checked": len(idx), "equal": all(ok), "mismatched": [r for r, v in zip(idx, ok) if not v],
            "against": f"oracle/_ref ({kind}: compiled unmodified reference headers)" if kind == "reference"
                       else "oracle restatement (reference not built)",
            "what": "realizations 0..%d of the last timed call, same seeds" % (len(idx) - 1),
            "seconds": round(time.perf_counter() - t0, 2)}


def cpu_reference_rate(ti, nf, cfg, n_real, workers, hd=None, master=None):
    """cells/s of the compiled reference (oracle/_ref) on n_real realizations
    (simulate_ensemble: seeds mix64(master, r+1)); also returns them."""
    pyoracle, impl, kind = reference_impl()
    c = pyoracle.Cfg(sg_height=cfg.sg_height, sg_width=cfg.sg_width,
                     template_size=cfg.template_size, overlap=cfg.overlap,
                     dwt_level=cfg.dwt_level, candidates=cfg.candidates,
                     n_realizations=n_real, master_seed=cfg.master_seed if master is None else master)
    t0 = time.perf_counter()
    out, _ = impl.simulate_ensemble(ti, nf, c, hd, workers=workers)
    dt = time.perf_counter() - t0
    return n_real * cfg.sg_height * cfg.sg_width / dt, dt, kind, out


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2404_00441_b200 import synth
    ti = synth.config1_ti()
    cfg = cfg1()
    cores = os.cpu_count() or 1
    sample = max(cores, 4)  # one realization per host thread per step
    for _ in range(args.warmup):
        cpu_reference_rate(ti, 3, cfg, min(sample, 4), cores)[:3]
    rates, times = [], []
    kind = "reference"
    for _ in range(args.steps):
        r, dt, kind, _ = cpu_reference_rate(ti, 3, cfg, sample, cores)
        rates.append(r)
        times.append(dt)
    value = statistics.median(rates)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "sample_realizations_per_step": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "cpu_model": cpu_model(),
                             "sample": f"{sample} config-1 realizations per step, "
                                       f"simulate_ensemble(workers={cores})"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2404_00441_b200 import _abi, ccwsim as cs, synth

    lib = _abi.lib()
    dev = cs.Device(local)
    stream = torch.cuda.ExternalStream(dev.stream_ptr, device=torch.device("cuda", local))
    ti_a = synth.config1_ti()
    nf = 3
    cfg = cfg1()
    grid = cs.CategoricalGrid(500, 500, nf, ti_a)
    tih = cs.TrainingImage(grid, cfg.dwt_level, "indicator", dev)
    base = rank * REAL_PER_GPU
    seeds = np.array([cs.mix64(MASTER, base + r + 1) for r in range(REAL_PER_GPU)], np.uint64)
    c = cfg.to_c()
    sg = cfg.sg_height * cfg.sg_width
    d_out = torch.empty(REAL_PER_GPU * sg, dtype=torch.uint8, device=f"cuda:{local}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    diags = (_abi.DiagC * REAL_PER_GPU)()

    def step_device():
        dev.check(lib.ccw_simulate_device(dev.handle, tih.handle, C.byref(c),
                                          seeds.ctypes.data_as(_abi.U64P), REAL_PER_GPU, None, 0,
                                          C.c_void_p(d_out.data_ptr()), diags))

    def step_device_async():  # (timed steps: a call's host planning overlaps the previous call's device work)
        dev.check(lib.ccw_simulate_device_async(dev.handle, tih.handle, C.byref(c),
                                                seeds.ctypes.data_as(_abi.U64P), REAL_PER_GPU, None, 0,
                                                C.c_void_p(d_out.data_ptr())))

    # warm-up: the same flush + call as a timed step (the flush buffer's first
    # touch is not left to the first timed step)
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        step_device()
    torch.cuda.synchronize()

    # device-resident timed region
    sampler = ClockSampler(local)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush (256 MiB > 126 MB L2), outside the events
            evs[k][0].record(stream)
        step_device_async()
        with torch.cuda.stream(stream):
            evs[k][1].record(stream)
    dev.synchronize()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    if os.environ.get("CCW_BENCH_STEPS"):  # diagnostics: every timed step's device time
        print("step ms: " + " ".join(f"{t:.3f}" for t in step_ms), file=sys.stderr)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    timing = dev.last_timing()
    launches_per_step = int(timing["launches"])
    cells = world * REAL_PER_GPU * sg * args.steps
    value = cells / (total_ms * 1e-3)

    # parity: the last timed call's realizations against the compiled reference
    got = d_out.view(REAL_PER_GPU, cfg.sg_height, cfg.sg_width).cpu().numpy()
    parity = check_parity(got, ti_a, nf, cfg, seeds) if rank == 0 else None

    # profiling pass (separate from the timed region): per-launch CCF time
    dev.set_profiling(True)
    step_device()
    prof = dev.last_timing()
    dev.set_profiling(False)
    ccf_avg_ms = prof["ccf_ms"] / max(prof["ccf_launches"], 1)
    # SURVEY 8(d) numerator: 2 x F channels x positions x mask cells per placement
    flop_per_launch = prof["ccf_flop_ref"] / max(prof["ccf_launches"], 1)
    screen_per_launch = prof["ccf_flop"] / max(prof["ccf_launches"], 1)
    mma_per_launch = prof["ccf_mma_flop"] / max(prof["ccf_launches"], 1)
    tensor = prof["ccf_variant"] == 2
    peak = dev.measure_i8_peak() if tensor else dev.measure_fp32_peak()
    achieved = flop_per_launch / (ccf_avg_ms * 1e-3) / 1e12
    traffic = load_traffic()
    # the screen kernel alone (no wave dependency, back-to-back launches) on
    # 1400 placements: what it reaches when it is not on the latency chain
    standalone = None
    if tensor:
        nj_sa, kpad_sa, npos_sa = 1400, 512, 110 * 110
        sa_ms = C.c_double()
        dev.check(lib.ccw_measure_ccf_screen(dev.handle, tih.handle, cfg.template_size, nj_sa, 30,
                                             C.byref(sa_ms)))
        sa_s = sa_ms.value * 1e-3
        standalone = {
            "placements_per_launch": nj_sa, "us_per_launch": sa_ms.value * 1e3,
            "mma_tops_issued": 2.0 * kpad_sa * npos_sa * nj_sa / sa_s / 1e12,
            "algorithmic_tops": 2.0 * nf * 112 * npos_sa * nj_sa / sa_s / 1e12,
            "frac": 2.0 * nf * 112 * npos_sa * nj_sa / sa_s / 1e12 / peak if peak else None,
            "note": "same kernel, 1400 L-shaped placements' weights per launch, no wave dependency"}
    # end-to-end through the public API with host buffers
    h_out = torch.empty(REAL_PER_GPU * sg, dtype=torch.uint8).pin_memory()
    ti_host = np.ascontiguousarray(ti_a)

    def step_e2e():
        h = C.c_void_p()
        dev.check(lib.ccw_ti_create(dev.handle, ti_host.ctypes.data_as(_abi.U8P), 500, 500, nf,
                                    cfg.dwt_level, 0, C.byref(h)))
        dev.check(lib.ccw_simulate(dev.handle, h, C.byref(c), seeds.ctypes.data_as(_abi.U64P),
                                   REAL_PER_GPU, None, 0,
                                   C.cast(C.c_void_p(h_out.data_ptr()), _abi.U8P), diags, None))
        lib.ccw_ti_destroy(h)

    step_e2e()
    e2e_times = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step_e2e()
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_times)
    d2h_bytes = int(dev.last_timing()["d2h_bytes"])
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_s], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = cells / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cores = os.cpu_count() or 1
        n = max(cores, 4)
        rate, dt, kind, _ = cpu_reference_rate(ti_a, nf, cfg, n, cores)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind, "cpu_model": cpu_model(),
               "sample": f"{n} config-1 realizations, simulate_ensemble(workers={cores}), "
                         f"{dt:.1f} s wall"}

    config2 = config3 = config4 = shim = None
    if world == 1 and not args.skip_cpu:
        shim = measure_shim(ti_a, max(3, min(args.steps, 10)))
    if world == 1 and not args.skip_config2:
        config2 = measure_config2(dev, lib, local, args, skip_cpu=args.skip_cpu)
    if world == 1 and not args.skip_3d:
        config3 = measure_3d(3, dev, lib, local, args, skip_cpu=args.skip_cpu)
        config4 = measure_3d(4, dev, lib, local, args, skip_cpu=args.skip_cpu)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "i8xi8->i32 screen + f64 rescoring", "data": "synthetic",
            "config": {"workload": WORKLOAD, "realizations_per_gpu": REAL_PER_GPU,
                       "parallelism": f"realization shards x{world}",
                       "l2": "flushed before each timed step (256 MiB write, outside events)",
                       "timing": "per-step CUDA events on the library stream, max over ranks; timed calls through "
                                 "ccw_simulate_device_async (each call's host planning overlaps the previous "
                                 "call's device work; synchronized before the first and after the last step)"},
            "roofline": {"bound": "tensor" if tensor else "fp32",
                         "kernel": "ccf_tc_kernel (tcgen05 kind::i8)" if tensor else "ccf_direct_kernel",
                         "achieved": achieved, "peak": peak,
                         "unit": "TOPS" if tensor else "TFLOP/s",
                         "frac": achieved / peak if peak else None,
                         "peak_source": ("measured in this run: tcgen05 kind::i8 MMA probe, the screen's "
                                         "M=128 N=256 shape, one CTA per SM (ccw_measure_i8_peak; "
                                         "MEASURED_PEAKS.json has only bf16)") if tensor else
                                        "measured in this run: FFMA probe (MEASURED_PEAKS.json has no FP32 figure)",
                         "algorithmic_ops_per_launch": flop_per_launch,
                         "algorithmic_ops_note": "SURVEY 8(d): 2 x F channels x TI window positions x coarse "
                                                 "mask cells per placement, summed over the launch's placements",
                         "screen_ops_per_launch": screen_per_launch,
                         "screen_ops_note": "the int8 screen computes F-1 channels (exact: one-hot TI)",
                         "mma_ops_issued_per_launch": mma_per_launch,
                         "avg_launch_ms": ccf_avg_ms,
                         "traffic": traffic.get("bytes_per_launch") if traffic else None,
                         "traffic_source": traffic.get("source") if traffic else None,
                         "step_ms_profiled": prof["total_ms"],
                         "ccf_ms_per_step": prof["ccf_ms"], "select_ms_per_step": prof["select_ms"],
                         "fp64_windows_rescored": prof["rescored"],
                         "standalone": standalone},
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e_shim": shim,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(ti_host.nbytes + seeds.nbytes),
                    "d2h_bytes_per_step": d2h_bytes,
                    "d2h_note": "realizations streamed as bit-packed bands (2 bits per cell for 3 facies), "
                                "unpacked by host threads into the caller's buffer"},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "config2": config2,
            "config3": config3,
            "config4": config4,
        }
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def measure_3d(which, dev, lib, local, args, skip_cpu=False):
    """BASELINE configs 3 / 4 (the 3D extension, oracle/ccw3d_oracle.h):
    device-resident cells/s, e2e through ccw_ti3d_create + ccw_simulate3d
    with host buffers, the screen's roofline against the measured integer
    peak of its inner loop, and the 3D CPU restatement (oracle, "port") on a
    bounded sample whose outputs double as the parity check."""
    import torch
    from paper_2404_00441_b200 import _abi, ccwsim as cs, ccwsim3d as c3, synth
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle3d as P3
    if which == 3:
        ti_a = np.ascontiguousarray(synth.config3_ti()[:, :148, :])  # 180x148x120
        nf, n_real, wells = 4, 16, None
        cfg = c3.SimConfig3D(sg=(100, 200, 200), template_size=32, overlap=8, dwt_level=2, candidates=1,
                             n_realizations=n_real, master_seed=MASTER)
        label = ("config3: TI 180x148x120 (x,y,z; 150 -> 148 so 2^J divides it, SURVEY H4(i)) 4-facies "
                 "ellipsoidal lenses, SG 200x200x100, T32 OV8 J2 K1, 16 realizations")
    else:
        ti_a = synth.config4_ti()
        nf, n_real = 5, 1
        cfg = c3.SimConfig3D(sg=(250, 500, 500), template_size=48, overlap=16, dwt_level=3, candidates=1,
                             n_realizations=1, master_seed=MASTER)
        label = ("config4: TI 400x400x200 (x,y,z) 5-facies channel belts + lenses, SG 500x500x250, "
                 "T48 OV16 (12 -> 16 so 2^J divides it, SURVEY H4(i)) J3 K1, 20 vertical wells, 1 realization")
    ti = c3.TrainingImage3D(ti_a, nf, cfg.dwt_level, dev)
    if which == 4:
        ref_real, _ = c3.simulate3d(ti, cfg, [777])
        wells = synth.wells3d_from(ref_real[0], 20, 404)
    hd_a = np.ascontiguousarray(wells, np.int32) if wells is not None else None
    seeds = np.array([cs.mix64(MASTER, r + 1) for r in range(n_real)], np.uint64)
    sgv = int(np.prod(cfg.sg))
    c = cfg.to_c()
    d_out = torch.empty(n_real * sgv, dtype=torch.uint8, device=f"cuda:{local}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    diags = (_abi.Diag3dC * n_real)()
    stream = torch.cuda.ExternalStream(dev.stream_ptr, device=torch.device("cuda", local))
    hdp = hd_a.ctypes.data_as(_abi.I32P) if hd_a is not None else None
    nhd = hd_a.shape[0] if hd_a is not None else 0

    def step_device():
        dev.check(lib.ccw_simulate3d_device(dev.handle, ti.handle, C.byref(c), seeds.ctypes.data_as(_abi.U64P),
                                            n_real, hdp, nhd, C.c_void_p(d_out.data_ptr()), diags))

    for _ in range(max(args.warmup, 3)):
        with torch.cuda.stream(stream):
            flush.zero_()
        step_device()
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 10))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            evs[k][0].record(stream)
        step_device()
        with torch.cuda.stream(stream):
            evs[k][1].record(stream)
    torch.cuda.synchronize()
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    launches = int(dev.last_timing()["launches"])
    got = d_out.view(n_real, *cfg.sg).cpu().numpy()
    dev.set_profiling(True)
    step_device()
    prof = dev.last_timing()
    dev.set_profiling(False)
    # tcgen05 int8 screen over the 3D im2col (option tc3d): 6 int8 counts, 7 9-bit counts as two digits
    tc3 = prof["ccf_variant"] in (6, 7)
    digits = prof["ccf_variant"] == 7
    kind = 1 if prof["ccf_variant"] == 3 else 0
    peak = dev.measure_i8_peak() if tc3 else dev.measure_int_peak(kind)
    achieved = prof["ccf_flop"] / (prof["ccf_ms"] * 1e-3) / 1e12 if prof["ccf_ms"] else None
    h_out = np.zeros(n_real * sgv, np.uint8)
    h_pin = torch.empty(n_real * sgv, dtype=torch.uint8).pin_memory()

    def step_e2e():
        h = C.c_void_p()
        d0, d1, d2 = ti_a.shape
        dev.check(lib.ccw_ti3d_create(dev.handle, ti_a.ctypes.data_as(_abi.U8P), d0, d1, d2, nf, cfg.dwt_level,
                                      C.byref(h)))
        dev.check(lib.ccw_simulate3d(dev.handle, h, C.byref(c), seeds.ctypes.data_as(_abi.U64P), n_real, hdp, nhd,
                                     C.cast(C.c_void_p(h_pin.data_ptr()), _abi.U8P), diags))
        lib.ccw_ti3d_destroy(h)

    step_e2e()
    e2e_s = 0.0
    for _ in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step_e2e()
        torch.cuda.synchronize()
        e2e_s += time.perf_counter() - t0
    e2e_equal = bool(np.array_equal(h_pin.numpy().reshape(got.shape), got))
    out = {"workload": label, "value": n_real * sgv * steps / (total_ms * 1e-3), "unit": UNIT,
           "ms_per_step": total_ms / steps, "steps": steps, "gpu_launches": launches * steps,
           "dtype": ("i8xi8->i32 tcgen05, 9-bit counts as two int8 digits (exact)" if digits else
                     "i8xi8->i32 tcgen05 (exact)") if tc3 else
                    "int8x4 dp4a -> int32 (exact)" if kind == 1 else "int32 IMAD (exact)",
           "roofline": {"bound": "tensor" if tc3 else "int (CUDA cores)",
                        "kernel": ("ccf_tc_kernel (tcgen05 kind::i8 over the two-digit 3D im2col, three rows per "
                                   "placement) + keys3d_digits_kernel" if digits else
                                   "ccf_tc_kernel (tcgen05 kind::i8 over the 3D im2col)") if tc3 else "screen3d_kernel (%s)" % ("dp4a" if kind == 1 else "IMAD"),
                        "achieved": achieved, "peak": peak, "unit": "TOPS",
                        "frac": achieved / peak if achieved and peak else None,
                        "peak_source": "measured in this run: tcgen05 kind::i8 MMA probe (ccw_measure_i8_peak)"
                                       if tc3 else
                                       "measured in this run: %s probe, 8 chains per thread (ccw_measure_int_peak)"
                                       % ("dp4a" if kind == 1 else "IMAD"),
                        "algorithmic_ops_per_step": prof["ccf_flop"],
                        "algorithmic_ops_note": "SURVEY 8(d): 2 x F channels x window positions x mask cells "
                                                "per placement",
                        "screen_ms_per_step": prof["ccf_ms"], "step_ms_profiled": prof["total_ms"]},
           "e2e": {"value": n_real * sgv * steps / e2e_s, "unit": UNIT,
                   "h2d_bytes_per_step": int(ti_a.nbytes + seeds.nbytes + (hd_a.nbytes if hd_a is not None else 0)),
                   "d2h_bytes_per_step": int(dev.last_timing()["d2h_bytes"]),
                   "equals_device_result": e2e_equal}}
    if not skip_cpu:
        o3 = P3.oracle3()
        cores = os.cpu_count() or 1
        oc = P3.Cfg3(sg=tuple(cfg.sg), template_size=cfg.template_size, overlap=cfg.overlap,
                     dwt_level=cfg.dwt_level, candidates=cfg.candidates)
        t0 = time.perf_counter()
        o = o3.simulate_one(ti_a, nf, oc, wells, seed=int(seeds[0]), threads=cores)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": sgv / dt, "unit": UNIT, "cores": cores, "kind": "port",
                               "cpu_model": cpu_model(),
                               "sample": f"realization 0 of the workload, every score map split over {cores} "
                                         f"threads, {dt:.1f} s wall (the reference has no 3D: builder's "
                                         f"exact-integer 3D restatement, oracle/ccw3d_oracle.c)"}
        out["parity"] = {"checked": 1, "equal": bool(np.array_equal(got[0], o["realization"])),
                         "against": "oracle/ccw3d_oracle.c (the cpu_baseline run's output), same seed"}
    return out


def measure_shim(ti_a, steps):
    """config 1 end to end through the C++ drop-in shim (include/ccwsim_gpu.hpp,
    tests/cpp/bench_shim.cpp): the reference's own CategoricalGrid /
    std::vector<SimResult> types in and out, as a reference user calls it."""
    import tempfile
    d = tempfile.mkdtemp(prefix="ccw_shim_")
    exe, tib = os.path.join(d, "bench_shim"), os.path.join(d, "ti.bin")
    np.ascontiguousarray(ti_a, np.uint8).tofile(tib)
    lib_dir = os.path.join(ROOT, "paper_2404_00441_b200")
    try:
        subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "bench_shim.cpp"), "-o", exe, "-L", lib_dir,
                        "-lccwgpu", "-Wl,-rpath," + lib_dir, "-pthread"], check=True, capture_output=True,
                       timeout=300)
        r = subprocess.run([exe, tib, str(steps), "2"], capture_output=True, text=True, timeout=600)
        out = json.loads(r.stdout.strip().splitlines()[-1])
        return {"value": out["cells_per_s"], "unit": UNIT, "ms_per_step": out["ms_per_step"],
                "steps": out["steps"], "path": "ccwsim::simulate_ensemble through include/ccwsim_gpu.hpp "
                "(std::vector<int> grids in and out, pageable host memory; tests/cpp/bench_shim.cpp)"}
    except Exception as e:  # (the measurement is informative; the line stands without it)
        return {"error": str(e)[:200]}


CONFIG2 = ("config2: TI 2000x2000 binary channels, SG 4000x4000, T96 OV24 J3 K1, 1% hard data "
           "(160,000 cells from a seeded realization), 8 realizations")


def measure_config2(dev, lib, local, args, skip_cpu=False):
    """BASELINE config 2, the largest single-GPU configuration: device-resident
    cells/s, e2e through the C-ABI with host buffers, the compiled reference on
    the host cores on the same 8 seeds (its outputs double as the parity check)."""
    import torch
    from paper_2404_00441_b200 import _abi, ccwsim as cs, synth
    n_real = 8
    ti_a = synth.config2_ti()
    hd = synth.config2_hard_data(ti_a)
    hd_a = np.ascontiguousarray(hd, np.int32)
    grid = cs.CategoricalGrid(2000, 2000, 2, ti_a)
    cfg = cs.SimConfig(4000, 4000, 96, 24, 3, 1, n_realizations=n_real, master_seed=MASTER)
    tih = cs.TrainingImage(grid, cfg.dwt_level, "indicator", dev)
    c = cfg.to_c()
    seeds = np.array([cs.mix64(MASTER, r + 1) for r in range(n_real)], np.uint64)
    sg = cfg.sg_height * cfg.sg_width
    d_out = torch.empty(n_real * sg, dtype=torch.uint8, device=f"cuda:{local}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    diags = (_abi.DiagC * n_real)()
    stream = torch.cuda.ExternalStream(dev.stream_ptr, device=torch.device("cuda", local))

    def step_device():
        dev.check(lib.ccw_simulate_device(dev.handle, tih.handle, C.byref(c),
                                          seeds.ctypes.data_as(_abi.U64P), n_real,
                                          hd_a.ctypes.data_as(_abi.I32P), hd_a.shape[0],
                                          C.c_void_p(d_out.data_ptr()), diags))

    def step_device_async():
        dev.check(lib.ccw_simulate_device_async(dev.handle, tih.handle, C.byref(c),
                                                seeds.ctypes.data_as(_abi.U64P), n_real,
                                                hd_a.ctypes.data_as(_abi.I32P), hd_a.shape[0],
                                                C.c_void_p(d_out.data_ptr())))

    for _ in range(max(args.warmup, 3)):
        with torch.cuda.stream(stream):
            flush.zero_()
        step_device()
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 10))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            evs[k][0].record(stream)
        step_device_async()
        with torch.cuda.stream(stream):
            evs[k][1].record(stream)
    dev.synchronize()
    torch.cuda.synchronize()
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    timing = dev.last_timing()
    got = d_out.view(n_real, cfg.sg_height, cfg.sg_width).cpu().numpy()
    mism = [d.pre_overwrite_mismatches for d in diags]
    h_out = torch.empty(n_real * sg, dtype=torch.uint8).pin_memory()
    ti_host = np.ascontiguousarray(ti_a)

    def step_e2e():
        h = C.c_void_p()
        dev.check(lib.ccw_ti_create(dev.handle, ti_host.ctypes.data_as(_abi.U8P), 2000, 2000, 2,
                                    cfg.dwt_level, 0, C.byref(h)))
        dev.check(lib.ccw_simulate(dev.handle, h, C.byref(c), seeds.ctypes.data_as(_abi.U64P), n_real,
                                   hd_a.ctypes.data_as(_abi.I32P), hd_a.shape[0],
                                   C.cast(C.c_void_p(h_out.data_ptr()), _abi.U8P), diags, None))
        lib.ccw_ti_destroy(h)

    step_e2e()
    e2e_s = 0.0
    for _ in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step_e2e()
        torch.cuda.synchronize()
        e2e_s += time.perf_counter() - t0
    d2h = int(dev.last_timing()["d2h_bytes"])
    e2e_equal = bool(np.array_equal(h_out.numpy().reshape(n_real, 4000, 4000), got))
    out = {"workload": CONFIG2, "value": n_real * sg * steps / (total_ms * 1e-3), "unit": UNIT,
           "ms_per_step": total_ms / steps, "steps": steps,
           "fp64_windows_rescored": int(timing["rescored"]), "bulk_jobs": int(timing["bulk_jobs"]),
           "gpu_launches": int(timing["launches"]) * steps,
           "e2e": {"value": n_real * sg * steps / e2e_s, "unit": UNIT,
                   "h2d_bytes_per_step": int(ti_host.nbytes + hd_a.nbytes + seeds.nbytes),
                   "d2h_bytes_per_step": d2h, "equals_device_result": e2e_equal}}
    if not skip_cpu:
        cores = os.cpu_count() or 1
        rate, dt, kind, ref = cpu_reference_rate(ti_a, 2, cfg, n_real, min(cores, n_real), hd, MASTER)
        ok = [bool(np.array_equal(got[r], ref[r])) for r in range(n_real)]
        out["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": min(cores, n_real), "kind": kind,
                               "cpu_model": cpu_model(),
                               "sample": f"the whole config-2 workload ({n_real} realizations), "
                                         f"simulate_ensemble(workers={min(cores, n_real)}), {dt:.1f} s wall"}
        out["parity"] = {"checked": n_real, "equal": all(ok),
                         "mismatched": [r for r, v in enumerate(ok) if not v],
                         "against": f"oracle/_ref ({kind}), the cpu_baseline run's own outputs, same seeds"}
    out["pre_overwrite_mismatches"] = mism
    return out


SINGLE_WORKLOAD = ("config2-single: TI 2000x2000 binary channels, SG 4000x4000, T96 OV24 J3 K1, "
                   "1% hard data, ONE realization, TI window positions sharded over the ranks "
                   "(per-wave ncclAllGather of the shards' top-K lists)")


def run_single(args):
    """--workload single: one config-2 realization whose every placement's
    TI window positions are split across the N ranks; strong
    scaling.  --virtual-shards V splits each rank's range V ways more."""
    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    from paper_2404_00441_b200 import _abi, ccwsim as cs, synth
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _abi.lib()
    dev = cs.Device(local)
    uid = None
    if world > 1 or args.nccl:
        box = [cs.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            torch.distributed.broadcast_object_list(box, src=0)
        uid = box[0]
    dev.set_position_shards(world, rank, uid, args.virtual_shards)
    stream = torch.cuda.ExternalStream(dev.stream_ptr, device=torch.device("cuda", local))
    ti_a = synth.config2_ti()
    hd = synth.config2_hard_data(ti_a)
    grid = cs.CategoricalGrid(2000, 2000, 2, ti_a)
    cfg = cs.SimConfig(4000, 4000, 96, 24, 3, 1, master_seed=MASTER)
    tih = cs.TrainingImage(grid, cfg.dwt_level, "indicator", dev)
    c = cfg.to_c()
    hd_a = np.ascontiguousarray(hd, np.int32)
    seeds = np.array([cs.mix64(MASTER, 1)], np.uint64)
    sg = cfg.sg_height * cfg.sg_width
    d_out = torch.empty(sg, dtype=torch.uint8, device=f"cuda:{local}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    diags = (_abi.DiagC * 1)()

    def step_device():
        dev.check(lib.ccw_simulate_device(dev.handle, tih.handle, C.byref(c),
                                          seeds.ctypes.data_as(_abi.U64P), 1,
                                          hd_a.ctypes.data_as(_abi.I32P), hd_a.shape[0],
                                          C.c_void_p(d_out.data_ptr()), diags))

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            evs[k][0].record(stream)
        step_device()
        with torch.cuda.stream(stream):
            evs[k][1].record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    if world > 1:
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    timing = dev.last_timing()
    value = sg * args.steps / (total_ms * 1e-3)
    # end to end: TI from host bytes, hard data and result through host memory
    h_out = torch.empty(sg, dtype=torch.uint8).pin_memory()
    ti_host = np.ascontiguousarray(ti_a)

    def step_e2e():
        h = C.c_void_p()
        dev.check(lib.ccw_ti_create(dev.handle, ti_host.ctypes.data_as(_abi.U8P), 2000, 2000, 2,
                                    cfg.dwt_level, 0, C.byref(h)))
        dev.check(lib.ccw_simulate(dev.handle, h, C.byref(c), seeds.ctypes.data_as(_abi.U64P), 1,
                                   hd_a.ctypes.data_as(_abi.I32P), hd_a.shape[0],
                                   C.cast(C.c_void_p(h_out.data_ptr()), _abi.U8P), diags, None))
        lib.ccw_ti_destroy(h)

    step_e2e()
    e2e_s = 0.0
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step_e2e()
        torch.cuda.synchronize()
        e2e_s += time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    d2h = int(dev.last_timing()["d2h_bytes"])
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "i8xi8->i32 screen + f64 rescoring",
                "data": "synthetic",
                "config": {"workload": SINGLE_WORKLOAD, "position_shards": world * args.virtual_shards,
                           "exchange": "ncclAllGather" if uid is not None else
                                       ("device memory (virtual shards)" if args.virtual_shards > 1 else "none"),
                           "virtual_shards_per_rank": args.virtual_shards,
                           "l2": "flushed before each timed step (256 MiB write, outside events)",
                           "timing": "per-step CUDA events on the library stream, max over ranks"},
                "e2e": {"value": sg * args.steps / e2e_s, "unit": UNIT,
                        "h2d_bytes_per_step": int(ti_host.nbytes + hd_a.nbytes + seeds.nbytes),
                        "d2h_bytes_per_step": d2h},
                "gpu_launches": int(timing["launches"]) * args.steps, "clocks": clocks}
        print(json.dumps(line))
    dev.set_position_shards(1, 0, None, 1)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def _rank_main(rank, argv, world, port):
    """One spawned rank of `bench.py --gpus N` (torchrun's environment)."""
    os.environ.update({"RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(world),
                       "LOCAL_WORLD_SIZE": str(world), "MASTER_ADDR": "127.0.0.1",
                       "MASTER_PORT": str(port)})
    sys.argv = [sys.argv[0]] + list(argv)
    rc = main()
    if rc:
        raise SystemExit(rc)


def spawn_ranks(n: int) -> int:
    """`--gpus N` outside torchrun: one process per GPU, as torchrun would."""
    import socket
    import torch
    import torch.multiprocessing as mp
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {n} but {have} GPUs visible"}))
        return 1
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.start_processes(_rank_main, args=(sys.argv[1:], n, port), nprocs=n, join=True,
                       start_method="spawn")
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-config2", action="store_true",
                    help="omit the nested config-2 measurement (N=1 only)")
    ap.add_argument("--skip-3d", action="store_true",
                    help="omit the nested config-3 / config-4 (3D) measurements (N=1 only)")
    ap.add_argument("--workload", default="config1", choices=["config1", "single"],
                    help="config1 (headline) or single: one config-2 realization, positions sharded")
    ap.add_argument("--virtual-shards", type=int, default=1)
    ap.add_argument("--nccl", action="store_true",
                    help="single: exchange through an NCCL communicator even on one rank")
    args = ap.parse_args()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "ours" and args.workload == "single":
        return run_single(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
