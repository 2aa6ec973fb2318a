"""Summaries for profiles/ from an evidence run's gpurun_out/ (see evidence_run.sh).

    python profiles/scripts/summarize.py <tag>     # e.g. r1h

writes profiles/<tag>_launch_shares.txt (per-kernel totals of the ncu launch
list) and profiles/<tag>_{ccf,sel}_ncu.txt (ncu --set full sections and raw
counters of one captured launch), read with `ncu -i` on this machine."""
import collections
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "gpurun_out")
SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
SECTIONS = ("Speed Of Light", "Compute Workload", "Memory Workload", "Scheduler", "Occupancy",
            "Launch Statistics", "Warp State")
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
       "launch__shared_mem_per_block_static", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
       "smsp__pcsamp_warps_issue_stalled_no_instructions", "smsp__pcsamp_warps_issue_stalled_wait",
       "smsp__pcsamp_sample_count"]


def launch_shares(tag):
    rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        us = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        name = r[ki].split("(")[0][:58]
        tot[name] += us
        cnt[name] += 1
    T = sum(tot.values())
    out = io.StringIO()
    out.write(f"# {tag}: ncu --metrics gpu__time_duration.sum --clock-control none launch list of "
              "`python bench.py --steps 1 --warmup 1 --skip-cpu` (cold caches, serialised -- compare shares)\n")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.write(f"{k:58s} n={cnt[k]:5d} total={v / 1000:8.3f} ms avg={v / cnt[k]:9.2f} us share={v / T:.3f}\n")
    open(os.path.join(ROOT, "profiles", f"{tag}_launch_shares.txt"), "w").write(out.getvalue())
    print(out.getvalue())


def ncu_summary(tag, rep, kernel):
    path = os.path.join(OUT, f"{rep}.ncu-rep")
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    out = io.StringIO()
    src = {"s3d": "profiles/scripts/config3_run.py (WHICH=3)", "s4d": "profiles/scripts/config3_run.py (WHICH=4)",
           "bulk": "profiles/scripts/config2_run.py",
           "wave": "WAVE=1 WAVE_CS=16 profiles/scripts/timeline_run.py (the experimental fused wave kernel, config 1)"}.get(rep, "python bench.py --steps 1 --warmup 1 --skip-cpu, config 1")
    out.write(f"# {tag} {kernel}: one launch, ncu --set full --clock-control none --import-source on ({src}); "
              "see profiles/scripts/evidence_run.sh\n")
    r = list(csv.reader(io.StringIO(det)))
    h = r[0]
    si, mi, ui, vi = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    for x in r[1:]:
        if any(x[si].startswith(k) for k in SECTIONS):
            out.write(f"{x[si][:40]:40s} | {x[mi][:40]:40s} | {x[vi]:>14s} {x[ui]}\n")
    out.write("# raw counters\n")
    r = list(csv.reader(io.StringIO(raw)))
    for w in RAW:
        if w in r[0]:
            i = r[0].index(w)
            out.write(f"{w:70s} {r[2][i]:>14s} {r[1][i]}\n")
    open(os.path.join(ROOT, "profiles", f"{tag}_{rep}_ncu.txt"), "w").write(out.getvalue())


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1h"
    launch_shares(tag)
    ncu_summary(tag, "ccf", "ccf_tc_kernel")
    ncu_summary(tag, "sel", "select_fast_kernel")
    for rep, kern in (("s3d", "ccf_tc_kernel over the 3D im2col (config 3, option tc3d)"), ("s4d", "ccf_tc_kernel over the two-digit 3D im2col (config 4, option tc3d)"),
                      ("bulk", "select_bulk_kernel (config 2)"), ("wave", "wave_kernel<16> (experimental)")):
        if os.path.exists(os.path.join(OUT, rep + ".ncu-rep")):
            ncu_summary(tag, rep, kern)
