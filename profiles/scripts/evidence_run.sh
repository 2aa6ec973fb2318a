#!/bin/bash
# usage (on the GPU box): bash profiles/scripts/evidence_run.sh -- round-2 evidence: bench lines,
# ncu launch list of the config-1 bench, ncu --set full captures of the hot kernels
cd "$GRAFT_REPO_ROOT"
python bench.py > gpurun_out/b.log 2> gpurun_out/b.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bref.log 2>&1
B1="bench.py --steps 1 --warmup 1 --skip-cpu --skip-config2 --skip-3d"
python $B1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python $B1 > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ccf_tc_kernel -s 200 -c 1 \
    -o gpurun_out/ccf python $B1 > gpurun_out/ncu_ccf.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:select_fast_kernel -s 200 -c 1 \
    -o gpurun_out/sel python $B1 > gpurun_out/ncu_sel.log 2>&1
# config 3 screens on the tensor cores (option tc3d, default on): the 2D ccf_tc_kernel over the 3D im2col
WHICH=3 REPS=1 ncu --set full --clock-control none --import-source on -k regex:ccf_tc -s 20 -c 1 \
    -o gpurun_out/s3d python profiles/scripts/config3_run.py > gpurun_out/ncu_s3d.log 2>&1
WHICH=3 REPS=1 PROF=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3d.csv \
    python profiles/scripts/config3_run.py > gpurun_out/ncu_list3d.log 2>&1
WHICH=4 REPS=1 ncu --set full --clock-control none --import-source on -k regex:ccf_tc -s 20 -c 1 \
    -o gpurun_out/s4d python profiles/scripts/config3_run.py > gpurun_out/ncu_s4d.log 2>&1
WHICH=4 REPS=1 PROF=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4d.csv \
    python profiles/scripts/config3_run.py > gpurun_out/ncu_list4d.log 2>&1
REPS=1 ncu --set full --clock-control none --import-source on -k regex:select_bulk -s 120 -c 1 \
    -o gpurun_out/bulk python profiles/scripts/config2_run.py > gpurun_out/ncu_bulk.log 2>&1
tail -c 400 gpurun_out/b.log; tail -c 300 gpurun_out/bref.log
# the experimental fused wave kernel (option wave=1, off by default): one launch, config 1
WAVE=1 WAVE_CS=16 REPS=1 ncu --set full --clock-control none --import-source on -k regex:wave_kernel -s 20 -c 1 \
    -o gpurun_out/wave python profiles/scripts/timeline_run.py > gpurun_out/ncu_wave.log 2>&1
CS=4,8,16 python profiles/scripts/wave_ab.py > gpurun_out/wave_ab.log 2>&1
