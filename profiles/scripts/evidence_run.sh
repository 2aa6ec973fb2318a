#!/bin/bash
# usage (on the GPU box): bash profiles/scripts/evidence_run.sh  -- writes gpurun_out/{t,smoke,b,bref,plain,ncu_*}.log, launches.csv, ccf/sel.ncu-rep
# round-1h evidence run: tests, bench lines, ncu launch list and kernel captures
cd "$GRAFT_REPO_ROOT"
python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; echo "rc=$?" >> gpurun_out/t.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/b.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bref.log 2>&1
python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ccf_tc_kernel -s 200 -c 1 \
    -o gpurun_out/ccf python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/ncu_ccf.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:select_fast_kernel -s 200 -c 1 \
    -o gpurun_out/sel python bench.py --steps 1 --warmup 1 --skip-cpu > gpurun_out/ncu_sel.log 2>&1
tail -2 gpurun_out/t.log; tail -1 gpurun_out/b.log
