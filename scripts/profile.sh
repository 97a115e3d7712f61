#!/bin/bash
# Runs on the GPU box: ncu launch list + full captures of the dominant kernels. Outputs under gpurun_out/.
mkdir -p gpurun_out
BENCH="python bench.py --e2e-steps 0 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    $BENCH --steps 2 --warmup 1 --flat-steps 1 > gpurun_out/launches_bench.log 2>&1
# -s 2: skip the warm-up call's two scorer launches; -c 2: stage 1 + stage 2 of the timed call
ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 2 -c 2 -f -o gpurun_out/prof_score_tc \
    $BENCH --steps 1 --warmup 1 --flat-steps 0 > gpurun_out/prof_score_tc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 2 -c 2 -f -o gpurun_out/prof_score_tc_fp8 \
    $BENCH --dtype fp8 --steps 1 --warmup 1 --flat-steps 0 > gpurun_out/prof_score_tc_fp8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:select_ -s 2 -c 2 -f -o gpurun_out/prof_select \
    $BENCH --steps 1 --warmup 1 --flat-steps 0 > gpurun_out/prof_select.log 2>&1
ls -la gpurun_out/
