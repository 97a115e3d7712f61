#!/bin/bash
# Runs on the GPU box: full ncu capture of the selection kernels of one hisa_select call (top-m blocks, top-k tokens).
mkdir -p gpurun_out
BENCH="python bench.py --e2e-steps 0 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:select_ -s 2 -c 2 -f -o gpurun_out/prof_select \
    $BENCH --steps 1 --warmup 1 --flat-steps 0 > gpurun_out/prof_select.log 2>&1
ls -la gpurun_out/*.ncu-rep
