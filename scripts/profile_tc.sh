#!/bin/bash
# Runs on the GPU box: full ncu capture of the scorer launches of one hisa_select call (stage 1 + stage 2).
# PROF_TAG names the output; environment knobs (HISA_TC_ATMEM, HISA_TC_PRODUCERS ...) pass through to the library.
mkdir -p gpurun_out
TAG=${PROF_TAG:-score_tc}
BENCH="python bench.py --e2e-steps 0 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 2 -c 2 -f -o gpurun_out/prof_$TAG \
    $BENCH --steps 1 --warmup 1 --flat-steps 0 > gpurun_out/prof_$TAG.log 2>&1
ls -la gpurun_out/*.ncu-rep
