#!/bin/bash
# Runs on the GPU box: ncu launch list + full captures of the dominant kernels + a racecheck pass over the selection kernels
# alone. Outputs under gpurun_out/ (scripts/make_profiles.py <tag> turns them into the committed summaries under profiles/).
mkdir -p gpurun_out
BENCH="python bench.py --e2e-steps 0 --no-cpu-baseline --no-configs"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    $BENCH --steps 2 --warmup 1 --flat-steps 1 > gpurun_out/launches_bench.log 2>&1
# -s 2: skip the warm-up call's two scorer launches; -c 2: stage 1 + stage 2 of the timed call
ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 2 -c 2 -f -o gpurun_out/prof_score_tc \
    $BENCH --steps 1 --warmup 1 --flat-steps 0 --attend-steps 0 > gpurun_out/prof_score_tc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_tc_kernel -s 2 -c 2 -f -o gpurun_out/prof_score_tc_fp8 \
    $BENCH --dtype fp8 --steps 1 --warmup 1 --flat-steps 0 --attend-steps 0 > gpurun_out/prof_score_tc_fp8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:select_ -s 2 -c 2 -f -o gpurun_out/prof_select \
    $BENCH --steps 1 --warmup 1 --flat-steps 0 --attend-steps 0 > gpurun_out/prof_select.log 2>&1
# the batch pooling kernel of the committed build (bench.py's pool_build leg launches it back to back)
ncu --set full --clock-control none --import-source on -k regex:pool_update -s 1 -c 1 -f -o gpurun_out/prof_pool \
    $BENCH --steps 1 --warmup 1 --flat-steps 0 --attend-steps 0 > gpurun_out/prof_pool.log 2>&1
# racecheck over tests that launch ONLY the selection kernels (top_k_tokens / select_blocks on given scores): no TMA /
# tcgen05 scorer in the process, so every reported hazard would be a real one
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report analysis python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
  -p no:cacheprovider -k "top_k_on_given_scores or select_blocks_on_given" > gpurun_out/racecheck_select_only.log 2>&1
echo "racecheck (selection kernels only) rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/racecheck_select_only.log
ls -la gpurun_out/
