#!/bin/bash
# Runs on the GPU box: smoke, GPU tests, default bench (both arms), fp8 bench, the other configurations. Logs under gpurun_out/.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
timeout 600 python bench.py --dtype fp8 > gpurun_out/bench_fp8.log 2> gpurun_out/bench_fp8.err; echo "fp8 rc=$?"

tail -c 3000 gpurun_out/bench_default.log; tail -c 1500 gpurun_out/bench_reference.log
