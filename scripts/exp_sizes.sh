#!/bin/bash
mkdir -p gpurun_out
for L in ${SIZES:-4096 8192 16384 32768 65536}; do
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --flat-steps ${FLAT:-0} --steps 3 --warmup 1 --seq-len $L > gpurun_out/size_$L.log 2>&1
  echo "L=$L rc=$? $(grep -v 'timed out' gpurun_out/size_$L.log | grep -o 'HisaError.*' | tail -1 | cut -c1-160) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/size_$L.log | head -1) $(grep -c 'timed out' gpurun_out/size_$L.log)"
done
