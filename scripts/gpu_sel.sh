#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --flat-steps 1 --steps 5 --warmup 2 --e2e-steps 3 > gpurun_out/bench_sel.log 2>&1
python - <<PY
import json
l=[x for x in open("gpurun_out/bench_sel.log") if x.startswith("{")]
j=json.loads(l[-1]); print("ms/step", j["ms_per_step"], j["stages_ms_per_step"], "e2e", j["e2e"], "flat", j["flat_dsa"])
PY
