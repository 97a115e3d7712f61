#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "pipeline or random_inputs or decode" > gpurun_out/pytest_pipe.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pipe.log
for P in 2048 4096 8192 16384; do
  HISA_PIPE_ROWS=$P timeout 300 python bench.py --no-cpu-baseline --flat-steps 0 --steps 3 --warmup 1 --e2e-steps 5 > gpurun_out/e2e_$P.log 2>&1
  python - <<PY
import json
l=[x for x in open("gpurun_out/e2e_$P.log") if x.startswith("{")]
j=json.loads(l[-1]); print("pipe=$P", j["e2e"], "ms/step", j["ms_per_step"])
PY
done
