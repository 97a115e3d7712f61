#!/bin/bash
mkdir -p gpurun_out
for d in ${DEBUG_SET:-0 1 2 3}; do
  HISA_TC_DEBUG=$d timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --flat-steps 1 --steps 5 > gpurun_out/dbg_$d.log 2>&1
  python - <<PY
import json
l=[x for x in open("gpurun_out/dbg_$d.log") if x.startswith("{")]
j=json.loads(l[-1])
print("debug=$d", "ms/step", round(j["ms_per_step"],3), "s2_ms", round(j["stages_ms_per_step"]["score_tokens_ms"],3), "s1_ms", round(j["stages_ms_per_step"]["score_blocks_ms"],3), "flat_scorer_ms", round(j["flat_dsa"]["scorer_ms"],3), j["scorer_stall_fraction_of_cta_time"]["stage2"], j["clocks"])
PY
done
