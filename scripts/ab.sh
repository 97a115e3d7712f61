#!/bin/bash
# Runs on the GPU box: A/B of an environment knob inside ONE call (boxes differ by several percent in sustained clocks).
# AB_VAR names the variable, AB_VALUES its values; AB_REPS repetitions (default 2).
mkdir -p gpurun_out
for i in $(seq 1 ${AB_REPS:-2}); do
  for v in ${AB_VALUES:-default}; do
    for dt in ${AB_DTYPES:-bf16 fp8}; do
      env ${AB_VAR:-HISA_AB_UNUSED}=$v python bench.py --dtype $dt --steps 5 --flat-steps ${AB_FLAT:-0} --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.log 2>&1
      python - <<PY
import json
j=json.loads([x for x in open("gpurun_out/ab.log") if x.startswith("{")][-1])
s=j["stages_ms_per_step"]; st=j["scorer_stall_fraction_of_cta_time"]["stage2"]
fl=j["flat_dsa"]["ms_per_step"] if j.get("flat_dsa") else 0
print("${AB_VAR}=$v $dt rep $i: step %.3f s1 %.3f s2 %.3f topk %.3f prep %.3f flat %.2f | qdata %.3f epi %.3f prodidle %.3f mhz %.0f" % (j["ms_per_step"], s["score_blocks_ms"], s["score_tokens_ms"], s["top_k_ms"], s["prepare_ms"], fl, st["mma_wait_qdata"], st["mma_wait_epilogue"], st["prod_wait_qstage"], st["sm_mhz_in_kernel"]), "balance", st.get("cta_balance"))
PY
    done
  done
done
