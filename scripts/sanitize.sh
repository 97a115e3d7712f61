#!/bin/bash
# Runs on the GPU box: compute-sanitizer passes over small-shape GPU tests (race detection / sanitizers).
#   memcheck  - every kernel, a cross-section of the tests
#   racecheck - the selection kernels (block barriers + shared memory). The tensor-core scorer synchronises through
#               mbarriers / the async proxy (TMA complete_tx, tcgen05.commit), which racecheck does not model: its
#               hazards on the scorer's meta slots are expected and not a finding.
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests -m gpu -q -x -p no:cacheprovider \
  -k "lattice_inputs_bit_exact and 1-shape1 or fp8_lattice or top_k_on_given_scores and 9000 or pool_append or decode_placement or tmem_tile_variant or decode_config_c5_128k or survives_a_larger_call or forced_in_budget_tiny or random_api_sessions" \
  > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/memcheck.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_attention.py -m gpu -q -x \
  -p no:cacheprovider -k "not full_size" > gpurun_out/memcheck_attend.log 2>&1; echo "memcheck (consumer) rc=$?"; tail -3 gpurun_out/memcheck_attend.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis python -m pytest tests -m gpu -q -x -p no:cacheprovider \
  -k "top_k_on_given_scores or select_blocks_on_given or eligible or spec_examples" > gpurun_out/racecheck.log 2>&1
echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/racecheck.log
