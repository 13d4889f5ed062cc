#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) on a reduced -m gpu subset:
# TMEM alloc/dealloc + cp.async rings (fb_chunk), last-block counters (reduce_mstep,
# variance pass), chain-warp and K-lane Viterbi, large-K split kernels.
mkdir -p gpurun_out
SUB='tests/test_gpu_parity.py::test_small_model_fixtures tests/test_gpu_parity.py::test_earthquake_fixture tests/test_gpu_parity.py::test_error_semantics tests/test_gpu_parity.py::test_single_state_and_single_step tests/test_gpu_training.py::test_variance_second_pass_forced tests/test_gpu_training.py::test_student_t_guard_many_candidates tests/test_gpu_training.py::test_collapse_guard_unreachable_state_frozen'
KSUB='test_posteriors_batch_ragged and (4 or 8) or test_fp32_viterbi_bitexact_ragged and (4 or 8) or test_large_k_short_sequences_split_pass or test_viterbi_equal_length_bitexact and 36'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 python -m pytest $SUB -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/sanitizer_${tool}.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_${tool}.log
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -k "$KSUB" -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/sanitizer_${tool}_k.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_${tool}_k.log
  tail -4 gpurun_out/sanitizer_${tool}.log gpurun_out/sanitizer_${tool}_k.log
done
