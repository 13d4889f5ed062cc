#!/bin/bash
# Round-2 call B: tests that need the reference install, compute-sanitizer on a reduced
# subset, Viterbi layout A/B inside the step, FB traffic capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shim.py tests/test_gpu_cli.py tests/test_gpu_init.py -q -m gpu --timeout 600 -p no:cacheprovider -rs > gpurun_out/pytest_ref.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ref.log
SUB='tests/test_gpu_parity.py::test_small_model_fixtures tests/test_gpu_parity.py::test_earthquake_fixture tests/test_gpu_parity.py::test_error_semantics tests/test_gpu_parity.py::test_single_state_and_single_step tests/test_gpu_training.py::test_variance_second_pass_forced tests/test_gpu_training.py::test_student_t_guard_many_candidates tests/test_gpu_training.py::test_collapse_guard_unreachable_state_frozen'
KSUB='test_posteriors_batch_ragged and (4 or 8) or test_fp32_viterbi_bitexact_ragged and (4 or 8) or test_large_k_short_sequences_split_pass'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 python -m pytest $SUB -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/sanitizer_${tool}.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_${tool}.log
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -k "$KSUB" -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/sanitizer_${tool}_k.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_${tool}_k.log
done
bash tools/gpu_ab_env.sh - LOGHMM_VIT_ALGO=pair
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,l1tex__m_l1tex2xbar_write_bytes.sum,gpu__time_duration.sum -k regex:"fb_chunk|fb_small" --csv --print-units base --log-file gpurun_out/traffic.csv python tools/fb_traffic.py > gpurun_out/traffic.log 2>&1
ls -la gpurun_out
