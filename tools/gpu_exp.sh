#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "equal_length and float32" > gpurun_out/pytest_sub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sub.log; tail -2 gpurun_out/pytest_sub.log
LOGHMM_FBC_WPB=3 timeout 600 python -m pytest tests -x -q -m gpu -k "equal_length and float32" > gpurun_out/pytest_sub3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sub3.log; tail -2 gpurun_out/pytest_sub3.log
for rep in 1 2; do for w in 4 3; do
  LOGHMM_FBC_WPB=$w timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_w$w.json 2>&1
  python3 -c "import json; d=json.loads(open('gpurun_out/bench_w$w.json').read().strip().splitlines()[-1]); print('fbc_wpb=$w', round(d['ms_per_step']*1000,1), round(d['roofline']['kernel_ms']*1000,1), round(d['pipeline_roofline']['viterbi_kernel_ms']*1000,1), round(d['e2e']['ms_per_step']*1000,1))"
done; done
for w in 4 3; do LOGHMM_FBC_WPB=$w timeout 300 python tools/prof_kernels.py --dtype float32 --only fb; done
