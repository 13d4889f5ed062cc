#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "equal_length or estep or config2 or baum_welch" > gpurun_out/pytest_sub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sub.log; tail -2 gpurun_out/pytest_sub.log
timeout 300 python tools/prof_kernels.py --dtype float32 --only fb > gpurun_out/prof_f32.json 2>&1; cat gpurun_out/prof_f32.json
for i in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$i.json 2>&1
  python3 -c "import json; d=json.loads(open('gpurun_out/bench_$i.json').read().strip().splitlines()[-1]); print('run$i', d['ms_per_step'], d['roofline']['kernel_ms'], d['pipeline_roofline']['viterbi_kernel_ms'], d['e2e']['ms_per_step'])"
done
