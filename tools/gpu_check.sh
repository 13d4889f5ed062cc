#!/bin/bash
# full GPU parity suite + standalone kernel timings + headline bench (no CPU baseline)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -6 gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_kernels.py --dtype float32 > gpurun_out/prof_f32.json 2>&1; cat gpurun_out/prof_f32.json
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python3 -c "import json; d=json.loads(open('gpurun_out/bench_quick.json').read().strip().splitlines()[-1]); print('bench', round(d['ms_per_step']*1e3,1), round(d['roofline']['kernel_ms']*1e3,1), round(d['pipeline_roofline']['viterbi_kernel_ms']*1e3,1), 'f64', round(d['per_dtype']['f64']['ms_per_step']*1e3,1), 'e2e', round(d['e2e']['ms_per_step']*1e3,1))"
