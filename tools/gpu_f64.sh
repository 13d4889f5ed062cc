#!/bin/bash
# fp64 config 2 through the chunk-operator kernel (tensor-memory park): parity, then timings A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_training.py -q -m gpu --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_f64.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f64.log
tail -8 gpurun_out/pytest_f64.log
timeout 300 python tools/prof_kernels.py --dtype float64 --only fb 2>&1 | tail -2
LOGHMM_FBC_F64=0 timeout 300 python tools/prof_kernels.py --dtype float64 --only fb 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python3 -c "import json; d=json.loads(open('gpurun_out/bench_quick.json').read().strip().splitlines()[-1]); print('bench', round(d['ms_per_step']*1e3,1), round(d['roofline']['kernel_ms']*1e3,1), round(d['pipeline_roofline']['viterbi_kernel_ms']*1e3,1), 'f64', round(d['per_dtype']['f64']['ms_per_step']*1e3,1), 'e2e', round(d['e2e']['ms_per_step']*1e3,1))"
