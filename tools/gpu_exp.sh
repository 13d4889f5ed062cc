#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "baum_welch or config or golden or large_k or host_slices or mstep" > gpurun_out/pytest_sub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sub.log; tail -3 gpurun_out/pytest_sub.log
timeout 300 python tools/prof_kernels.py --dtype float32 --only small
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_$i.json 2>&1
python3 -c "import json; d=json.loads(open('gpurun_out/bench_$i.json').read().strip().splitlines()[-1]); print('bench', round(d['ms_per_step']*1000,1), round(d['roofline']['kernel_ms']*1000,1), round(d['pipeline_roofline']['viterbi_kernel_ms']*1000,1), round(d['e2e']['ms_per_step']*1000,1))"; done
