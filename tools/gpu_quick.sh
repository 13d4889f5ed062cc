#!/bin/bash
# Quick GPU check: new-kernel parity tests, kernel timings, bench line, one ncu capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 300 python tools/prof_kernels.py --dtype float32 > gpurun_out/prof_f32.json 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_f32.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fb_chunk" -c 1 -o gpurun_out/fbc_float32 python tools/prof_kernels.py --dtype float32 --reps 1 --only fb > gpurun_out/ncu_fbc_float32.log 2>&1
tail -3 gpurun_out/pytest_all.log; cat gpurun_out/prof_f32.json
python3 -c "import json; d=json.loads(open('gpurun_out/bench_f32.json').read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d['value'], d['roofline']['kernel_ms'], d['pipeline_roofline']['viterbi_kernel_ms'], d['e2e']['ms_per_step'])"
