#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 300 python tools/prof_kernels.py --dtype float32 > gpurun_out/prof_f32.json 2>&1
timeout 300 python tools/prof_kernels.py --dtype float64 --only vit > gpurun_out/prof_f64v.json 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_f32.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --dtype float64 > gpurun_out/bench_f64.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"viterbi_seq" -c 1 -o gpurun_out/vseq python tools/prof_kernels.py --dtype float32 --reps 1 --only vit > gpurun_out/ncu_vseq.log 2>&1
tail -15 gpurun_out/pytest_all.log; cat gpurun_out/prof_f32.json gpurun_out/prof_f64v.json
for f in bench_f32 bench_f64; do python3 -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['value'], d['roofline']['kernel_ms'], d['pipeline_roofline']['viterbi_kernel_ms'], d['e2e']['ms_per_step'])"; done
