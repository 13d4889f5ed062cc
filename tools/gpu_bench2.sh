#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_kl.json 2>&1
LOGHMM_VIT_ALGO=pair timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_pair.json 2>&1
LOGHMM_VIT_ALGO=pair timeout 300 python tools/prof_kernels.py --dtype float32 --only vit > gpurun_out/prof_vit_pair.json 2>&1
LOGHMM_VIT_ALGO=pair timeout 600 ncu --set full --clock-control none -k regex:"viterbi" -c 1 -o gpurun_out/vit_pair python tools/prof_kernels.py --dtype float32 --reps 1 --only vit > gpurun_out/ncu_vp.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"viterbi" -c 1 -o gpurun_out/vit_kl python tools/prof_kernels.py --dtype float32 --reps 1 --only vit > gpurun_out/ncu_vk.log 2>&1
for f in gpurun_out/bench_kl.json gpurun_out/bench_pair.json; do python3 -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['value'], d['roofline']['kernel_ms'], d['pipeline_roofline']['viterbi_kernel_ms'], d['e2e']['ms_per_step'])"; done
cat gpurun_out/prof_vit_pair.json
