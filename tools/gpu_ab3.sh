#!/bin/bash
mkdir -p gpurun_out abtest/B
ln -sf $PWD/paper_2605_29208_b200/_lib/libloghmm_b200.so abtest/B/libloghmm_b200.so
for rep in 1 2 3; do for v in B C; do
  LOGHMM_B200_LIB=$PWD/abtest/$v/libloghmm_b200.so timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ab_$v.json 2>&1
  python3 -c "import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1000,1), round(d['roofline']['kernel_ms']*1000,1), round(d['pipeline_roofline']['viterbi_kernel_ms']*1000,1))"
done; done
for v in B C; do LOGHMM_B200_LIB=$PWD/abtest/$v/libloghmm_b200.so timeout 300 python tools/prof_kernels.py --dtype float32 --only fb; done
