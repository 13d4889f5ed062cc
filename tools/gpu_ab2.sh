#!/bin/bash
# A/B of environment variants on library abtest/C vs the main build (B).
mkdir -p gpurun_out abtest/B
ln -sf $PWD/paper_2605_29208_b200/_lib/libloghmm_b200.so abtest/B/libloghmm_b200.so
run() { # name lib env...
  local name=$1 lib=$2; shift 2
  env "$@" LOGHMM_B200_LIB=$PWD/abtest/$lib/libloghmm_b200.so timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ab_$name.json 2>&1
  python3 -c "import json; d=json.loads(open('gpurun_out/ab_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['ms_per_step']*1000,1), round(d['roofline']['kernel_ms']*1000,1), round(d['pipeline_roofline']['viterbi_kernel_ms']*1000,1))" 2>/dev/null || tail -3 gpurun_out/ab_$name.json
}
for rep in 1 2; do
  run base B X=1
  run c4g C LOGHMM_VIT_GLOBAL=1
  run c8g C LOGHMM_VIT_GLOBAL=1 LOGHMM_VIT_WPB=8
  run c16g C LOGHMM_VIT_GLOBAL=1 LOGHMM_VIT_WPB=16
  run c2g C LOGHMM_VIT_GLOBAL=1 LOGHMM_VIT_WPB=2
done
