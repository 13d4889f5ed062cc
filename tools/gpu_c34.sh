#!/bin/bash
# configs 3 / 4 (Student-t ECME, Gamma + von Mises): Viterbi layout A/B
for c in c3 c4; do
  for v in lanes chain auto; do
    if [ $v = auto ]; then unset LOGHMM_VIT_ALGO; else export LOGHMM_VIT_ALGO=$v; fi
    timeout 600 python bench.py --config $c --dtype float64 --no-cpu-baseline --single-dtype --steps 10 --warmup 3 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $v', round(d['ms_per_step'],3), 'fb', round(d['roofline']['kernel_ms'],3), 'vit', round(d['pipeline_roofline']['viterbi_kernel_ms'],3))"
  done
done
