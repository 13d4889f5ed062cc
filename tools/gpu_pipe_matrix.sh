#!/bin/bash
# pipeline composition matrix: Viterbi variant x launch order (fp32 config 2, graph replay)
mkdir -p gpurun_out
for v in lanes nw8 nw16; do
  for o in vit_first fb_first serial; do
    if [ $v = lanes ]; then export LOGHMM_VIT_ALGO=lanes; unset LOGHMM_VIT_NW; else unset LOGHMM_VIT_ALGO; export LOGHMM_VIT_NW=${v#nw}; fi
    LOGHMM_PIPE_ORDER=$o timeout 300 python bench.py --no-cpu-baseline --single-dtype > gpurun_out/pm_${v}_${o}.json 2> gpurun_out/pm_${v}_${o}.err
    python3 -c "import json; d=json.loads(open('gpurun_out/pm_${v}_${o}.json').read().strip().splitlines()[-1]); print('$v $o', round(d['ms_per_step']*1e3,1), round(d['roofline']['kernel_ms']*1e3,1), round(d['pipeline_roofline']['viterbi_kernel_ms']*1e3,1))"
  done
done
