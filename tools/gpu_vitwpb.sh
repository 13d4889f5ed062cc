#!/bin/bash
# A/B of the Viterbi CTA size (LOGHMM_VIT_WPB) inside the config-2 pipeline step.
mkdir -p gpurun_out
for w in 4 8 2 16 4 8; do
  LOGHMM_VIT_WPB=$w timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/vw_$w.json 2> gpurun_out/vw_$w.err
  python3 -c "import json; d=json.loads(open('gpurun_out/vw_$w.json').read().strip().splitlines()[-1]); print('wpb $w', round(d['ms_per_step']*1e3,1), 'us fb', round(d['roofline']['kernel_ms']*1e3,1), 'vit', round(d['pipeline_roofline']['viterbi_kernel_ms']*1e3,1))" || tail -3 gpurun_out/vw_$w.err
done
