#!/bin/bash
# A/B of lanes per destination state in viterbi_large_kernel (LOGHMM_VL_LPS).
mkdir -p gpurun_out
for l in 1 2 4; do
  LOGHMM_VL_LPS=$l timeout 600 python -m pytest tests -x -q -m gpu -k "large_k" > gpurun_out/vl_pt_$l.log 2>&1; echo "lps $l tests: $(tail -1 gpurun_out/vl_pt_$l.log)"
  for dt in float32 float64; do
  LOGHMM_VL_LPS=$l timeout 300 python bench.py --config c5 --dtype $dt --T 4096 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/vl.json 2> gpurun_out/vl.err
  python3 -c "import json; d=json.loads(open('gpurun_out/vl.json').read().strip().splitlines()[-1]); print('lps $l $dt', round(d['ms_per_step'],3), 'ms fb', round(d['roofline']['kernel_ms'],3), 'vit', round(d['pipeline_roofline']['viterbi_kernel_ms'],3))" || tail -3 gpurun_out/vl.err
  done
done
