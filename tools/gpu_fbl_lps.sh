#!/bin/bash
# A/B of lanes per state in fb_large_kernel (LOGHMM_FBL_LPS) on a shortened c5.
mkdir -p gpurun_out
for l in 1 2 4; do
  LOGHMM_FBL_LPS=$l timeout 600 python -m pytest tests -x -q -m gpu -k "large_k_posteriors" > gpurun_out/fbl_pt_$l.log 2>&1; echo "lps $l tests: $(tail -1 gpurun_out/fbl_pt_$l.log)"
  LOGHMM_FBL_LPS=$l timeout 300 python bench.py --config c5 --T 4096 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fbl_$l.json 2> gpurun_out/fbl_$l.err
  python3 -c "import json; d=json.loads(open('gpurun_out/fbl_$l.json').read().strip().splitlines()[-1]); print('lps $l', round(d['ms_per_step'],3), 'ms fb', round(d['roofline']['kernel_ms'],3), 'vit', round(d['pipeline_roofline']['viterbi_kernel_ms'],3))" || tail -3 gpurun_out/fbl_$l.err
done
