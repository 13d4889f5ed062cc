#!/bin/bash
# pipeline composition matrix: Viterbi variant (fp32 config 2, graph replay, Viterbi launched first)
mkdir -p gpurun_out
run() {
  timeout 300 python bench.py --no-cpu-baseline --single-dtype > gpurun_out/pm_$1.json 2> gpurun_out/pm_$1.err
  python3 -c "import json; d=json.loads(open('gpurun_out/pm_$1.json').read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step']*1e3,1), round(d['roofline']['kernel_ms']*1e3,1), round(d['pipeline_roofline']['viterbi_kernel_ms']*1e3,1))"
}
LOGHMM_VIT_ALGO=lanes run lanes
LOGHMM_VIT_ALGO=chain LOGHMM_VIT_NW=8 run nw8
LOGHMM_VIT_ALGO=chain LOGHMM_VIT_NW=16 run nw16
LOGHMM_PIPE_ORDER=serial LOGHMM_VIT_ALGO=chain LOGHMM_VIT_NW=16 run nw16_serial
