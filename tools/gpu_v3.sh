#!/bin/bash
# chain-warp Viterbi: parity tests, standalone timings (8 / 16 warps, old K-lane kernel), bench A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "viterbi or Viterbi" -p no:cacheprovider > gpurun_out/pytest_vit.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_vit.log
tail -5 gpurun_out/pytest_vit.log
for nw in 8 16; do
  LOGHMM_VIT_ALGO=chain LOGHMM_VIT_NW=$nw timeout 300 python tools/prof_kernels.py --dtype float32 --only vit > gpurun_out/prof_vit_f32_nw$nw.json 2>&1
  LOGHMM_VIT_ALGO=chain LOGHMM_VIT_NW=$nw timeout 300 python tools/prof_kernels.py --dtype float64 --only vit > gpurun_out/prof_vit_f64_nw$nw.json 2>&1
  LOGHMM_VIT_ALGO=chain LOGHMM_VIT_NW=$nw timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_nw$nw.json 2> gpurun_out/bench_nw$nw.err
done
LOGHMM_VIT_ALGO=lanes timeout 300 python tools/prof_kernels.py --dtype float32 --only vit > gpurun_out/prof_vit_f32_lanes.json 2>&1
LOGHMM_VIT_ALGO=lanes timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_lanes.json 2> gpurun_out/bench_lanes.err
cat gpurun_out/prof_vit_*.json
for f in bench_nw8 bench_nw16 bench_lanes; do python3 -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'], d['pipeline_roofline']['viterbi_kernel_ms'], d['per_dtype']['f64']['ms_per_step'], d['e2e']['ms_per_step'])"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"viterbi_chain" -c 1 -o gpurun_out/v3_f32 python tools/prof_kernels.py --dtype float32 --reps 1 --only vit > gpurun_out/ncu_v3.log 2>&1
