#!/bin/bash
# Auxiliary bench lines for BASELINE configs 3-5 and a capture of the K=64 kernels.
mkdir -p gpurun_out
for spec in "c3 float64" "c4 float64" "c4 float32" "c5 float32" "c5 float64"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --dtype $2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$1_$2.json 2> gpurun_out/bench_$1_$2.err
  python3 -c "import json; d=json.loads(open('gpurun_out/bench_$1_$2.json').read().strip().splitlines()[-1]); print('$1 $2', round(d['ms_per_step'],3), 'ms', '%.3e'%d['value'], 'frac', round(d['pipeline_roofline']['frac'],3), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), round(d['pipeline_roofline']['viterbi_kernel_ms'],3))" || tail -3 gpurun_out/bench_$1_$2.err
done
#timeout 600 python bench.py --config c5 --impl reference --steps 1 --warmup 1 > gpurun_out/bench_c5_ref.json 2>&1; tail -1 gpurun_out/bench_c5_ref.json | cut -c1-300
#timeout 900 ncu --set full --clock-control none -k regex:"large" -c 2 -o gpurun_out/c5_large python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/ncu_c5.log 2>&1
