#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log; tail -3 gpurun_out/pytest_all.log
timeout 300 python tools/prof_kernels.py --dtype float64 --only fb
for spec in "c2 float64" "c2 float32" "c5 float64" "c3 float64" "c4 float64"; do set -- $spec
  timeout 600 python bench.py --config $1 --dtype $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$1_$2.json 2> gpurun_out/bench_$1_$2.err
  python3 -c "import json; d=json.loads(open('gpurun_out/bench_$1_$2.json').read().strip().splitlines()[-1]); print('$1 $2', round(d['ms_per_step'],4), 'ms', '%.3e'%d['value'], round(d['roofline']['kernel_ms'],4), round(d['pipeline_roofline']['viterbi_kernel_ms'],4))" || tail -3 gpurun_out/bench_$1_$2.err
done
