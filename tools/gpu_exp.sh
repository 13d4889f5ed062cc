#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "config5 or c5 or large or ragged" > gpurun_out/pytest_sub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sub.log; tail -3 gpurun_out/pytest_sub.log
for dt in float32 float64; do
  timeout 600 python bench.py --config c5 --dtype $dt --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_$dt.json 2> gpurun_out/bench_c5_$dt.err
  python3 -c "import json; d=json.loads(open('gpurun_out/bench_c5_$dt.json').read().strip().splitlines()[-1]); print('c5 $dt', round(d['ms_per_step'],3), 'ms', '%.3e'%d['value'], round(d['roofline']['kernel_ms'],3), round(d['pipeline_roofline']['viterbi_kernel_ms'],3))" || tail -3 gpurun_out/bench_c5_$dt.err
done
