#!/bin/bash
# config 5 (K=64, T=65536, banded): large-K parity tests, then the c5 bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "large_k" --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_largek.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_largek.log
tail -5 gpurun_out/pytest_largek.log
for dt in float32 float64; do
  timeout 900 python bench.py --config c5 --dtype $dt --no-cpu-baseline --single-dtype --steps 3 --warmup 3 > gpurun_out/bench_c5_$dt.json 2> gpurun_out/bench_c5_$dt.err
  python3 -c "import json; d=json.loads(open('gpurun_out/bench_c5_$dt.json').read().strip().splitlines()[-1]); print('c5 $dt', round(d['ms_per_step'],2), 'ms; fb', round(d['roofline']['kernel_ms'],2), 'vit', round(d['pipeline_roofline']['viterbi_kernel_ms'],2))"
done
