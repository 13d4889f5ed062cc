#!/bin/bash
mkdir -p gpurun_out
for s in 1 2 3 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --steps 30 --e2e-slices $s > gpurun_out/bench_s$s.json 2>gpurun_out/bench_s$s.err
  python3 -c "import json; d=json.loads(open('gpurun_out/bench_s$s.json').read().strip().splitlines()[-1]); print('slices=$s', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['launch'])" || tail -3 gpurun_out/bench_s$s.err
done
