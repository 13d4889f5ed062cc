#!/bin/bash
# A/B of the e2e host-to-device slice count (bench.py --e2e-slices).
mkdir -p gpurun_out
for rep in 1 2; do for s in 1 2 3 4 6 8; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-slices $s > gpurun_out/e2e_$s.json 2> gpurun_out/e2e_$s.err
  python3 -c "import json; d=json.loads(open('gpurun_out/e2e_$s.json').read().strip().splitlines()[-1]); print('slices $s', round(d['e2e']['ms_per_step']*1e3,1), 'us e2e', round(d['ms_per_step']*1e3,1), 'us dev')" || tail -2 gpurun_out/e2e_$s.err
done; done
