#!/bin/bash
# A/B: bench.py under env settings given as arguments ("NAME=VAL NAME2=VAL" per arg, "-" = none)
mkdir -p gpurun_out
: > gpurun_out/ab.txt
for setting in "$@"; do
  for rep in 1 2; do
    if [ "$setting" = "-" ]; then envs=""; else envs="$setting"; fi
    line=$(env $envs timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | tail -1)
    echo "$setting | $(echo "$line" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1), "us  fb", round(d["roofline"]["kernel_ms"]*1000,1), "vit", round(d["pipeline_roofline"]["viterbi_kernel_ms"]*1000,1), "e2e", round(d["e2e"]["ms_per_step"]*1000,1))')" >> gpurun_out/ab.txt
  done
done
