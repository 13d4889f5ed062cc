#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "equal_length or estep or config2 or baum_welch" > gpurun_out/pytest_sub.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sub.log; tail -2 gpurun_out/pytest_sub.log
timeout 300 python tools/prof_kernels.py --dtype float32 > gpurun_out/prof_f32.json 2>&1; cat gpurun_out/prof_f32.json
for w in 4 1; do
  LOGHMM_VIT_WPB=$w timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_w$w.json 2>&1
  python3 -c "import json; d=json.loads(open('gpurun_out/bench_w$w.json').read().strip().splitlines()[-1]); print('wpb=$w', d['ms_per_step'], d['roofline']['kernel_ms'], d['pipeline_roofline']['viterbi_kernel_ms'], d['e2e']['ms_per_step'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_launch.log 2>&1
python3 - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches.csv')))
i=[k for k,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[i]
for r in rows[i+1:]:
    d=dict(zip(h,r)); print(d['Kernel Name'][:70], d['Metric Value'])
PY
