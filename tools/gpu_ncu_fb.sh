#!/bin/bash
mkdir -p gpurun_out
for dt in float32 float64; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fb_" -c 1 -o gpurun_out/fbc_${dt} python tools/prof_kernels.py --dtype $dt --reps 1 --only fb > gpurun_out/ncu_fbc_${dt}.log 2>&1
done
ls -la gpurun_out
