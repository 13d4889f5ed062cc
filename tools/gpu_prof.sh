#!/bin/bash
# Kernel-level timing (both FB decompositions, both dtypes) and full ncu
# captures of the FB kernel at config 2 (one launch each, to stay small).
mkdir -p gpurun_out
for dt in float32 float64; do
  for algo in chunked mitm; do
    LOGHMM_FB_ALGO=$algo timeout 300 python tools/prof_kernels.py --dtype $dt > gpurun_out/prof_${dt}_${algo}.json 2>&1
  done
done
for dt in float32 float64; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fb_small" -c 1 -o gpurun_out/fb_${dt} python tools/prof_kernels.py --dtype $dt --reps 1 --only fb > gpurun_out/ncu_fb_${dt}.log 2>&1
done
LOGHMM_FB_ALGO=mitm timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fb_mitm" -c 1 -o gpurun_out/fbm_float32 python tools/prof_kernels.py --dtype float32 --reps 1 --only fb > gpurun_out/ncu_fbm.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"reduce_mstep" -c 1 -o gpurun_out/rm_float32 python tools/prof_kernels.py --dtype float32 --reps 1 --only small > gpurun_out/ncu_rm.log 2>&1
du -sh gpurun_out/*
