#!/bin/bash
# Kernel-level timing (both FB decompositions, both dtypes) and full ncu
# captures of the FB and Viterbi kernels at config 2.
mkdir -p gpurun_out
for dt in float32 float64; do
  for algo in chunked mitm; do
    LOGHMM_FB_ALGO=$algo timeout 300 python tools/prof_kernels.py --dtype $dt > gpurun_out/prof_${dt}_${algo}.json 2>&1
  done
done
for dt in float32 float64; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fb_small|viterbi_small|reduce_mstep" -c 3 -o gpurun_out/full_${dt} python tools/prof_kernels.py --dtype $dt --reps 1 > gpurun_out/ncu_full_${dt}.log 2>&1
done
ls -la gpurun_out
