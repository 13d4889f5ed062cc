#!/bin/bash
# full ncu capture (with source) of the fp32 config-2 forward-backward kernel, standalone
mkdir -p gpurun_out
timeout 300 python tools/prof_kernels.py --dtype float32 --only fb > gpurun_out/prof_fb_f32.json 2>&1
cat gpurun_out/prof_fb_f32.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fb_chunk" -c 1 -o gpurun_out/fbc_f32 python tools/prof_kernels.py --dtype float32 --reps 1 --only fb > gpurun_out/ncu_fbc.log 2>&1
tail -3 gpurun_out/ncu_fbc.log
