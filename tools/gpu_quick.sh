#!/bin/bash
# Quick GPU check: new-kernel parity tests, kernel timings, one ncu capture.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "equal_length or estep_statistics" > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
timeout 300 python tools/prof_kernels.py --dtype float32 > gpurun_out/prof_f32.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fb_chunk" -c 1 -o gpurun_out/fbc_float32 python tools/prof_kernels.py --dtype float32 --reps 1 --only fb > gpurun_out/ncu_fbc_float32.log 2>&1
tail -3 gpurun_out/pytest_new.log; cat gpurun_out/prof_f32.json
