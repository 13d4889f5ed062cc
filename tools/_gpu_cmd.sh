timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu2.log 2>&1; tail -15 gpurun_out/pytest_gpu2.log
for dt in float32 float64; do timeout 120 python tools/prof_kernels.py --only vit --dtype $dt; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:viterbi -c 1 -f -o gpurun_out/prof_vitk5 python tools/prof_kernels.py --only vit --reps 1 > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log
