#!/bin/bash
# Round-2 final GPU round trip: every parity test, smoke, the headline bench (fp32 + per_dtype
# fp64 + CPU baseline), the reference arm, the ncu launch list of an eager step, full captures
# of the hot kernels, the FB traffic capture, the auxiliary configs.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/prof_kernels.py --dtype float32 > gpurun_out/prof_f32.json 2>&1
timeout 300 python tools/prof_kernels.py --dtype float64 > gpurun_out/prof_f64.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_f32.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-graph --single-dtype > gpurun_out/ncu_launch.log 2>&1
# (the .ncu-rep files exceed the 64 MiB return limit: summarised on the box, then removed)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fb_chunk|viterbi_small|reduce_mstep" -c 3 -o /tmp/full_f32 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-graph --single-dtype > gpurun_out/ncu_full.log 2>&1
python tools/summarize_ncu.py /tmp/full_f32.ncu-rep > gpurun_out/ncu_full_f32.md 2>&1
python tools/ncu_regions.py /tmp/full_f32.ncu-rep fb_chunk > gpurun_out/fb_chunk_regions.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"fb_small" -c 1 -o /tmp/full_f64 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-graph --single-dtype --dtype float64 > gpurun_out/ncu_full64.log 2>&1
python tools/summarize_ncu.py /tmp/full_f64.ncu-rep > gpurun_out/ncu_full_f64_fb.md 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,l1tex__m_l1tex2xbar_write_bytes.sum,gpu__time_duration.sum -k regex:"fb_chunk|fb_small" --csv --print-units base --log-file gpurun_out/traffic.csv python tools/fb_traffic.py > gpurun_out/traffic.log 2>&1
for c in c3 c4; do
  timeout 600 python bench.py --config $c --dtype float64 --no-cpu-baseline --single-dtype --steps 10 --warmup 3 > gpurun_out/bench_${c}_float64.json 2> gpurun_out/bench_${c}.err
done
for dt in float32 float64; do
  timeout 900 python bench.py --config c5 --dtype $dt --no-cpu-baseline --single-dtype --steps 3 --warmup 3 > gpurun_out/bench_c5_$dt.json 2> gpurun_out/bench_c5_$dt.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c5_f32_T8192.csv python tools/prof_c5.py --T 8192 --reps 1 > gpurun_out/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"fb_split_sweep|viterbi_large" -c 4 -o /tmp/full_c5 python tools/prof_c5.py --T 8192 --reps 1 > gpurun_out/ncu_c5_full.log 2>&1
python tools/summarize_ncu.py /tmp/full_c5.ncu-rep > gpurun_out/ncu_c5_sparse_f32.md 2>&1
rm -f /tmp/full_f32.ncu-rep /tmp/full_f64.ncu-rep /tmp/full_c5.ncu-rep
ls -la gpurun_out | head -50
