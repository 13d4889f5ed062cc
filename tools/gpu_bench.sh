#!/bin/bash
# headline bench (fp32 line + fp64 per_dtype + cpu baseline), the reference arm, and the FB traffic capture
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,l1tex__m_l1tex2xbar_write_bytes.sum,gpu__time_duration.sum -k regex:"fb_chunk|fb_small" --csv --print-units base --log-file gpurun_out/traffic.csv python tools/fb_traffic.py > gpurun_out/traffic.log 2>&1
