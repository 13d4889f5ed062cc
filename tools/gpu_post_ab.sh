mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "large_k" > gpurun_out/p_pt.log 2>&1; tail -1 gpurun_out/p_pt.log
for dt in float32 float64; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"fb_post|fb_split" --log-file gpurun_out/p_$dt.csv python bench.py --config c5 --dtype $dt --T 4096 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
python3 - $dt <<'PY'
import csv,collections,io,sys
txt=open('gpurun_out/p_%s.csv'%sys.argv[1]).read().splitlines()
i=[k for k,l in enumerate(txt) if l.startswith('"ID"')][0]
d=collections.defaultdict(list)
for r in csv.DictReader(io.StringIO("\n".join(txt[i:]))): d[r['Kernel Name'][:40]].append(float(r['Metric Value']))
for k,v in d.items(): print(sys.argv[1], round(sum(v)/len(v)/1e3,1),'us', k)
PY
done
