timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --config 1 --no-e2e --no-cpu > gpurun_out/bench_c1.json 2>/dev/null; python -c "import json; print(json.load(open('gpurun_out/bench_c1.json'))['per_mv'])"
python tools/host_latency.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --config 1 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv,re
rows=[r for r in csv.reader(open('gpurun_out/launches_c1.csv')) if len(r)>5]
idx={h:i for i,h in enumerate(rows[0])}
for r in rows[1:]:
    name=re.sub(r'\(.*','',r[idx['Kernel Name']]).replace('void ','')
    if 'seg' in name or 'fill' in name: print(f"{name:40s} {float(r[idx['Metric Value']].replace(',',''))/1e3:9.2f} us grid={r[idx['Grid Size']]}")
PY
