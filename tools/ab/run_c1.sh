ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --config 1 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv,re,collections
rows=[r for r in csv.reader(open('gpurun_out/launches_c1.csv')) if len(r)>5]
idx={h:i for i,h in enumerate(rows[0])}
for r in rows[1:]:
    name=re.sub(r'\(.*','',r[idx['Kernel Name']]).replace('void ','')
    print(f"{name:60s} {float(r[idx['Metric Value']].replace(',',''))/1e3:9.2f} us  grid={r[idx['Grid Size']] if 'Grid Size' in idx else ''}")
PY
