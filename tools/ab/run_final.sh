timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench_full.json 2>/dev/null
for c in 1 3 4 5; do python bench.py --config $c --no-e2e > gpurun_out/bench_c$c.json 2>/dev/null; done
python -c "
import json
for f in ['bench_full','bench_c1','bench_c3','bench_c4','bench_c5']:
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, round(d.get('value'),2), round(d.get('ms_per_step'),3), (d.get('roofline') or {}).get('frac'))"
