timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench_full.json 2>/dev/null
python bench.py --config 6 --no-e2e --no-cpu > gpurun_out/bench_c6.json 2>/dev/null
python bench.py --impl reference > gpurun_out/bench_ref.json 2>/dev/null
python -c "
import json
for f in ['bench_full','bench_c6','bench_ref']:
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'))"
