timeout 900 python -m pytest tests/test_gpu_fill.py -x -q > gpurun_out/t2.log 2>&1; tail -2 gpurun_out/t2.log
python tools/ab/c1_split.py 2>&1
python tools/ab/host_prof2.py 2>&1 | grep -v "^$" | head -30
for rep in 1 2; do
python bench.py --config 1 --no-e2e --no-cpu --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value'],2), d.get('per_mv'))"
done
