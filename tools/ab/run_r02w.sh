timeout 900 python -m pytest tests/test_gpu_fill.py tests/test_gpu_garner.py tests/test_gpu_fused.py -x -q > gpurun_out/t1.log 2>&1; tail -2 gpurun_out/t1.log
python tools/ab/c1_split.py > gpurun_out/c1_split2.txt 2>&1; cat gpurun_out/c1_split2.txt
for rep in 1 2; do
python bench.py --no-e2e --no-cpu --no-sub --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), {k:round(v['gnumbers_s'],2) for k,v in d['roofline']['per_exponent'].items()})"
python bench.py --config 3 --no-e2e --no-cpu --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['value'],2))"
python bench.py --config 1 --no-e2e --no-cpu --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value'],2), d.get('per_mv'))"
done
