timeout 900 python -m pytest tests/test_gpu_fill.py -x -q -k "segmented or scalar or lookahead or replay or concurrent or buffers" 2>&1 | tail -1
for rep in 1 2; do for lib in paper_1811_11629_b200/librsarand_b200.so tools/ab/lib_pd2.so; do echo "== $lib"; RSARAND_B200_LIB=$lib python tools/ab/c1_split.py 2>&1 | head -2; done; done
python bench.py --config 1 --no-e2e --no-cpu --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value'],2), d.get('per_mv'))"
