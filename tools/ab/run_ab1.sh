set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for lib in tools/ab/lib_nogf.so paper_1811_11629_b200/librsarand_b200.so tools/ab/lib_nogf.so paper_1811_11629_b200/librsarand_b200.so; do
  echo "== $lib"
  RSARAND_B200_LIB=$lib python bench.py --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], {k:round(v['gnumbers_s'],2) for k,v in d['roofline']['per_exponent'].items()})"
  RSARAND_B200_LIB=$lib python bench.py --config 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'])"
  RSARAND_B200_LIB=$lib python bench.py --config 4 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'])"
done
