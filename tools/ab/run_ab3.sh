# A/B of the fl(c) formation in float-only fills (RSA_FL_FMA 0 / 2 / 3)
for v in fl2 fl3; do
  echo "== tests $v"; RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 600 python -m pytest tests/test_gpu_fill.py tests/test_gpu_garner.py tests/test_gpu_fused.py -x -q 2>&1 | tail -1
done
for rep in 1 2; do
for v in base fl2 fl3; do
  echo "== $v"
  RSARAND_B200_LIB=tools/ab/lib_$v.so python bench.py --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), {k:round(v['gnumbers_s'],2) for k,v in d['roofline']['per_exponent'].items()})"
  RSARAND_B200_LIB=tools/ab/lib_$v.so python bench.py --config 4 --no-e2e --no-cpu --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['value'],2))"
done
done
