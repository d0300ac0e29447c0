# round-2 (session 2) A/B: instance constants as grid constants (vu), rare-case skip reduction (vb)
for v in vu vb; do
  echo "== tests $v"; RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 600 python -m pytest tests/test_gpu_fill.py tests/test_gpu_garner.py -x -q 2>&1 | tail -1
done
for rep in 1 2; do
for lib in paper_1811_11629_b200/librsarand_b200.so tools/ab/lib_vu.so tools/ab/lib_vb.so; do
  echo "== $lib"
  RSARAND_B200_LIB=$lib python bench.py --no-e2e --no-cpu --no-sub --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), {k:round(v['gnumbers_s'],2) for k,v in d['roofline']['per_exponent'].items()})"
  RSARAND_B200_LIB=$lib python bench.py --config 3 --no-e2e --no-cpu --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', round(d['value'],2))"
done
done
