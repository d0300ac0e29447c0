# fused histogram counters: u16 read-modify-write (shipped) vs u32 shared atomics
for v in h32 h32m7; do echo "== tests $v"; RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 600 python -m pytest tests/test_gpu_fused.py -q -x 2>&1 | tail -1; done
for rep in 1 2; do for v in h16 h32 h32m7; do
  echo "== $v"; RSARAND_B200_LIB=tools/ab/lib_$v.so python bench.py --config 4 --no-e2e --no-cpu --steps 3 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],2))"
done; done
