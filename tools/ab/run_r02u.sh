#!/bin/bash
for v in m1 m2; do
  RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 900 python -m pytest tests/test_gpu_setup.py -x -q -p no:cacheprovider > gpurun_out/r02u_pytest_$v.log 2>&1
  echo "$v pytest rc=$? $(tail -1 gpurun_out/r02u_pytest_$v.log)"
done
for rep in 1 2; do
  for v in m0 m1 m2; do
    RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$rep', round(d['ms_per_step'],4), d['phases']['scan_ms'], d['literal_mr']['ms'], round(d['literal_mr']['roofline']['frac'],3))"
  done
done
