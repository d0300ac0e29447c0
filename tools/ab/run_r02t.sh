#!/bin/bash
for v in u2 u3; do
  RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 900 python -m pytest tests/test_gpu_fill.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "not config4" > gpurun_out/r02t_pytest_$v.log 2>&1
  echo "$v pytest rc=$? $(tail -1 gpurun_out/r02t_pytest_$v.log)"
done
for rep in 1 2; do
  for v in u0 u1 u2 u3; do
    RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --sub 3 > gpurun_out/r02t_bench_${v}_$rep.json 2>/dev/null
    echo "$v rep$rep rc=$?"
  done
done
