#!/bin/bash
# round 2 A/B: source variants of the draw path (tools/ab/lib_*.so), parity tests + bench
mkdir -p gpurun_out
for v in v0 v2 v6 v7; do
  RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 900 python -m pytest tests/test_gpu_fill.py tests/test_gpu_garner.py tests/test_gpu_fused.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/r02b_pytest_$v.log 2>&1
  echo "$v pytest rc=$? $(tail -1 gpurun_out/r02b_pytest_$v.log)"
done
for rep in 1 2; do
  for v in v0 v2 v6 v7; do
    RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02b_bench_${v}_$rep.json 2>/dev/null
    echo "$v rep$rep rc=$?"
  done
done
