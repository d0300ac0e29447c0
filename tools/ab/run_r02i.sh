#!/bin/bash
for rep in 1 2; do
  for v in x0 x1 x2 x3; do
    RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --sub 3 > gpurun_out/r02i_bench_${v}_$rep.json 2>/dev/null
    echo "$v rep$rep rc=$?"
  done
done
