#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_battery_fused.py tests/test_gpu_battery.py -x -q -p no:cacheprovider > gpurun_out/r02j_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02j_pytest.log
python tools/prof_battery.py > gpurun_out/r02j_prof_battery.txt 2>&1; grep -E "max_of_t|permutation|total" gpurun_out/r02j_prof_battery.txt
for rep in 1 2; do
  for v in x0 x3; do
    RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --sub 3 > gpurun_out/r02j_bench_${v}_$rep.json 2>/dev/null
    echo "$v rep$rep rc=$?"
  done
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo "bench rc=$?"
