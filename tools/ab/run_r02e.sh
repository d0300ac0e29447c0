#!/bin/bash
# round 2: F1 fused battery tests + config 6 timing
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_battery_fused.py tests/test_gpu_battery.py tests/test_gpu_bitsource.py -x -q -p no:cacheprovider > gpurun_out/r02e_pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/r02e_pytest.log
timeout 600 python bench.py --config 6 --no-cpu > gpurun_out/r02e_bench_c6.json 2> gpurun_out/r02e_bench_c6.err; echo "c6 rc=$?"; tail -3 gpurun_out/r02e_bench_c6.err
