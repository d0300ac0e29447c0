#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_battery_fused.py tests/test_gpu_battery.py -x -q -p no:cacheprovider > gpurun_out/r02h_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02h_pytest.log
python tools/prof_battery.py > gpurun_out/r02h_prof_battery.txt 2>&1; tail -26 gpurun_out/r02h_prof_battery.txt
timeout 600 python bench.py --config 6 --no-cpu > gpurun_out/r02h_bench_c6.json 2> gpurun_out/r02h_bench_c6.err; echo "c6 rc=$?"
