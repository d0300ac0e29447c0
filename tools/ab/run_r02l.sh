#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_battery.py tests/test_gpu_fill.py -x -q -p no:cacheprovider -k "fourier or battery or launch_counter" > gpurun_out/r02l_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02l_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err; echo "bench rc=$?"
