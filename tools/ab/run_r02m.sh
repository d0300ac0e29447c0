#!/bin/bash
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02m_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02m_ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_bat_|k_pw_" -c 12 -o gpurun_out/r02m_prof_battery -f python tools/prof_battery_kernels.py > gpurun_out/r02m_ncu_battery.log 2>&1; echo "ncu battery rc=$?"
