#!/bin/bash
# round 2: full GPU tests + smoke + default bench + ncu launch list + ncu --set full of the fills / fused
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02d_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02d_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02d_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02d_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -c 4 -o gpurun_out/r02d_prof_fill -f python tools/prof_fill.py 3 5 17 65537 > gpurun_out/r02d_ncu_fill.log 2>&1; echo "ncu fill rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -c 1 -o gpurun_out/r02d_prof_c3 -f python bench.py --config 3 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r02d_ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/r02d_prof_fused -f python bench.py --config 4 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r02d_ncu_fused.log 2>&1; echo "ncu fused rc=$?"
ls -la gpurun_out/r02d_*
