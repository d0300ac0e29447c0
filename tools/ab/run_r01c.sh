# tests, default bench, config 3/4 lines, launch list and ncu --set full of the fills + fused
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --config 3 --no-e2e > gpurun_out/bench_c3.json 2>&1
python bench.py --config 4 --no-e2e > gpurun_out/bench_c4.json 2>&1
python bench.py --config 1 --no-e2e > gpurun_out/bench_c1.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fill_fast -o gpurun_out/prof_fill_r01c -f python tools/prof_fill.py > gpurun_out/ncu_fill.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o gpurun_out/prof_fused_r01c -f python bench.py --config 4 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_fused.log 2>&1
ls -la gpurun_out
