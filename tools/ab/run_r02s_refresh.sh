# session-2 refresh: default bench line, reference arm, launch list of the default run
python bench.py --steps 20 --warmup 5 > gpurun_out/r02s_bench_default.json 2> gpurun_out/r02s_bench_default.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/r02s_bench_reference_arm.json 2> gpurun_out/r02s_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02s_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02s_ncu_launch.log 2>&1; echo "ncu rc=$?"
