timeout 900 python -m pytest tests/test_gpu_setup.py -x -q 2>&1 | tail -2
python bench.py --config 5 --no-e2e --no-cpu > gpurun_out/bench_c5.json 2>gpurun_out/bench_c5.err; tail -3 gpurun_out/bench_c5.err
python -c "import json; d=json.load(open('gpurun_out/bench_c5.json')); print(d['phases']); print(d['literal_mr'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --config 5 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_mr_ -c 2 -o gpurun_out/prof_mr -f python -c "
import paper_1811_11629_b200 as R; from paper_1811_11629_b200 import paramfactory
paramfactory.safe_primes_u32(1<<31, (1<<31) + (1<<28), literal_mr=True)" > gpurun_out/ncu_mr.log 2>&1; tail -2 gpurun_out/ncu_mr.log
