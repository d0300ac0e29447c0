#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02k_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02k_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02k_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02k_ref.json 2> gpurun_out/r02k_ref.err; echo "ref rc=$?"
RSARAND_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/r02k_bench_g2.json 2> gpurun_out/r02k_bench_g2.err; echo "bench2 rc=$?"
