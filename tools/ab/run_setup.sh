timeout 900 python -m pytest tests/test_gpu_setup.py -q -x 2>&1 | tail -2
python bench.py --config 5 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases'])"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_setup -c 3 python -c "
import paper_1811_11629_b200 as R
for _ in range(3): R.derive_params_table(R.DEFAULT_MASTER_SEED, 0, 1 << 20)" 2>&1 | grep -E "k_setup|gpu__time_duration" | tail -6
