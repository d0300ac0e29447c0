timeout 900 python -m pytest tests/test_gpu_setup.py -q -x 2>&1 | tail -1
python bench.py --config 5 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phases'])"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_scan_ -c 12 python -c "
from paper_1811_11629_b200 import paramfactory
paramfactory.safe_primes_u32(1 << 31, 1 << 32)" 2>&1 | grep -E "^  k_scan|gpu__time" | paste - - | awk '{print $1, $(NF)}'
