timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/host_latency.py
python bench.py --config 1 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['per_mv'])"
