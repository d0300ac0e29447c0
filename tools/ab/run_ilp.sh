# SPRP ladders interleaved per thread (RSA_SPRP_ILP) in the scan and the literal census
for rep in 1 2; do for v in ilp2 ilp1 ilp4; do
  echo "== $v"; RSARAND_B200_LIB=tools/ab/lib_$v.so python bench.py --config 5 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['phases']['scan_ms'],4), round(d['literal_mr']['ms'],2), d['literal_mr']['equal_count'])"
done; done
