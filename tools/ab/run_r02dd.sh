for v in dd1 dd2; do echo "== tests $v"; RSARAND_B200_LIB=tools/ab/lib_$v.so timeout 600 python -m pytest tests/test_gpu_fill.py tests/test_gpu_fused.py -x -q -k "config3 or float_map or lane_subset or many_instance" 2>&1 | tail -1; done
for rep in 1 2 3; do for lib in paper_1811_11629_b200/librsarand_b200.so tools/ab/lib_dd1.so tools/ab/lib_dd2.so; do
  echo "$lib $(RSARAND_B200_LIB=$lib python bench.py --config 3 --no-e2e --no-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2))")"
done; done
