#!/bin/bash
# Build a copy of librsarand_b200.so with extra nvcc flags for an A/B run:
#   tools/ab/build_lib_variant.sh NAME -DRSA_SIEVE_MAX=8192
#   RSARAND_B200_LIB=tools/ab/lib_NAME.so python bench.py --config 5
set -e
cd "$(dirname "$0")/../.."
name=$1; shift
out=tools/ab/obj_$name; mkdir -p "$out"
for f in paper_1811_11629_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC,-O2 -Iinclude "$@" \
       -c "$f" -o "$out/$(basename "${f%.cu}").o" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/ab/lib_$name.so "$out"/*.o
rm -rf "$out"
echo tools/ab/lib_$name.so
