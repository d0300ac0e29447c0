#!/bin/bash
# Build a copy of librsarand_b200.so from an alternative csrc directory (A/B of
# source-level variants):  tools/ab/build_src_variant.sh NAME /path/to/csrc
#   RSARAND_B200_LIB=tools/ab/lib_NAME.so python bench.py ...
# The csrc copy must sit two levels below a directory holding include/ (the
# sources include ../../include/rsarand_b200.h).
set -e
cd "$(dirname "$0")/../.."
name=$1; src=$2
out=tools/ab/obj_$name; mkdir -p "$out"
pids=()
for f in "$src"/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC,-O2 -Iinclude \
       -c "$f" -o "$out/$(basename "${f%.cu}").o" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/ab/lib_$name.so "$out"/*.o
rm -rf "$out"
echo tools/ab/lib_$name.so
