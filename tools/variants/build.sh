#!/bin/bash
# builds the A/B variants of the draw path into tools/variants/bin/
set -e
cd "$(dirname "$0")"
rm -rf bin; mkdir -p bin
build() { nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -Xptxas -v -o bin/$1 bench_variants.cu ${@:2} 2> bin/$1.ptxas & }
build v_base
build v_m6 -DMINB=6
build v_m8 -DMINB=8
build v_l4 -DLPT=4
build v_l4m4 -DLPT=4 -DMINB=4
build v_l1m8 -DLPT=1 -DMINB=8
build v_l1 -DLPT=1
wait
