#!/bin/bash
# builds the A/B variants of the draw path into tools/variants/bin/
set -e
cd "$(dirname "$0")"
mkdir -p bin
build() { nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -o bin/$1 bench_variants.cu ${@:2} & }
build v_base
build v_add -DADD=1
build v_skip -DSKIP=1
build v_fl -DFL=1
build v_div -DDIV=1
build v_clamp -DCLAMP=1
build v_all -DADD=1 -DSKIP=1 -DFL=1 -DDIV=1 -DCLAMP=1
build v_base1 -DLPT=1
build v_all1 -DADD=1 -DSKIP=1 -DFL=1 -DDIV=1 -DCLAMP=1 -DLPT=1
build v_fldivclamp -DFL=1 -DDIV=1 -DCLAMP=1
wait
