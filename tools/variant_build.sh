#!/bin/bash
# developer A/B: build libhiermoe.<name>.so with extra nvcc flags on gemm_sm100.cu
# usage: tools/variant_build.sh <name> [-DFOO ...]
set -eu
cd "$(dirname "$0")/.."
name=$1; shift
P=paper_2508_09591_b200
B=$P/build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden -I include "$@" -c $P/csrc/gemm_sm100.cu -o $B/gemm_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libhiermoe.$name.so $B/planner.cu.o $B/layer.cu.o $B/gemm_$name.o $B/migrate.cu.o -lcudart_static -lrt -ldl -lpthread
echo built $P/libhiermoe.$name.so
