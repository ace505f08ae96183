#!/bin/bash
# developer A/B: build libhiermoe.<name>.so with extra nvcc flags on one source
# (SRC=gemm_sm100 by default, or SRC=layer)
# usage: [SRC=layer] tools/variant_build.sh <name> [-DFOO ...]
set -eu
cd "$(dirname "$0")/.."
name=$1; shift
P=paper_2508_09591_b200
B=$P/build
SRC=${SRC:-gemm_sm100}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden -I include "$@" -c $P/csrc/$SRC.cu -o $B/${SRC}_$name.o
objs="$B/planner.cu.o $B/layer.cu.o $B/gemm_sm100.cu.o $B/migrate.cu.o"
objs=${objs/$B\/$SRC.cu.o/$B\/${SRC}_$name.o}
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libhiermoe.$name.so $objs -lcudart_static -lrt -ldl -lpthread
echo built $P/libhiermoe.$name.so
