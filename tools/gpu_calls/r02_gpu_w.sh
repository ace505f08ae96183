#!/bin/bash
set -u
OUT=gpurun_out/r02w
mkdir -p $OUT
for v in a k i; do
  echo "{\"variant\": \"$v\"}" >> $OUT/grid.jsonl
  HM_LIB=paper_2508_09591_b200/libhiermoe.$v.so timeout 600 python tools/gemm_probe.py --grid=148 --grid=128 --grid=112 --grid=96 --grid=74 >> $OUT/grid.jsonl 2>&1
done
echo done
