#!/bin/bash
# A/B of two library builds on the same box (interleaved): HM_LIB picks the build
set -u
OUT=gpurun_out/ab
mkdir -p $OUT
: > $OUT/ab.jsonl
for rep in 1 2 3; do
  for v in a b; do
    echo "{\"variant\": \"$v\", \"rep\": $rep}" >> $OUT/ab.jsonl
    HM_LIB=paper_2508_09591_b200/libhiermoe.$v.so timeout 300 python ${1:-tools/gemm_probe.py} >> $OUT/ab.jsonl 2>&1
  done
done
echo done
