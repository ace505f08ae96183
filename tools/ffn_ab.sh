#!/bin/bash
# A/B of library builds on tools/ffn_bench.py (interleaved): HM_LIB picks the build
set -u
OUT=gpurun_out/ab
mkdir -p $OUT
: > $OUT/ffn_ab.jsonl
for rep in 1 2; do
  for v in "$@"; do
    echo "{\"variant\": \"$v\", \"rep\": $rep}" >> $OUT/ffn_ab.jsonl
    HM_LIB=paper_2508_09591_b200/libhiermoe.$v.so timeout 300 python tools/ffn_bench.py >> $OUT/ffn_ab.jsonl 2>&1
  done
done
echo done
