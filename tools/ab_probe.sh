#!/bin/bash
# A/B of library builds on the same box (interleaved): HM_LIB picks the build.
# usage: tools/ab_probe.sh <probe.py> <variant> [<variant> ...]
set -u
OUT=gpurun_out/ab
mkdir -p $OUT
: > $OUT/ab.jsonl
probe=$1; shift
for rep in 1 2 3; do
  for v in "$@"; do
    echo "{\"variant\": \"$v\", \"rep\": $rep}" >> $OUT/ab.jsonl
    HM_LIB=paper_2508_09591_b200/libhiermoe.$v.so timeout 300 python $probe >> $OUT/ab.jsonl 2>&1
  done
done
echo done
