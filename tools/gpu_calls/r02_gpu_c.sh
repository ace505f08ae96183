#!/bin/bash
set -u
OUT=gpurun_out/r02c
mkdir -p $OUT
timeout 300 python tools/gather_probe.py > $OUT/probe.jsonl 2> $OUT/probe.err
timeout 600 ncu --set full --clock-control none -k regex:k_grouped_gemm_pair -c 2 -o $OUT/gemm_copy python tools/gather_probe.py --only copy > $OUT/ncu_copy.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_grouped_gemm_pair -c 2 -o $OUT/gemm_gather python tools/gather_probe.py --only gather > $OUT/ncu_gather.log 2>&1
echo done
