#!/bin/bash
set -u
OUT=gpurun_out/r02u
mkdir -p $OUT
timeout 300 python tools/dgrad_probe.py > $OUT/dgrad.jsonl 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_grouped_gemm -o $OUT/dgrad python tools/dgrad_probe.py --once > $OUT/ncu.log 2>&1
echo done
