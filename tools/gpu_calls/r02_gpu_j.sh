#!/bin/bash
set -u
OUT=gpurun_out/r02j
mkdir -p $OUT
timeout 300 python tools/ffn_bench.py > $OUT/ffn.jsonl 2> $OUT/ffn.err
timeout 600 ncu --set full --clock-control none -k regex:k_grouped_gemm -c 12 -o $OUT/ffn_dsv3 python tools/ffn_bench.py > $OUT/ncu.log 2>&1
echo done
