#!/bin/bash
set -u
OUT=gpurun_out/r02e
mkdir -p $OUT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_grouped_gemm_pair -c 1 -o $OUT/gemm_gather_lsu python tools/gather_probe.py --only gather > $OUT/ncu_gather.log 2>&1
echo done
