#!/bin/bash
set -u
OUT=gpurun_out/r02v
mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_grouped_gemm -o $OUT/gemm_src python tools/gemm_probe.py --once > $OUT/ncu.log 2>&1
echo done
