#!/bin/bash
# ncu --set full of the shipped expert GEMMs at one Qwen3 rank (tools/gemm_probe.py --once):
# GEMM1 (SwiGLU), GEMM2, GEMM1 + GEMM2 of the saving forward, gX (MN-major B)
set -u
OUT=gpurun_out/gemm_ncu
mkdir -p $OUT
timeout 300 python tools/gemm_probe.py --once > $OUT/once.log 2>&1 || { echo "probe failed"; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_grouped_gemm_pair -c 5 \
  -o $OUT/gemm_shipped -f python tools/gemm_probe.py --once > $OUT/ncu.log 2>&1
echo done
