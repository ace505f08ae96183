#!/bin/bash
# ncu --set full of GEMM1 (SwiGLU) on 256 x 256 and 256 x 512 pair tiles (one Qwen3 rank)
set -u
OUT=gpurun_out/wide
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_ffn.py -q -x -p no:cacheprovider > $OUT/tests.log 2>&1; echo "exit=$?" >> $OUT/tests.log
for w in 0 1; do
  timeout 300 python tools/gemm_probe.py --once --wide=$w > $OUT/once_$w.log 2>&1 || { echo "probe failed"; exit 1; }
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_grouped_gemm_pair -c 2 \
    -o $OUT/gemm_wide$w -f python tools/gemm_probe.py --once --wide=$w > $OUT/ncu_$w.log 2>&1
done
echo done
