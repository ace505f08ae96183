#!/bin/bash
# 256 x 512 vs 256 x 256 pair tiles: bit-exactness tests, per-GEMM timing, FFN fwd/bwd
set -u
OUT=gpurun_out/wide
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_ffn.py -q -x -p no:cacheprovider > $OUT/tests.log 2>&1; echo "exit=$?" >> $OUT/tests.log
timeout 600 python tools/gemm_probe.py --wide=0,2 > $OUT/gemm_probe.jsonl 2>&1
# wide 1 = the shipped policy
for w in 0 1 0 1; do HM_WIDE=$w timeout 300 python tools/ffn_bench.py | sed "s/^{/{\"wide\": $w, /" >> $OUT/ffn.jsonl 2>&1; done
echo done
