#!/bin/bash
# TMA tensor-store epilogue vs LSU stores: bit-exactness tests, per-GEMM timing, FFN fwd/bwd
set -u
OUT=gpurun_out/tma
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_ffn.py -q -x -p no:cacheprovider > $OUT/tests.log 2>&1; echo "exit=$?" >> $OUT/tests.log
timeout 600 python tools/gemm_probe.py --tma=0,1 > $OUT/gemm_probe.jsonl 2>&1
for t in 0 1 0 1; do HM_TMA_STORE=$t timeout 300 python tools/ffn_bench.py | sed "s/^{/{\"tma\": $t, /" >> $OUT/ffn.jsonl 2>&1; done
echo done
