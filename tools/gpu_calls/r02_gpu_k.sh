#!/bin/bash
set -u
OUT=gpurun_out/r02k
mkdir -p $OUT
timeout 300 python tools/gemm_probe.py > $OUT/gemm.jsonl 2>&1
timeout 300 python tools/ffn_bench.py > $OUT/ffn.jsonl 2> $OUT/ffn.err
timeout 300 python tools/gather_probe.py > $OUT/probe.jsonl 2> $OUT/probe.err
timeout 900 python -m pytest tests/test_gpu_gemm_pair.py tests/test_gpu_ffn.py tests/test_gpu_fused_dispatch.py tests/test_gpu_moe_backward.py tests/test_gpu_moe_layer.py -q -p no:cacheprovider -x > $OUT/tests.log 2>&1; echo "exit=$?" >> $OUT/tests.log
echo done
