#!/bin/bash
# round-2 pass B (1 GPU): fused dispatch (TMA gather4 GEMM) parity + bench
set -u
OUT=gpurun_out/r02b
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fused_dispatch.py tests/test_gpu_moe_backward.py tests/test_gpu_moe_layer.py tests/test_gpu_ffn.py -q -p no:cacheprovider -x > $OUT/tests.log 2>&1; echo "exit=$?" >> $OUT/tests.log
timeout 900 python bench.py --steps 50 --warmup 5 --no-planner > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "exit=$?" >> $OUT/bench_n1.err
echo done
