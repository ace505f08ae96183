#!/bin/bash
set -u
OUT=gpurun_out/r02d
mkdir -p $OUT
timeout 300 python tools/gather_probe.py > $OUT/probe.jsonl 2> $OUT/probe.err
timeout 900 python -m pytest tests/test_gpu_fused_dispatch.py tests/test_gpu_moe_backward.py tests/test_gpu_moe_layer.py tests/test_gpu_ffn.py tests/test_gpu_gemm_pair.py -q -p no:cacheprovider -x > $OUT/tests.log 2>&1; echo "exit=$?" >> $OUT/tests.log
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_fused_dispatch.py -q -p no:cacheprovider -x >> $OUT/tests_repeat.log 2>&1; echo "exit=$?" >> $OUT/tests_repeat.log; done
timeout 900 python bench.py --steps 50 --warmup 5 --no-planner --no-cpu-baseline > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "exit=$?" >> $OUT/bench_n1.err
echo done
