#!/bin/bash
set -u
OUT=gpurun_out/r02n
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/gpu_tests.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-planner --no-cpu-baseline --no-e2e > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "exit=$?" >> $OUT/bench_n1.err
timeout 600 python tools/ffn_bench.py > $OUT/ffn.jsonl 2>&1
echo done
