#!/bin/bash
set -u
OUT=gpurun_out/r02l
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/gpu_tests.log
timeout 900 python bench.py --steps 50 --warmup 5 --no-planner --no-cpu-baseline > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "exit=$?" >> $OUT/bench_n1.err
echo done
