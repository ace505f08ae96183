#!/bin/bash
set -u
OUT=gpurun_out/health
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "exit=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "exit=$?" >> $OUT/bench_n1.err
timeout 600 python tools/ffn_bench.py > $OUT/ffn.jsonl 2>&1
echo done
