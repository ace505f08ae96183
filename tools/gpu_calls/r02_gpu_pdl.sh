#!/bin/bash
# programmatic dependent launch A/B: GPU suite, then the N = 1 bench with and
# without the launch attribute (alternating, two runs each)
set -u
OUT=gpurun_out/pdl
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/gpu_tests.log
for i in 1 2; do
  timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer > $OUT/bench_pdl_$i.json 2> $OUT/bench_pdl_$i.err
  timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer --no-pdl > $OUT/bench_nopdl_$i.json 2> $OUT/bench_nopdl_$i.err
done
timeout 600 python bench.py --config dsv3 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer > $OUT/bench_dsv3_pdl.json 2> $OUT/bench_dsv3_pdl.err
timeout 600 python bench.py --config dsv3 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer --no-pdl > $OUT/bench_dsv3_nopdl.json 2> $OUT/bench_dsv3_nopdl.err
echo done
