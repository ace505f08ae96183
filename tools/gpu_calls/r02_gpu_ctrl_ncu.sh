#!/bin/bash
# ncu --set full of the N = 1 dispatch's short kernels (route, plan, notify,
# index) from the bench command: where their latency goes
set -u
OUT=gpurun_out/ctrl_ncu
mkdir -p $OUT
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_notify|k_plan|k_route_quad|k_index_local" -s 40 -c 4 -o $OUT/ctrl \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer > $OUT/ncu.log 2>&1
echo done
