#!/bin/bash
# router top-K with the threshold pre-pass in 4-warp CTAs + modulo-free notify (w4) vs HEAD (base): the quad ==
# lane router test on both builds, interleaved N = 1 steps, ncu of the
# router kernel, then the GPU suite on pre
set -u
OUT=gpurun_out/route_w4
mkdir -p $OUT
for v in base w4; do
  HM_LIB=paper_2508_09591_b200/libhiermoe.$v.so timeout 600 python -m pytest tests/test_gpu_layer.py -q -p no:cacheprovider -k "route" > $OUT/route_tests_$v.log 2>&1; echo "exit=$?" >> $OUT/route_tests_$v.log
done
: > $OUT/ab.jsonl
for rep in 1 2 3; do
  for v in base w4; do
    echo "{\"variant\": \"$v\", \"rep\": $rep}" >> $OUT/ab.jsonl
    HM_LIB=paper_2508_09591_b200/libhiermoe.$v.so timeout 300 python tools/gather_ab.py >> $OUT/ab.jsonl 2>&1
  done
done
for v in base w4; do
  HM_LIB=paper_2508_09591_b200/libhiermoe.$v.so timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
    -k regex:"k_route_quad|k_notify" -c 20 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer > $OUT/ncu_$v.csv 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/gpu_tests.log
echo done
