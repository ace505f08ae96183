#!/bin/bash
# k_gather with the next token's pick metadata loaded one token ahead (pf)
# vs HEAD (base): interleaved N = 1 steps (3 reps), then the GPU suite on pf
set -u
OUT=gpurun_out/gather_pf
mkdir -p $OUT
: > $OUT/ab.jsonl
for rep in 1 2 3; do
  for v in base pf; do
    echo "{\"variant\": \"$v\", \"rep\": $rep}" >> $OUT/ab.jsonl
    HM_LIB=paper_2508_09591_b200/libhiermoe.$v.so timeout 300 python tools/gather_ab.py >> $OUT/ab.jsonl 2>&1
  done
done
HM_LIB=paper_2508_09591_b200/libhiermoe.base.so timeout 600 python bench.py --config dsv3 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer > $OUT/dsv3_base.json 2>&1
HM_LIB=paper_2508_09591_b200/libhiermoe.pf.so timeout 600 python bench.py --config dsv3 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer > $OUT/dsv3_pf.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/gpu_tests.log
echo done
