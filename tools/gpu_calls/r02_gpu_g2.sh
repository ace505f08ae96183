#!/bin/bash
set -u
OUT=gpurun_out/r02g2
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=29841
for rep in 1 2; do
for v in a b; do
  echo "{\"variant\": \"$v\"}" >> $OUT/ov.jsonl
  HM_LIB=paper_2508_09591_b200/libhiermoe.$v.so CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port $port tools/overlap_probe.py 2>/dev/null | grep "{" >> $OUT/ov.jsonl; port=$((port+1))
  HM_LIB=paper_2508_09591_b200/libhiermoe.$v.so timeout 600 $TR --nproc-per-node 4 --master-port $port tools/overlap_probe.py 2>/dev/null | grep "{" >> $OUT/ov.jsonl; port=$((port+1))
done
done
echo done
