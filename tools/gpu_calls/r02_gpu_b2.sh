#!/bin/bash
set -u
OUT=gpurun_out/r02b2
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/overlap_probe.py --grad 1 > $OUT/ov_n1.jsonl 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29781 tools/overlap_probe.py --grad 1 > $OUT/ov_n2.jsonl 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29782 tools/overlap_probe.py --grad 1 > $OUT/ov_n4.jsonl 2>&1
echo done
