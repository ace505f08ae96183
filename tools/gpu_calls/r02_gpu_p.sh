#!/bin/bash
set -u
OUT=gpurun_out/r02p
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29681 tools/layer_mb.py --mbs 1 2 4 > $OUT/mb_n2.jsonl 2> $OUT/mb_n2.err
timeout 900 $TR --nproc-per-node 4 --master-port 29682 tools/layer_mb.py --mbs 1 2 4 --gemm-ctas 0 128 > $OUT/mb_n4.jsonl 2> $OUT/mb_n4.err
echo done
