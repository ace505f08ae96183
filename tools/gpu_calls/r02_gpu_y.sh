#!/bin/bash
set -u
OUT=gpurun_out/r02y
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29751 tests/mgpu_worker.py > $OUT/mgpu2.log 2>&1; echo "exit=$?" >> $OUT/mgpu2.log
timeout 600 $TR --nproc-per-node 4 --master-port 29752 tests/mgpu_worker.py > $OUT/mgpu4.log 2>&1; echo "exit=$?" >> $OUT/mgpu4.log
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29753 tools/layer_mb.py --mbs 1 > $OUT/layer_n2.jsonl 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29754 tools/layer_mb.py --mbs 1 > $OUT/layer_n4.jsonl 2>&1
echo done
