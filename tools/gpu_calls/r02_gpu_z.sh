#!/bin/bash
set -u
OUT=gpurun_out/r02z
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29761 tests/mgpu_worker.py > $OUT/mgpu2.log 2>&1; echo "exit=$?" >> $OUT/mgpu2.log
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29762 tools/overlap_probe.py > $OUT/ov_n2.jsonl 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29763 tools/overlap_probe.py > $OUT/ov_n4.jsonl 2>&1
echo done
