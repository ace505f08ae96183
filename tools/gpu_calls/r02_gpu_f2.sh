#!/bin/bash
set -u
OUT=gpurun_out/r02f2
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29831 tests/mgpu_worker.py > $OUT/mgpu2.log 2>&1; echo "exit=$?" >> $OUT/mgpu2.log
timeout 600 $TR --nproc-per-node 4 --master-port 29832 tests/mgpu_worker.py > $OUT/mgpu4.log 2>&1; echo "exit=$?" >> $OUT/mgpu4.log
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29833 tools/overlap_probe.py --grad 1 > $OUT/ov_n2_g.jsonl 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29834 tools/overlap_probe.py --grad 1 > $OUT/ov_n4_g.jsonl 2>&1
echo done
