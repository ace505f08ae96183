#!/bin/bash
set -u
OUT=gpurun_out/r02d2
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fused_dispatch.py tests/test_gpu_moe_layer.py tests/test_gpu_backward.py -q -p no:cacheprovider -x > $OUT/t1.log 2>&1; echo "exit=$?" >> $OUT/t1.log
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29811 tests/mgpu_worker.py > $OUT/mgpu2.log 2>&1; echo "exit=$?" >> $OUT/mgpu2.log
timeout 600 $TR --nproc-per-node 4 --master-port 29812 tests/mgpu_worker.py > $OUT/mgpu4.log 2>&1; echo "exit=$?" >> $OUT/mgpu4.log
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29813 tools/overlap_probe.py --grad 1 > $OUT/ov_n2_g.jsonl 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29814 tools/overlap_probe.py --grad 1 > $OUT/ov_n4_g.jsonl 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29815 tools/overlap_probe.py > $OUT/ov_n2.jsonl 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29816 tools/overlap_probe.py > $OUT/ov_n4.jsonl 2>&1
echo done
