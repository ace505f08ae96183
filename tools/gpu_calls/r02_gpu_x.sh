#!/bin/bash
set -u
OUT=gpurun_out/r02x
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_moe_backward.py tests/test_gpu_fused_dispatch.py tests/test_gpu_ffn.py tests/test_gpu_moe_layer.py -q -p no:cacheprovider -x > $OUT/t1.log 2>&1; echo "exit=$?" >> $OUT/t1.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29741 tests/mgpu_worker.py > $OUT/mgpu2.log 2>&1; echo "exit=$?" >> $OUT/mgpu2.log
timeout 900 $TR --nproc-per-node 4 --master-port 29742 tests/mgpu_worker.py > $OUT/mgpu4.log 2>&1; echo "exit=$?" >> $OUT/mgpu4.log
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29743 tools/layer_mb.py --mbs 1 > $OUT/layer_n2.jsonl 2>&1
timeout 900 $TR --nproc-per-node 4 --master-port 29744 tools/layer_mb.py --mbs 1 > $OUT/layer_n4.jsonl 2>&1
echo done
