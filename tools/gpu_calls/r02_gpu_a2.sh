#!/bin/bash
set -u
OUT=gpurun_out/r02a2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_moe_backward.py tests/test_gpu_fused_dispatch.py tests/test_gpu_ffn.py tests/test_gpu_moe_layer.py tests/test_gpu_migrate.py -q -p no:cacheprovider -x > $OUT/t1.log 2>&1; echo "exit=$?" >> $OUT/t1.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29771 tests/mgpu_worker.py > $OUT/mgpu2.log 2>&1; echo "exit=$?" >> $OUT/mgpu2.log
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29772 tools/layer_mb.py --mbs 1 > $OUT/layer_n2.jsonl 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29773 tools/layer_mb.py --mbs 1 > $OUT/layer_n4.jsonl 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/layer_mb.py --mbs 1 > $OUT/layer_n1.jsonl 2>&1
echo done
