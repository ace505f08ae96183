#!/bin/bash
set -u
OUT=gpurun_out/r02i
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29651 tools/nvlink_counters.py > $OUT/nvlink_n2.json 2> $OUT/nvlink_n2.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/gather_probe.py > $OUT/probe.jsonl 2> $OUT/probe.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/ffn_bench.py > $OUT/ffn.jsonl 2> $OUT/ffn.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_gemm_pair.py tests/test_gpu_ffn.py tests/test_gpu_fused_dispatch.py -q -p no:cacheprovider -x > $OUT/tests.log 2>&1; echo "exit=$?" >> $OUT/tests.log
echo done
