#!/bin/bash
set -u
OUT=gpurun_out/r02o
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/gpu_tests.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29671 bench.py --gpus 2 --steps 50 --warmup 5 > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "exit=$?" >> $OUT/bench_n2.err
timeout 900 $TR --nproc-per-node 4 --master-port 29672 bench.py --gpus 4 --steps 50 --warmup 5 > $OUT/bench_n4.json 2> $OUT/bench_n4.err; echo "exit=$?" >> $OUT/bench_n4.err
echo done
