#!/bin/bash
set -u
OUT=gpurun_out/r02c2
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29801 tests/mgpu_worker.py > $OUT/mgpu2.log 2>&1; echo "exit=$?" >> $OUT/mgpu2.log
timeout 600 $TR --nproc-per-node 4 --master-port 29802 tests/mgpu_worker.py > $OUT/mgpu4.log 2>&1; echo "exit=$?" >> $OUT/mgpu4.log
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29803 bench.py --gpus 2 --steps 30 --warmup 5 --no-planner > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "exit=$?" >> $OUT/bench_n2.err
timeout 900 $TR --nproc-per-node 4 --master-port 29804 bench.py --gpus 4 --steps 30 --warmup 5 --no-planner > $OUT/bench_n4.json 2> $OUT/bench_n4.err; echo "exit=$?" >> $OUT/bench_n4.err
echo done
