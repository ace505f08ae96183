#!/bin/bash
set -u
OUT=gpurun_out/r02q
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29691 bench.py --gpus 4 --config qwen3_ep4 --steps 30 --warmup 3 > $OUT/bench_ep4_n4.json 2> $OUT/bench_ep4_n4.err; echo "exit=$?" >> $OUT/bench_ep4_n4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29692 bench.py --impl reference --gpus 4 --steps 20 --warmup 3 > $OUT/ref_n4.json 2> $OUT/ref_n4.err; echo "exit=$?" >> $OUT/ref_n4.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/ref_n1.json 2> $OUT/ref_n1.err; echo "exit=$?" >> $OUT/ref_n1.err
echo done
