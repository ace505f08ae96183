#!/bin/bash
set -u
OUT=gpurun_out/r02r
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $TR --nproc-per-node 4 --master-port 29701 tools/sweep.py --tokens 4096 16384 65536 > $OUT/sweep_n4.jsonl 2> $OUT/sweep_n4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 $TR --nproc-per-node 2 --master-port 29702 tools/sweep.py --tokens 4096 16384 > $OUT/sweep_n2.jsonl 2> $OUT/sweep_n2.err
timeout 1500 $TR --nproc-per-node 4 --master-port 29703 tools/swap_demo.py --steps 150 > $OUT/swap_demo_n4.json 2> $OUT/swap_demo_n4.err
echo done
