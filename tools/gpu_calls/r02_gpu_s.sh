#!/bin/bash
set -u
OUT=gpurun_out/r02s
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29711 tools/calibrate.py --runtime --out $OUT/b200_runtime_n2.json > $OUT/calib_n2.json 2> $OUT/calib_n2.err
timeout 900 $TR --nproc-per-node 4 --master-port 29712 tools/calibrate.py --runtime --out $OUT/b200_runtime_n4.json > $OUT/calib_n4.json 2> $OUT/calib_n4.err
cp $OUT/b200_runtime_n2.json $OUT/b200_runtime_n4.json paper_2508_09591_b200/params/
timeout 1500 $TR --nproc-per-node 4 --master-port 29713 tools/sweep.py --tokens 4096 16384 65536 > $OUT/sweep_n4.jsonl 2> $OUT/sweep_n4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 $TR --nproc-per-node 2 --master-port 29714 tools/sweep.py --tokens 4096 16384 > $OUT/sweep_n2.jsonl 2> $OUT/sweep_n2.err
echo done
