#!/bin/bash
# round-2 pass A (4 GPUs): full GPU suite (multi-GPU parity at N=4), runtime
# alpha/beta fits at N=2 and N=4, bench at N=1/2/4 (NCCL baseline at N>1)
set -u
OUT=gpurun_out/r02a
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi -L > $OUT/gpus.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/gpu_tests.log
mkdir -p paper_2508_09591_b200/params
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29611 tools/calibrate.py --runtime --out $OUT/b200_runtime_n2.json > $OUT/calib_n2.json 2> $OUT/calib_n2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29612 tools/calibrate.py --runtime --out $OUT/b200_runtime_n4.json > $OUT/calib_n4.json 2> $OUT/calib_n4.err
timeout 900 python bench.py --steps 50 --warmup 5 > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "exit=$?" >> $OUT/bench_n1.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29613 bench.py --gpus 2 --steps 50 --warmup 5 > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "exit=$?" >> $OUT/bench_n2.err
timeout 900 $TR --nproc-per-node 4 --master-port 29614 bench.py --gpus 4 --steps 50 --warmup 5 > $OUT/bench_n4.json 2> $OUT/bench_n4.err; echo "exit=$?" >> $OUT/bench_n4.err
echo done
