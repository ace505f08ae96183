#!/bin/bash
# round-2 measurement pass (4 GPUs): benches N=1/2/4 (Qwen3), DSv3 N=1/4,
# N=1 ncu launch list + --set full of the step kernels, expert GEMM ncu
set -u
OUT=gpurun_out/r02m
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $OUT/gpus.csv
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "exit=$?" >> $OUT/bench_n1.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29661 bench.py --gpus 2 > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "exit=$?" >> $OUT/bench_n2.err
timeout 900 $TR --nproc-per-node 4 --master-port 29662 bench.py --gpus 4 > $OUT/bench_n4.json 2> $OUT/bench_n4.err; echo "exit=$?" >> $OUT/bench_n4.err
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py --config dsv3 --steps 50 > $OUT/bench_dsv3_n1.json 2> $OUT/bench_dsv3_n1.err; echo "exit=$?" >> $OUT/bench_dsv3_n1.err
timeout 1200 $TR --nproc-per-node 4 --master-port 29663 bench.py --gpus 4 --config dsv3 --steps 50 > $OUT/bench_dsv3_n4.json 2> $OUT/bench_dsv3_n4.err; echo "exit=$?" >> $OUT/bench_dsv3_n4.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-planner"
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/n1_launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "exit=$?" >> $OUT/ncu_launch.log
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_index_local|k_gather|k_plan|k_notify|k_route|k_pack_local" -s 30 -c 12 -o $OUT/n1_step $CMD --no-layer > $OUT/ncu_step.log 2>&1; echo "exit=$?" >> $OUT/ncu_step.log
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none -k regex:k_grouped_gemm -c 8 -o $OUT/ffn python tools/ffn_bench.py > $OUT/ncu_ffn.log 2>&1; echo "exit=$?" >> $OUT/ncu_ffn.log
echo done
