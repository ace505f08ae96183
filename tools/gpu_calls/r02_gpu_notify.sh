#!/bin/bash
# chunk prefix moved into k_plan's last CTA (k_notify = barrier + derived
# offsets): GPU suite on 4 GPUs (multi-GPU count exchange), bench N = 1 (x2),
# N = 2 / 4, launch list of the N = 1 bench command
set -u
OUT=gpurun_out/notify
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/gpu_tests.log
for i in 1 2; do
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer > $OUT/bench_n1_$i.json 2> $OUT/bench_n1_$i.err
done
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29721 bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer > $OUT/bench_n2.json 2> $OUT/bench_n2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29722 bench.py --gpus 4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-planner --no-hd2 --no-layer > $OUT/bench_n4.json 2> $OUT/bench_n4.err
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/bench_n1_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  --no-e2e --no-planner --no-hd2 --no-layer > $OUT/ncu.log 2>&1
echo done
