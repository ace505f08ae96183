#!/bin/bash
# Multi-GPU verification + measurements on all visible GPUs (gpurun --gpus N)
set -u
OUT=gpurun_out
N=$(python -c "import torch; print(torch.cuda.device_count())")
TAG=${1:-m}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > $OUT/${TAG}_n${N}_tests.log 2>&1; echo "exit=$?" >> $OUT/${TAG}_n${N}_tests.log
timeout 600 $TR --master-port 29601 bench.py --gpus $N > $OUT/${TAG}_n${N}_bench.json 2> $OUT/${TAG}_n${N}_bench.err; echo "exit=$?" >> $OUT/${TAG}_n${N}_bench.err
timeout 600 $TR --master-port 29602 tools/calibrate.py --out $OUT/${TAG}_params_b200_n${N}.json > $OUT/${TAG}_n${N}_calib.json 2> $OUT/${TAG}_n${N}_calib.err
timeout 600 $TR --master-port 29603 tools/swap_stress.py > $OUT/${TAG}_n${N}_swap.json 2> $OUT/${TAG}_n${N}_swap.err
if [ "${2:-}" = "sweep" ]; then
  timeout 1200 $TR --master-port 29604 tools/sweep.py > $OUT/${TAG}_n${N}_sweep.jsonl 2> $OUT/${TAG}_n${N}_sweep.err
fi
echo done
