#!/bin/bash
# round-2 final measurement pass: GPU suite (4 GPUs: multi-GPU parity
# included), smoke, bench N = 1 / 2 / 4 (Qwen3) and N = 1 / 4 (DSv3), the
# reference arm, and the FFN bench
set -u
OUT=${OUT:-gpurun_out/final}
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "exit=$?" >> $OUT/smoke.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err; echo "exit=$?" >> $OUT/bench_n1.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29791 bench.py --gpus 2 --steps 30 --warmup 5 > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "exit=$?" >> $OUT/bench_n2.err
timeout 900 $TR --nproc-per-node 4 --master-port 29792 bench.py --gpus 4 --steps 30 --warmup 5 > $OUT/bench_n4.json 2> $OUT/bench_n4.err; echo "exit=$?" >> $OUT/bench_n4.err
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py --config dsv3 --steps 20 --warmup 3 > $OUT/bench_dsv3_n1.json 2> $OUT/bench_dsv3_n1.err; echo "exit=$?" >> $OUT/bench_dsv3_n1.err
timeout 1200 $TR --nproc-per-node 4 --master-port 29793 bench.py --gpus 4 --config dsv3 --steps 20 --warmup 3 > $OUT/bench_dsv3_n4.json 2> $OUT/bench_dsv3_n4.err; echo "exit=$?" >> $OUT/bench_dsv3_n4.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference > $OUT/ref_n1.json 2> $OUT/ref_n1.err; echo "exit=$?" >> $OUT/ref_n1.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/ffn_bench.py > $OUT/ffn.jsonl 2>&1
# launch list of the N = 1 bench command (short run; its numbers are not bench values)
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/bench_n1_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  --no-e2e --no-planner --no-hd2 > $OUT/bench_n1_ncu.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/layer_qwen3_launches.csv python tools/profile_layer.py --steps 3 > $OUT/layer_ncu.log 2>&1
echo done
