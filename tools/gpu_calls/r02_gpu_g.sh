#!/bin/bash
# full GPU suite (4 GPUs: multi-GPU parity) + N=1 bench after the option cleanup
set -u
OUT=gpurun_out/r02g
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "exit=$?" >> $OUT/smoke.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29631 bench.py --gpus 4 --steps 50 --warmup 5 > $OUT/bench_n4.json 2> $OUT/bench_n4.err; echo "exit=$?" >> $OUT/bench_n4.err
echo done
