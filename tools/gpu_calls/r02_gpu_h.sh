#!/bin/bash
# counters + sanitizers (2 GPUs): NVML NVLink bytes at N=2, ncu tensor-pipe on
# the expert GEMMs, compute-sanitizer memcheck / racecheck on dispatch+combine
set -u
OUT=gpurun_out/r02h
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29641 tools/nvlink_counters.py > $OUT/nvlink_n2.json 2> $OUT/nvlink_n2.err
SEL='configA_bf16 or ragged_tokens or qwen3_small'
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_layer.py -q -p no:cacheprovider -k "$SEL" > $OUT/memcheck.log 2>&1; echo "exit=$?" >> $OUT/memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_layer.py -q -p no:cacheprovider -k "configA_bf16 and gpu" > $OUT/racecheck.log 2>&1; echo "exit=$?" >> $OUT/racecheck.log
timeout 900 ncu --set full --clock-control none -k regex:k_grouped_gemm -c 6 -o $OUT/ffn python tools/ffn_bench.py > $OUT/ncu_ffn.log 2>&1; echo "exit=$?" >> $OUT/ncu_ffn.log
echo done
