#!/bin/bash
# layer fwd+bwd launch list at N = 1 (Qwen3 / DSv3) + PCIe copy rates
set -u
OUT=gpurun_out/layer
mkdir -p $OUT
timeout 300 python tools/pcie_probe.py > $OUT/pcie.jsonl 2>&1
timeout 300 python tools/profile_layer.py --steps 3 > $OUT/plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/layer_qwen3_launches.csv python tools/profile_layer.py --steps 3 > $OUT/ncu_q.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/layer_dsv3_launches.csv python tools/profile_layer.py --steps 2 --config dsv3 > $OUT/ncu_d.log 2>&1
echo done
# A/B: IEEE-division SiLU vs the MUFU reciprocal, interleaved on this box
bash tools/ab_probe.sh tools/ffn_bench.py ieee cur > /dev/null 2>&1
cp gpurun_out/ab/ab.jsonl $OUT/silu_ab.jsonl
