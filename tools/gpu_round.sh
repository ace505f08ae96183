#!/bin/bash
# one GPU verification pass: tests, smoke, bench, launch list, ncu capture
set -u
OUT=gpurun_out
TAG=${1:-r}
lscpu | grep -E "Model name|Flags" | sed 's/Flags:.*avx512f.*/Flags: avx512f present/' > $OUT/${TAG}_host.txt
python -c "from numpy._core._multiarray_umath import __cpu_features__ as f; print('AVX512_SKX', f.get('AVX512_SKX'))" >> $OUT/${TAG}_host.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/${TAG}_gpu_tests.log 2>&1; echo "exit=$?" >> $OUT/${TAG}_gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "exit=$?" >> $OUT/${TAG}_smoke.log
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "exit=$?" >> $OUT/${TAG}_bench.err
if [ "${2:-}" = "ncu" ]; then
  CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-layer --no-planner"
  timeout 300 $CMD > $OUT/${TAG}_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $CMD > $OUT/${TAG}_ncu1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pack|k_gather|k_plan|k_notify|k_route" -s 20 -c 10 -o $OUT/${TAG}_prof $CMD > $OUT/${TAG}_ncu2.log 2>&1
  echo "ncu exit=$?" >> $OUT/${TAG}_ncu2.log
fi
