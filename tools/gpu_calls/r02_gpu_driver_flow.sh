#!/bin/bash
# the driver's round-end flow on one GPU at HEAD: GPU suite, smoke, default
# bench and the reference arm, each with its wall-clock seconds
set -u
OUT=gpurun_out/driver_flow
mkdir -p $OUT
run() {   # name, command...
  local name=$1; shift
  local t0=$SECONDS
  "$@"
  local rc=$?
  echo "$name rc=$rc wall_s=$((SECONDS - t0))" >> $OUT/wall.txt
}
run tests bash -c "timeout 1200 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > $OUT/gpu_tests.log 2>&1"
run smoke bash -c "timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.log 2>&1"
run ref bash -c "timeout 900 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err"
run bench bash -c "timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err"
echo done
