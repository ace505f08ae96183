#!/bin/bash
set -u
OUT=gpurun_out/r02f
mkdir -p $OUT
timeout 300 python tools/gather_probe.py > $OUT/probe.jsonl 2> $OUT/probe.err
timeout 300 python tools/gather_probe.py --bwd >> $OUT/probe.jsonl 2>> $OUT/probe.err
echo done
