#!/bin/bash
set -u
OUT=gpurun_out/r02i2
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_ffn.py -q -x -p no:cacheprovider -k "wgrad_pair" > $OUT/t_pair.log 2>&1; echo "exit=$?" >> $OUT/t_pair.log
timeout 900 python -m pytest tests/test_gpu_ffn.py tests/test_gpu_moe_backward.py tests/test_gpu_fused_dispatch.py tests/test_gpu_backward.py tests/test_gpu_router.py -q -x -p no:cacheprovider > $OUT/t_all.log 2>&1; echo "exit=$?" >> $OUT/t_all.log
timeout 600 python tools/ffn_bench.py > $OUT/ffn_pair.jsonl 2>&1
timeout 600 python -c "
import sys; sys.argv=['x']
from paper_2508_09591_b200 import _lib
_lib.call('hm_ffn_set_option', 2, 0)
import runpy; runpy.run_path('tools/ffn_bench.py', run_name='__main__')
" > $OUT/ffn_single.jsonl 2>&1
echo done
