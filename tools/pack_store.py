"""Pack kernel store-hint comparison on one GPU (Qwen3 shape, per-GPU dedup):
mean pack time (library CUDA events) for L1::no_allocate / .cs / default."""

import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2508_09591_b200 import _lib  # noqa: E402
from paper_2508_09591_b200.layer import EPWorld, route_topk  # noqa: E402

G, E, K, M, T_r = 8, 128, 8, 2048, 4096
g = torch.Generator(device="cuda").manual_seed(1)
logits = torch.randn(G * T_r, E, device="cuda", generator=g)
x = torch.randn(G * T_r, M, device="cuda", generator=g).to(torch.bfloat16)
slot, w, _ = route_topk(logits, K)
ep = EPWorld(G, E, K, M, T_r, n_cap_rows=3 * T_r * K)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
_lib.call("hm_world_set_timing", ep._h, 1)
for hint in (0, 1, 2, 0, 1, 2):
    _lib.call("hm_world_set_option", ep._h, 6, hint)
    acc = []
    for it in range(12):
        flush.zero_()
        ep.dispatch(x, slot, w, dedup="gpu")
        torch.cuda.synchronize()
        buf = (ctypes.c_float * 8)()
        _lib.call("hm_world_timings", ep._h, buf, 8)
        if it >= 2:
            acc.append(buf[2])
    print(json.dumps({"store_hint": hint, "pack_ms": round(float(np.mean(acc)), 4)}), flush=True)
ep.check_status()
