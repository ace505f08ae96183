"""Data-gradient GEMMs of one Qwen3 / DSv3 EP rank with K-major transposed
weights (hm_grouped_gemm on W^T) vs the weights as stored, read MN-major
(hm_grouped_gemm_kn).  Checks equality and times both."""

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2508_09591_b200 import _lib  # noqa: E402
from paper_2508_09591_b200._lib import ptr, stream_ptr  # noqa: E402


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n


ONCE = "--once" in sys.argv     # one launch of each (for ncu), DSv3 gx only
for name, G, M, I, per in (("qwen3", 16, 2048, 768, 2048), ("dsv3", 32, 7168, 2048, 1024)):
    if ONCE and name != "dsv3":
        continue
    torch.manual_seed(0)
    n = torch.full((G,), per, dtype=torch.int32, device="cuda")
    rows = G * per
    for lab, K, N in (("dh=gy.w2", M, I), ("gx=dg13.w13", 2 * I, M)):
        if ONCE and lab[0] != "g":
            continue
        a = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(G, K, N, device="cuda") * K ** -0.5).to(torch.bfloat16)   # [g][K][N]
        wt = w.transpose(1, 2).contiguous()                                         # [g][N][K]
        o1 = torch.empty(rows, N, device="cuda", dtype=torch.bfloat16)
        o2 = torch.empty_like(o1)
        f1 = lambda: _lib.call("hm_grouped_gemm", ptr(a), rows, ptr(wt), G, ptr(n), N, K, 0,  # noqa: E731
                               ptr(o1), N, stream_ptr())
        f2 = lambda: _lib.call("hm_grouped_gemm_kn", ptr(a), rows, ptr(w), G, ptr(n), N, K,  # noqa: E731
                               ptr(o2), N, stream_ptr())
        if ONCE:
            f1(), f2()
            torch.cuda.synchronize()
            continue
        ms1, ms2 = t(f1), t(f2)
        fl = 2 * rows * N * K
        print(json.dumps({"shape": name, "gemm": lab, "kmajor_ms": round(ms1, 4),
                          "mn_major_ms": round(ms2, 4), "kmajor_tf": round(fl / ms1 / 1e9, 1),
                          "mn_major_tf": round(fl / ms2 / 1e9, 1),
                          "equal": bool(torch.equal(o1, o2))}), flush=True)
