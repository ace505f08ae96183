"""Grouped-GEMM timing of one EP rank's expert FFN pieces (ragged groups like
tools/ffn_bench.py): GEMM1 (SwiGLU), GEMM2, the saving forward, and the
data-gradient GEMM.  Used with HM_LIB for A/B builds (tools/ab_probe.sh)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_09591_b200 import _lib  # noqa: E402
from paper_2508_09591_b200.ffn import expert_ffn_save_ptrs  # noqa: E402


ONCE = "--once" in sys.argv     # one launch of each, Qwen3 only (for ncu)
GRIDS = [int(a.split("=")[1]) for a in sys.argv if a.startswith("--grid=")] or [0]
# --wide=0,2: hm_ffn_set_option(5, w) per run (256 x 256 vs 256 x 512 tiles), interleaved
WIDE = [int(w) for a in sys.argv if a.startswith("--wide=") for w in a.split("=")[1].split(",")] or [1]
# --tma=0,1: hm_ffn_set_option(6, t) (LSU vs TMA epilogue stores), interleaved
TMA = [int(w) for a in sys.argv if a.startswith("--tma=") for w in a.split("=")[1].split(",")] or [1]
REPS = 2 if len(WIDE) > 1 or len(TMA) > 1 else 1


def t(fn, n=20):
    if ONCE:
        fn()
        torch.cuda.synchronize()
        return 1.0
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


for name, G, M, I, per in (("qwen3", 16, 2048, 768, 2048), ("dsv3", 32, 7168, 2048, 1024)):
    if ONCE and name != "qwen3":
        continue
    torch.manual_seed(0)
    n = torch.full((G,), per) + torch.randint(-per // 8, per // 8 + 1, (G,))
    rows = int(n.sum())
    cap = rows + 256
    nr = n.to(torch.int32).cuda()
    x = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    h = torch.empty(cap, I, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(cap, M, device="cuda", dtype=torch.bfloat16)
    g13 = torch.empty(cap, 2 * I, device="cuda", dtype=torch.bfloat16)
    st = _lib.stream_ptr()
    for grid, wide, tma in [(g, w, t) for _ in range(REPS) for g in GRIDS for w in WIDE
                            for t in TMA]:
        _lib.call("hm_ffn_set_option", 1, grid)
        _lib.call("hm_ffn_set_option", 5, wide)
        _lib.call("hm_ffn_set_option", 6, tma)
        g1 = t(lambda: _lib.call("hm_grouped_gemm", x.data_ptr(), cap, w13.data_ptr(), G,
                                 nr.data_ptr(), 2 * I, M, 1, h.data_ptr(), I, st))
        g2 = t(lambda: _lib.call("hm_grouped_gemm", h.data_ptr(), cap, w2.data_ptr(), G,
                                 nr.data_ptr(), M, I, 0, y.data_ptr(), M, st))
        fs = t(lambda: expert_ffn_save_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h,
                                            y.data_ptr(), g13.data_ptr()))
        gx = t(lambda: _lib.call("hm_grouped_gemm_kn", g13.data_ptr(), cap, w13.data_ptr(), G,
                                 nr.data_ptr(), M, 2 * I, y.data_ptr(), M, st))
        f1, f2 = 2 * rows * 2 * I * M, 2 * rows * M * I
        print(json.dumps({"shape": name, "rows": rows, "grid": grid, "wide": wide, "tma": tma,
                          "gemm1_ms": round(g1, 4), "gemm1_tf": round(f1 / g1 / 1e9, 1),
                          "gemm2_ms": round(g2, 4), "gemm2_tf": round(f2 / g2 / 1e9, 1),
                          "fwd_save_ms": round(fs, 4),
                          "fwd_save_tf": round((f1 + f2) / fs / 1e9, 1),
                          "dgrad_x_ms": round(gx, 4), "dgrad_x_tf": round(f1 / gx / 1e9, 1)}),
              flush=True)
    _lib.call("hm_ffn_set_option", 1, 0)
