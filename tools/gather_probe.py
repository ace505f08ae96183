"""GEMM1 of one Qwen3 EP rank (16 experts x ~2048 rows, hidden 2048, I = 768,
SwiGLU) with the rows copied expert-major vs gathered from the token-major x
by index (cp.async producer warps).  python tools/gather_probe.py [--only copy|gather]"""

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2508_09591_b200.ffn import expert_ffn_gather_ptrs, expert_ffn_ptrs  # noqa: E402


def main():
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    G, M, I, T = 16, 2048, 768, 32768
    torch.manual_seed(0)
    n = torch.full((G,), 2048, dtype=torch.int32)
    rows = int(n.sum())
    cap = rows + 256
    x = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    # each expert's rows: 2048 distinct tokens in ascending order (as the dispatch emits)
    idx = torch.cat([torch.sort(torch.randperm(T)[:2048])[0] for _ in range(G)]).to(torch.int32)
    idx = torch.cat([idx, torch.zeros(256, dtype=torch.int32)]).cuda()
    xm = x[idx.long()].contiguous()
    nr = n.cuda()
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    h = torch.empty(cap, I, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(cap, M, device="cuda", dtype=torch.bfloat16)
    runs = {"copy": lambda: expert_ffn_ptrs(xm.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I,
                                            h, y.data_ptr()),
            "gather": lambda: expert_ffn_gather_ptrs(x.data_ptr(), T, idx.data_ptr(), cap,
                                                     nr.data_ptr(), G, w13, w2, M, I, h,
                                                     y.data_ptr())}
    for name, fn in runs.items():
        if only and not name.startswith(only):
            continue
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"path": name, "ffn_fwd_ms": round(ms, 4),
                          "tflops": round(6 * rows * M * I / (ms * 1e-3) / 1e12, 1)}), flush=True)


def backward():
    """FFN backward of the same rank: dW13's token operand gathered (fused)
    vs read from the materialised rows."""
    from paper_2508_09591_b200.ffn import (FFNBackwardScratch, expert_ffn_backward_gather_ptrs,
                                           expert_ffn_backward_ptrs, expert_ffn_save_ptrs)
    G, M, I, T = 16, 2048, 768, 32768
    torch.manual_seed(1)
    n = torch.full((G,), 2048, dtype=torch.int32)
    rows = int(n.sum())
    cap = rows + 256
    x = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    idx = torch.cat([torch.sort(torch.randperm(T)[:2048])[0] for _ in range(G)]).to(torch.int32)
    idx = torch.cat([idx, torch.zeros(256, dtype=torch.int32)]).cuda()
    xm = x[idx.long()].contiguous()
    nr = n.cuda()
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    h = torch.empty(cap, I, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(cap, M, device="cuda", dtype=torch.bfloat16)
    g13 = torch.empty(cap, 2 * I, device="cuda", dtype=torch.bfloat16)
    gy = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    sc = FFNBackwardScratch(cap, G, M, I)
    gx = torch.empty(cap, M, device="cuda", dtype=torch.bfloat16)
    dw13, dw2 = torch.empty_like(w13), torch.empty_like(w2)
    expert_ffn_save_ptrs(xm.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h, y.data_ptr(),
                         g13.data_ptr())
    runs = {"bwd_copy": lambda: expert_ffn_backward_ptrs(
                xm.data_ptr(), cap, nr.data_ptr(), G, w13, w2, gy.data_ptr(), M, I, sc,
                gx.data_ptr(), dw13, dw2, g13.data_ptr()),
            "bwd_gather": lambda: expert_ffn_backward_gather_ptrs(
                x.data_ptr(), T, idx.data_ptr(), cap, nr.data_ptr(), G, w13, w2, gy.data_ptr(),
                M, I, sc, gx.data_ptr(), dw13, dw2, g13.data_ptr())}
    outs = {}
    for name, fn in runs.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        outs[name] = dw13.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"path": name, "ffn_bwd_ms": round(ms, 4),
                          "tflops": round(12 * rows * M * I / (ms * 1e-3) / 1e12, 1)}), flush=True)
    print(json.dumps({"dw13_equal": bool(torch.equal(outs["bwd_copy"], outs["bwd_gather"]))}))


if __name__ == "__main__":
    if "--bwd" in sys.argv:
        backward()
        sys.exit(0)
    main()
