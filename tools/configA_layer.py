"""the CPU restatement of dispatch -> FFN -> combine for config A
(topology [8], E = 16, top-2, hidden 256, I = 512, 512 tokens per rank = 4096
tokens) timed on the host cores beside the same layer forward on one B200
(HierMoELayer: our router GEMM + top-K, fused dispatch, tcgen05 SwiGLU experts,
combine).  The CPU side is torch (fp32 math on the layer's bf16 weights,
every host thread, best of 5 after a warm-up); outputs are compared at the
bf16 tolerance.  python tools/configA_layer.py"""

import json
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2508_09591_b200.moe import HierMoELayer  # noqa: E402

G, E, K, M, I, T_R = 8, 16, 2, 256, 512, 512


def cpu_layer(x, wr, w13, w2):
    """softmax top-K router -> per-expert SwiGLU -> gate-weighted sum (fp32)."""
    logits = x @ wr.T
    top, ids = torch.topk(logits, K, dim=1)
    gates = torch.softmax(top, dim=1)
    out = torch.zeros_like(x)
    nb = I // 128
    for e in range(E):
        tok, kk = torch.nonzero(ids == e, as_tuple=True)
        if tok.numel() == 0:
            continue
        xe = x[tok]
        w = w13[e].view(nb, 2, 128, M)
        g = xe @ w[:, 0].reshape(I, M).T
        u = xe @ w[:, 1].reshape(I, M).T
        y = (torch.nn.functional.silu(g) * u) @ w2[e].T
        out.index_add_(0, tok, gates[tok, kk][:, None] * y)
    return out


def main():
    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    layer = HierMoELayer(G, E, K, M, I, T_R, seed=11)
    gen = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randn(G * T_R, M, device="cuda", generator=gen).to(torch.bfloat16)
    for _ in range(5):
        y = layer(x)
    torch.cuda.synchronize()
    steps = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        y = layer(x)
    e1.record()
    e1.synchronize()
    gpu_ms = e0.elapsed_time(e1) / steps
    xc = x.float().cpu()
    wr = layer.w_router.to(torch.bfloat16).float().cpu()
    w13 = layer.w13.reshape(E, 2 * I, M).float().cpu()
    w2 = layer.w2.reshape(E, M, I).float().cpu()
    ref = cpu_layer(xc, wr, w13, w2)
    times = []
    for i in range(6):
        t0 = time.perf_counter()
        cpu_layer(xc, wr, w13, w2)
        if i:
            times.append(time.perf_counter() - t0)
    cpu_ms = min(times) * 1e3
    err = ((y.float().cpu() - ref).abs().max() / ref.abs().max()).item()
    t = G * T_R
    print(json.dumps({"config": "A", "tokens": t, "gpu_ms": round(gpu_ms, 4),
                      "gpu_tokens_per_s": t / gpu_ms * 1e3, "cpu_ms": round(cpu_ms, 3),
                      "cpu_tokens_per_s": t / cpu_ms * 1e3, "cpu_cores": cores,
                      "max_rel_err_vs_cpu": err, "tolerance": 2e-2,
                      "within_tolerance": err < 2e-2}))
    layer.close()


if __name__ == "__main__":
    main()
