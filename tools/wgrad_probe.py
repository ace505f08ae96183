"""Weight-gradient GEMMs of one expert-FFN backward at small ragged shapes
(crash / equality probe for kernel variants).  HM_LIB=... python tools/wgrad_probe.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_09591_b200.ffn import (FFNBackwardScratch, expert_ffn_backward_ptrs,  # noqa: E402
                                       expert_ffn_save_ptrs)

for sizes in ([128], [64, 128], [100], [300, 77]):
    torch.manual_seed(1)
    G, M, I = len(sizes), 512, 256
    n = torch.tensor(sizes, dtype=torch.int32)
    cap = int(n.sum()) + 64
    nr = n.cuda()
    x = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    gy = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    h = torch.zeros(cap, I, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(cap, M, dtype=torch.bfloat16, device="cuda")
    g13 = torch.zeros(cap, 2 * I, dtype=torch.bfloat16, device="cuda")
    expert_ffn_save_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h, y.data_ptr(),
                         g13.data_ptr())
    sc = FFNBackwardScratch(cap, G, M, I)
    gx = torch.zeros(cap, M, dtype=torch.bfloat16, device="cuda")
    dw13, dw2 = torch.zeros_like(w13), torch.zeros_like(w2)
    expert_ffn_backward_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, gy.data_ptr(), M, I,
                             sc, gx.data_ptr(), dw13, dw2, g13.data_ptr())
    torch.cuda.synchronize()
    # reference dW2 = gy^T h per group
    r0 = 0
    err = 0.0
    for gi, ne in enumerate(sizes):
        ref = gy[r0:r0 + ne].float().T @ sc.h[r0:r0 + ne].float()
        err = max(err, ((dw2[gi].float() - ref).abs().max() / (ref.abs().max() + 1e-6)).item())
        r0 += ne
    print(sizes, "ok", "dw2 rel err", round(err, 5), flush=True)
