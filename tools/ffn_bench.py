"""Expert FFN forward (with saved pre-activations) and backward throughput on
one GPU for the Qwen3 / DeepSeek-V3 expert shapes, uniform ragged groups
(the rows one EP rank receives).  python tools/ffn_bench.py"""

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2508_09591_b200.ffn import (FFNBackwardScratch, expert_ffn_backward_ptrs,  # noqa: E402
                                       expert_ffn_save_ptrs)


def run(name, G, M, I, rows_per_group, steps=10):
    torch.manual_seed(0)
    n = (torch.full((G,), rows_per_group) + torch.randint(-rows_per_group // 8,
                                                           rows_per_group // 8 + 1, (G,)))
    rows = int(n.sum())
    cap = rows + 256
    nr = n.to(torch.int32).cuda()
    x = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    gy = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    h = torch.empty(cap, I, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(cap, M, device="cuda", dtype=torch.bfloat16)
    g13 = torch.empty(cap, 2 * I, device="cuda", dtype=torch.bfloat16)
    sc = FFNBackwardScratch(cap, G, M, I)
    gx = torch.empty(cap, M, device="cuda", dtype=torch.bfloat16)
    dw13, dw2 = torch.empty_like(w13), torch.empty_like(w2)

    def fwd():
        expert_ffn_save_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h, y.data_ptr(),
                             g13.data_ptr())

    def bwd():
        expert_ffn_backward_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2,
                                 gy.data_ptr(), M, I, sc, gx.data_ptr(), dw13, dw2,
                                 g13.data_ptr())

    res = {"name": name, "groups": G, "hidden": M, "inter": I, "rows": rows}
    for label, fn, fl in (("fwd", fwd, 6), ("bwd", bwd, 12)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
        res[f"{label}_ms"] = round(ms, 4)
        res[f"{label}_tflops"] = round(fl * rows * M * I / (ms * 1e-3) / 1e12, 1)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    import os
    from paper_2508_09591_b200 import _lib
    if "HM_WIDE" in os.environ:   # hm_ffn_set_option(5, .): 256 x 512 tiles
        _lib.call("hm_ffn_set_option", 5, int(os.environ["HM_WIDE"]))
    if "HM_TMA_STORE" in os.environ:   # hm_ffn_set_option(6, .): TMA epilogue stores
        _lib.call("hm_ffn_set_option", 6, int(os.environ["HM_TMA_STORE"]))
    run("qwen3_rank", 16, 2048, 768, 2048)
    run("dsv3_rank", 32, 7168, 2048, 1024)
