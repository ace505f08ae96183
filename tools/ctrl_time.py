"""Control-path kernels of one dispatch+combine step (router, plan, notify)
timed warm in isolation on the Qwen3 N = 1 step (32768 tokens, E = 128, top-8).
Usage: python tools/ctrl_time.py [--reps 200]"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_09591_b200 import _lib                      # noqa: E402
from paper_2508_09591_b200.layer import EPWorld, route_topk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=200)
ap.add_argument("--tokens", type=int, default=32768)
args = ap.parse_args()
G, E, K, M = 8, 128, 8, 2048
T = args.tokens
lg = torch.randn(T, E, device="cuda")
x = torch.randn(T, M, device="cuda").to(torch.bfloat16)


def timeit(fn, reps=args.reps):
    """Device time per call: 20 calls captured in a CUDA graph, replayed (no
    host overhead in the number)."""
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(1, reps // 20)
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / (n * 20) * 1e3


res = {"tokens": T}
for mode, name in ((0, "lane"), (1, "quad")):
    _lib.call("hm_route_set_option", mode)
    res[f"route_{name}_us"] = timeit(lambda: route_topk(lg, K))
    res[f"route_{name}_full_softmax_us"] = timeit(lambda: route_topk(lg, K, renormalize=False))
_lib.call("hm_route_set_option", 1)
lg256 = torch.randn(T, 256, device="cuda")
res["route_default_E256_us"] = timeit(lambda: route_topk(lg256, K))
w = EPWorld(ranks=G, experts=E, top_k=K, hidden=M, tokens_per_rank=T // G, dtype=torch.bfloat16)
slot, wts, _ = route_topk(lg, K)
res["dispatch_combine_us"] = timeit(lambda: (w.dispatch(x, slot, wts, dedup="gpu"),
                                             w.combine(slot, wts, dedup="gpu")))
torch.cuda.synchronize()
w.check_status()
print(json.dumps(res))
w.close()
