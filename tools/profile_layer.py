"""Run a few forward+backward steps of the Qwen3-shaped HierMoELayer (for ncu
launch lists / captures).  python tools/profile_layer.py [--steps 3]"""

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2508_09591_b200.moe import HierMoELayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--no-backward", action="store_true")
    ap.add_argument("--config", default="qwen3", choices=["qwen3", "dsv3"])
    args = ap.parse_args()
    if args.config == "qwen3":
        G, E, K, M, I, T_r = 8, 128, 8, 2048, 768, args.tokens
        kw = {}
    else:
        G, E, K, M, I, T_r = 8, 256, 8, 7168, 2048, args.tokens
        kw = dict(router="dsv3", n_group=8, topk_group=4, route_scale=2.5, shared_inter=2048,
                  optimizer_state=False)
    layer = HierMoELayer(G, E, K, M, I, T_r, dedup=True, grad=not args.no_backward,
                         n_cap_rows=2 * T_r * K, **kw)
    x = torch.randn(G * T_r, M, device="cuda").to(torch.bfloat16)
    g = torch.randn(G * T_r, M, device="cuda").to(torch.bfloat16)
    for _ in range(args.steps):
        layer(x)
        if not args.no_backward:
            layer.backward(g)
    torch.cuda.synchronize()
    layer.world.check_status()
    print("ok")


if __name__ == "__main__":
    main()
