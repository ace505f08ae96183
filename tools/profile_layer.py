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
    args = ap.parse_args()
    G, E, K, M, I, T_r = 8, 128, 8, 2048, 768, args.tokens
    layer = HierMoELayer(G, E, K, M, I, T_r, dedup=True, grad=not args.no_backward,
                         n_cap_rows=3 * T_r * K)
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
