"""Layer forward / forward+backward time with 1, 2 and 4 micro-batches (one
EP world per micro-batch on its own stream: exchange overlapped with the
expert GEMMs).  torchrun for N > 1.

    torchrun --nproc-per-node N tools/layer_mb.py [--config qwen3|dsv3]
"""

import argparse
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2508_09591_b200.moe import HierMoELayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen3")
    ap.add_argument("--mbs", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--gemm-ctas", type=int, nargs="+", default=[0])
    ap.add_argument("--exch-blocks", type=int, nargs="+", default=[0])
    ap.add_argument("--gemm-pair", type=int, nargs="+", default=[1])
    ap.add_argument("--shared-overlap", type=int, nargs="+", default=[1])
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    if args.config == "qwen3":
        G, E, K, M, I, T_r = 8, 128, 8, 2048, 768, 4096
        kw = dict(optimizer_state=False)
    else:
        G, E, K, M, I, T_r = 8, 256, 8, 7168, 2048, 4096
        kw = dict(router="dsv3", n_group=8, topk_group=4, route_scale=2.5, shared_inter=2048,
                  optimizer_state=False)
    L = G // world
    gen = torch.Generator(device="cuda").manual_seed(5 + rank)
    x = torch.randn(L * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    g = torch.randn(L * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    from paper_2508_09591_b200.ffn import set_gemm_ctas
    for mb, ctas, xb, gp, so in [(m, c, b, p, o) for m in args.mbs for c in args.gemm_ctas
                                 for b in args.exch_blocks for p in args.gemm_pair
                                 for o in args.shared_overlap]:
        set_gemm_ctas(ctas)
        layer = HierMoELayer(G, E, K, M, I, T_r, gpus=world, gpu_index=rank, grad=True,
                             n_cap_rows=2 * T_r * K, micro_batches=mb, **kw)
        for wd in layer.worlds:
            wd.set_max_blocks(xb)
        layer.shared_overlap = bool(so)
        for _ in range(3):
            layer(x)
            layer.backward(g)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        tf = tb = 0.0
        for _ in range(args.steps):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            layer(x)
            e[1].record()
            layer.backward(g)
            e[2].record()
            e[2].synchronize()
            tf += e[0].elapsed_time(e[1])
            tb += e[1].elapsed_time(e[2])
        t = torch.tensor([tf / args.steps, tb / args.steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        for wd in layer.worlds:
            wd.check_status()
        # one forward with phase events (stream timeline, µs from the first mark)
        layer.timeline = []
        layer(x)
        torch.cuda.synchronize()
        t0 = layer.timeline[0][1]
        tl = {lab: round(t0.elapsed_time(ev) * 1e3, 1) for lab, ev in layer.timeline}
        layer.timeline = None
        if rank == 0:
            print(json.dumps({"timeline_us": tl}), flush=True)
        if rank == 0:
            print(json.dumps({"config": args.config, "n_gpus": world, "micro_batches": mb,
                              "gemm_ctas": ctas, "exch_blocks": xb, "gemm_pair": gp,
                              "shared_overlap": so,
                              "fwd_ms": round(t[0].item(), 4), "bwd_ms": round(t[1].item(), 4),
                              "fwd_bwd_ms": round(t[0].item() + t[1].item(), 4)}), flush=True)
        layer.close()
        del layer
        torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
