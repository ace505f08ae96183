"""Layer forward (+ backward with --grad 1) with the exchange overlaps on vs
off: the dispatch inside the expert GEMM at N > 1 (hm_experts_overlap) and
the dispatch backward beside the weight-gradient GEMMs; per-phase device
times (world segment events, rank 0) and fwd / bwd times, max over ranks.

    torchrun --nproc-per-node N tools/overlap_probe.py [--config qwen3|dsv3] [--grad 1]
"""

import argparse
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2508_09591_b200 import _lib  # noqa: E402
from paper_2508_09591_b200.moe import HierMoELayer  # noqa: E402

SEGS = ["plan", "notify", "pack", "barrier1", "expand", "reduce", "barrier2", "gather",
        "ffn_local_push", "ffn_rest"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen3")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--grad", type=int, default=0)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl",
                                device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    else:   # one GPU: no collectives to run
        dist.barrier = lambda: None
        dist.all_reduce = lambda t, op=None: None
    if args.config == "qwen3":
        G, E, K, M, I, T_r = 8, 128, 8, 2048, 768, 4096
        kw = {}
    else:
        G, E, K, M, I, T_r = 8, 256, 8, 7168, 2048, 4096
        kw = dict(router="dsv3", n_group=8, topk_group=4, route_scale=2.5, shared_inter=2048)
    L = G // world
    gen = torch.Generator(device="cuda").manual_seed(5 + rank)
    x = torch.randn(L * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    g = torch.randn(L * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    for overlap in (False, True, False, True):
        layer = HierMoELayer(G, E, K, M, I, T_r, gpus=world, gpu_index=rank, dedup="gpu",
                             grad=bool(args.grad), n_cap_rows=2 * T_r * K, optimizer_state=False,
                             overlap=overlap, **kw)
        layer.bwd_overlap = overlap
        for _ in range(3):
            layer(x)
            if args.grad:
                layer.backward(g)
        torch.cuda.synchronize()
        dist.barrier()
        tf = tb = 0.0
        for _ in range(args.steps):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            layer(x)
            e[1].record()
            if args.grad:
                layer.backward(g)
            e[2].record()
            e[2].synchronize()
            tf += e[0].elapsed_time(e[1])
            tb += e[1].elapsed_time(e[2])
        t = torch.tensor([tf / args.steps, tb / args.steps], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wd = layer.worlds[0]
        _lib.call("hm_world_set_timing", wd._h, 1)
        layer(x)
        torch.cuda.synchronize()
        buf = (_lib.c_float * len(SEGS))()
        _lib.call("hm_world_timings", wd._h, buf, len(SEGS))
        _lib.call("hm_world_set_timing", wd._h, 0)
        seg = {k: round(v * 1e3, 1) for k, v in zip(SEGS, list(buf)) if v >= 0}
        if rank == 0:
            print(json.dumps({"config": args.config, "n_gpus": world, "overlap": overlap,
                              "grad": args.grad, "fwd_ms": round(t[0].item(), 4),
                              "bwd_ms": round(t[1].item(), 4),
                              "segments_us_rank0": seg}), flush=True)
        layer.close()
        del layer
        torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
