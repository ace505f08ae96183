"""Layer forward at N > 1 with the dispatch inside the expert GEMM
(hm_experts_overlap) vs the serial path: per-phase device times (world
segment events) and the forward time, max over ranks.

    torchrun --nproc-per-node N tools/overlap_probe.py [--config qwen3|dsv3]
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
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    if args.config == "qwen3":
        G, E, K, M, I, T_r = 8, 128, 8, 2048, 768, 4096
        kw = {}
    else:
        G, E, K, M, I, T_r = 8, 256, 8, 7168, 2048, 4096
        kw = dict(router="dsv3", n_group=8, topk_group=4, route_scale=2.5, shared_inter=2048)
    L = G // world
    gen = torch.Generator(device="cuda").manual_seed(5 + rank)
    x = torch.randn(L * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    for overlap in (False, True, False, True):
        layer = HierMoELayer(G, E, K, M, I, T_r, gpus=world, gpu_index=rank, dedup="gpu",
                             grad=bool(args.grad), n_cap_rows=2 * T_r * K, optimizer_state=False,
                             overlap=overlap, **kw)
        for _ in range(3):
            layer(x)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            layer(x)
        e1.record()
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device="cuda")
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
                              "grad": args.grad, "fwd_ms": round(t.item(), 4),
                              "segments_us_rank0": seg}), flush=True)
        layer.close()
        del layer
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
