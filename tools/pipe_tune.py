"""Pipelined per-GPU dedup exchange: dispatch+combine time (qwen3 layer shape,
EP = 8 on the launched GPUs) for the barrier-separated kernels and the
pipelined kernels over pusher shares and stage counts.  torchrun, N >= 2.

    torchrun --nproc-per-node 2 tools/pipe_tune.py
"""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2508_09591_b200 import _lib  # noqa: E402
from paper_2508_09591_b200.layer import EPWorld, route_topk  # noqa: E402


def main():
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    G, E, K, M, T_r = 8, 128, 8, 2048, int(os.environ.get("TOKENS", "4096"))
    L = G // world
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    logits = torch.randn(L * T_r, E, device="cuda", generator=g)
    x = torch.randn(L * T_r, M, device="cuda", generator=g).to(torch.bfloat16)
    slot, w, _ = route_topk(logits, K)
    ep = EPWorld(G, E, K, M, T_r, gpus=world, gpu_index=rank)
    out = torch.empty_like(x)
    ref = None

    def run(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        for _ in range(n):
            ep.dispatch(x, slot, w, dedup="gpu")
            ep.combine(slot, w, dedup="gpu", out=out)
        e1.record()
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / n], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def segs():
        import ctypes
        _lib.call("hm_world_set_timing", ep._h, 1)
        acc = np.zeros(8)
        for _ in range(5):
            ep.dispatch(x, slot, w, dedup="gpu")
            ep.combine(slot, w, dedup="gpu", out=out)
            torch.cuda.synchronize()
            buf = (ctypes.c_float * 8)()
            _lib.call("hm_world_timings", ep._h, buf, 8)
            acc += np.maximum(np.array(buf[:]), 0)
        _lib.call("hm_world_set_timing", ep._h, 0)
        return [round(v / 5 * 1e3, 1) for v in acc]

    cases = [(False, 50, 8)] + [(True, p, s) for s in (4, 8, 16, 32) for p in (25, 50, 75)]
    for pipelined, pct, stages in cases:
        ep.set_pipelined(pipelined, pct, stages)
        run(3)
        ms = run(20)
        sg = segs()
        ep.check_status()
        if ref is None:
            ref = out.clone()
        same = bool(torch.equal(out, ref))
        if rank == 0:
            print(json.dumps({"n_gpus": world, "pipelined": pipelined, "push_pct": pct,
                              "stages": stages, "ms": round(ms, 4), "seg_us": sg,
                              "bitwise_equal": same}), flush=True)
    ep.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
