"""Grid size of the exchange kernels on the Qwen3 step (EP = 8, 32768 tokens
over N GPUs): dispatch-only and combine-only device time per grid cap
(CUDA-graph replay, max over ranks).  N = 1: python tools/pack_grid.py;
N > 1: torchrun --nproc-per-node N tools/pack_grid.py"""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_09591_b200.layer import EPWorld, route_topk  # noqa: E402

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
G, E, K, M, T_r = 8, 128, 8, 2048, 4096
T = G // world * T_r
gen = torch.Generator(device="cuda").manual_seed(7 + rank)
lg = torch.randn(T, E, device="cuda", generator=gen)
x = torch.randn(T, M, device="cuda", generator=gen).to(torch.bfloat16)
w = EPWorld(G, E, K, M, T_r, dtype=torch.bfloat16, gpus=world, gpu_index=rank,
            n_cap_rows=3 * T_r * K)
slot, wts, _ = route_topk(lg, K)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def gtime(fn, n=20):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
    torch.cuda.current_stream().wait_stream(st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tot = 0.0
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    t = torch.tensor([tot / n * 1e3], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


w.dispatch(x, slot, wts, dedup="gpu")   # the combine below needs a dispatched step
for cap in (0, 592, 1184, 1776, 2368, 4736):
    w.set_max_blocks(cap)
    d = gtime(lambda: w.dispatch(x, slot, wts, dedup="gpu"))
    c = gtime(lambda: w.combine(slot, wts, dedup="gpu"))
    if rank == 0:
        print(json.dumps({"gpus": world, "grid": cap or "default", "dispatch_us": round(d, 1),
                          "combine_us": round(c, 1)}), flush=True)
torch.cuda.synchronize()
w.check_status()
w.close()
if world > 1:
    dist.destroy_process_group()
