"""Config D (BASELINE.json configs[3]): expert-swap stress on the Qwen3 layer.

Zipf(s=1.2)-skewed routing (persistent popularity ranking, fresh Gumbel draws
each step: top-K of log w + Gumbel noise is weighted sampling without
replacement, the reference's exponential race, routing.py:166-173), full layer
forward every step (gating, dedup dispatch, tcgen05 experts, combine), and
every `swap_every` steps the GPU swap planner on the current routing
(token-sharded statistics all-reduced over NCCL for N > 1) followed by
peer-to-peer migration of the chosen experts' weights + fp32 master + Adam
moments.  Prints one JSON line.

    python tools/swap_stress.py [--steps 200] [--swap-every 50]
    torchrun --nproc-per-node N tools/swap_stress.py ...
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2508_09591_b200 as hm  # noqa: E402
from paper_2508_09591_b200.layer import route_topk  # noqa: E402
from paper_2508_09591_b200.moe import HierMoELayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--swap-every", type=int, default=10)
    ap.add_argument("--zipf", type=float, default=1.2)
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--gamma", type=float, default=10.0)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    G, E, K, M, I, T_r = 8, 128, 8, 2048, 768, args.tokens
    L = G // world
    layer = HierMoELayer(G, E, K, M, I, T_r, gpus=world, gpu_index=rank, dedup=True)
    # the runtime's hierarchy: GPUs (per-GPU dedup over NVLink), then the EP
    # ranks inside a GPU; one GPU plans for the virtual [2, 4] split.  alpha/
    # beta are the B200 fits of tools/calibrate.py (profiles/r01_calib_n4.json:
    # inter.1 = the GPU-level phase, std / intra.1 = the flat / in-group ones)
    fan = [world, L] if world > 1 else [2, 4]
    topo = hm.build_topology(fan, E, M, 2)
    params = hm.LevelParams((3.14e-5,), (1.80e-13,), (3.36e-5, 3.15e-5), (2.84e-13, 3.59e-13))
    g = torch.Generator(device="cuda").manual_seed(2024)
    ranking = torch.randperm(E, device="cuda", generator=g)
    zipf_bias = torch.empty(E, device="cuda")
    zipf_bias[ranking] = -args.zipf * torch.log(torch.arange(1, E + 1, device="cuda", dtype=torch.float32))
    x = torch.randn(L * T_r, M, device="cuda", generator=g).to(torch.bfloat16)
    grp = dist.group.WORLD if world > 1 else None

    def logits_for(step):
        gs = torch.Generator(device="cuda").manual_seed(10_000 * step + rank)
        u = torch.rand(L * T_r, E, device="cuda", generator=gs).clamp_min(1e-20)
        return zipf_bias[None, :] - torch.log(-torch.log(u))   # + Gumbel(0, 1)

    out = torch.empty_like(x)
    step_ms, plan_ms, mig_ms, swaps, loads, gpu_rows = [], [], [], [], [], []
    for step in range(args.steps):
        lg = logits_for(step)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        slot, w, _ = route_topk(lg, K, layer.expert_to_slot)
        layer.world.dispatch(x, slot, w, dedup=True)
        layer.experts_forward()
        layer.world.combine(slot, w, dedup=True, out=out)
        e1.record()
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        rows = layer.world.rows_received()[:, 1].astype(np.int64)
        loads.append(int(rows.max()))
        gpu_rows.append(int(layer.world.gpu_counts().sum()))
        if args.swap_every and step % args.swap_every == 0:
            p0, p1, p2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            p0.record()
            mask = hm.mask_from_ids(slot, E)            # slot space (current placement)
            plan = hm.select_swap(mask, topo, params, args.gamma, None, group=grp)
            p1.record()
            layer.apply_swap(plan.pair)
            p2.record()
            p2.synchronize()
            plan_ms.append(p0.elapsed_time(p1))
            mig_ms.append(p1.elapsed_time(p2))
            swaps.append({"step": step, "pair": list(plan.pair) if plan.pair else None,
                          "d_star": plan.d_star,
                          "predicted_saving_s": plan.predicted_saving,
                          "no_swap_time_s": plan.no_swap_time})
    layer.world.check_status()
    layer.store.check_status()
    t = torch.tensor([np.mean(step_ms[5:]), np.mean(step_ms[5:55]), np.mean(step_ms[-50:]),
                      max(plan_ms) if plan_ms else 0.0, max(mig_ms) if mig_ms else 0.0,
                      np.mean(gpu_rows[:10]), np.mean(gpu_rows[-10:])],
                     dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({
            "config": "expert-swap stress: Qwen3 layer (E=128, top-8, hidden 2048, I=768, bf16), "
                      f"Zipf s={args.zipf}, {args.steps} steps, swap every {args.swap_every}",
            "n_gpus": world, "tokens_per_rank": T_r, "layer_fwd_ms_mean": t[0].item(),
            "layer_fwd_ms_first50": t[1].item(), "layer_fwd_ms_last50": t[2].item(),
            "planner_ms_max": t[3].item(), "migration_ms_max": t[4].item(),
            "migration_bytes_per_expert": layer.store.bytes_per_slot(),
            "expert_rows_max_per_rank_first": loads[0], "expert_rows_max_per_rank_last": loads[-1],
            "topology": fan,
            "gpu_dedup_rows_first10": t[5].item(), "gpu_dedup_rows_last10": t[6].item(),
            "swaps_taken": sum(1 for s_ in swaps if s_["pair"]),
            "swaps": swaps}))
    layer.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
