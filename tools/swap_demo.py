"""Expert swap end to end on structured routing: tokens pick most of their
experts from one of 16 co-selection clusters whose members start spread over
all EP ranks; the planner (reference rule, B200 alpha/beta, [N, L] hierarchy)
runs every step and each chosen pair is migrated (weights + optimizer state)
before the next step.  Records, per step, the per-GPU dedup rows of the
dispatch and the layer forward time.  torchrun for N > 1.

    torchrun --nproc-per-node N tools/swap_demo.py [--steps 300]
"""

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
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--in-cluster", type=int, default=6, help="picks from the token's cluster")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    G, E, K, M, I, T_r = 8, 128, 8, 2048, 768, args.tokens
    L = G // world
    layer = HierMoELayer(G, E, K, M, I, T_r, gpus=world, gpu_index=rank, dedup=True, seed=3)
    fan = [world, L] if world > 1 else [2, 4]
    topo = hm.build_topology(fan, E, M, 2)
    params = hm.LevelParams((3.14e-5,), (1.80e-13,), (3.36e-5, 3.15e-5), (2.84e-13, 3.59e-13))
    n_cl = 16
    member = torch.arange(E, device="cuda")
    cluster_of = member % n_cl          # cluster c = {c, c + 16, ...}: one member per rank
    x = torch.randn(L * T_r, M, device="cuda").to(torch.bfloat16)
    grp = dist.group.WORLD if world > 1 else None

    def logits_for(step):
        g = torch.Generator(device="cuda").manual_seed(1000 * step + rank)
        t = L * T_r
        cl = torch.randint(0, n_cl, (t,), device="cuda", generator=g)
        noise = torch.rand(t, E, device="cuda", generator=g)
        # the token's own cluster's 8 members rank first (the top in_cluster
        # of them win), the rest of the picks are random experts
        bonus = (cluster_of[None, :] == cl[:, None]).float() * 1.0
        keep = torch.rand(t, E, device="cuda", generator=g) < (args.in_cluster / 8.0)
        return noise + bonus * keep

    log = []
    for step in range(args.steps):
        lg = logits_for(step)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        slot, w, _ = route_topk(lg, K, layer.expert_to_slot)
        e0.record()
        layer._x_cur = x
        layer.world.set_fused(layer.fused_now())
        layer.world.dispatch(x, slot, w, dedup=True)
        layer.experts_forward()
        layer.world.combine(slot, w, dedup=True)
        e1.record()
        e1.synchronize()
        rows = torch.tensor([float(layer.world.gpu_counts().sum()), e0.elapsed_time(e1)],
                            dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(rows, op=dist.ReduceOp.MAX)
        p0, p1, p2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        p0.record()
        plan = hm.select_swap(hm.mask_from_ids(slot, E), topo, params, 10.0, None, group=grp)
        p1.record()
        layer.apply_swap(plan.pair)
        p2.record()
        p2.synchronize()
        kind = None
        if plan.pair is not None:   # same GPU (local slice swap) or across GPUs (NVLink push)
            per_gpu = layer.local * layer.e_loc
            kind = "same_gpu" if plan.pair[0] // per_gpu == plan.pair[1] // per_gpu else "cross_gpu"
        log.append((step, rows[0].item(), rows[1].item(), plan.pair is not None,
                    plan.predicted_saving, p0.elapsed_time(p1), p1.elapsed_time(p2), kind))
    layer.world.check_status()
    layer.store.check_status()
    if rank == 0:
        first, last = log[:10], log[-10:]
        print(json.dumps({
            "n_gpus": world, "topology": fan, "steps": args.steps,
            "swaps_taken": sum(1 for r in log if r[3]),
            "gpu_dedup_rows_first10": float(np.mean([r[1] for r in first])),
            "gpu_dedup_rows_last10": float(np.mean([r[1] for r in last])),
            "step_ms_first10": float(np.mean([r[2] for r in first])),
            "step_ms_last10": float(np.mean([r[2] for r in last])),
            "planner_ms_median": float(np.median([r[5] for r in log[5:]])),
            "migration_ms_median_when_swapped": float(np.median([r[6] for r in log[5:] if r[3]]))
            if any(r[3] for r in log[5:]) else None,
            # per kind: a cross-GPU swap moves one expert each way (bytes_per_slot
            # per direction over NVLink); a same-GPU swap exchanges two slices in HBM
            "bytes_per_slot": layer.store.bytes_per_slot(),
            "migration_by_kind": {
                kd: {"swaps": len(ts), "median_ms": float(np.median(ts)),
                     "GBps_per_direction": layer.store.bytes_per_slot() / (np.median(ts) * 1e-3) / 1e9
                     if kd == "cross_gpu" else None,
                     "HBM_GBps": 4 * layer.store.bytes_per_slot() / (np.median(ts) * 1e-3) / 1e9
                     if kd == "same_gpu" else None}
                for kd in ("same_gpu", "cross_gpu")
                for ts in [[r[6] for r in log[5:] if r[7] == kd]] if ts},
            "trace": [[r[0], r[1], round(r[2], 4), r[3]] for r in log[::10]]}))
    layer.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
