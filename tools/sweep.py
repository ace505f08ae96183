"""Config E sweep (BASELINE.json configs[4]): dispatch+combine time over
tokens/rank x top-k x hierarchy at the launched GPU count.

For each (T_r, K, topology): synthetic uniform routing of the Qwen3 layer
(E=128, hidden 2048, bf16, G = 8 EP ranks on N GPUs); measured (CUDA events,
max over ranks) dispatch+combine ms for
  flat [8]      dedup per destination GPU ("gpu", rows re-expanded at the
                destination), per destination rank ("remote") and none
  [2,4], [4,2]  the two-level HD2 path (TwoLevelWorld) and the flat dedup
plus the rows moved and the time model's d* for the mask (reference
params).  One JSON line per case.

    python tools/sweep.py [--tokens 4096 8192 16384] [--topk 2 4 8]
    torchrun --nproc-per-node N tools/sweep.py ...
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2508_09591_b200 as hm  # noqa: E402
from paper_2508_09591_b200.layer import EPWorld, TwoLevelWorld, route_topk  # noqa: E402


def timed(step, n_warm=3, n=10, world=1):
    for _ in range(n_warm):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        step()
    e1.record()
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / n], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, nargs="+", default=[4096, 8192, 16384, 32768, 65536])
    ap.add_argument("--topk", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--max-tokens-per-gpu", type=int, default=131072)
    ap.add_argument("--hd2", action="store_true", help="also time the two-level relay worlds")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    G, E, M = 8, 128, 2048
    L = G // world
    params = hm.LevelParams((0.497,), (5.29e-07,), (0.722, 0.571), (5.7e-07, 1.27e-07))
    for t_r in args.tokens:
        if L * t_r > args.max_tokens_per_gpu:
            continue
        for k in args.topk:
            g = torch.Generator(device="cuda").manual_seed(t_r + k)
            logits = torch.randn(L * t_r, E, device="cuda", generator=g)
            x = torch.randn(L * t_r, M, device="cuda", generator=g).to(torch.bfloat16)
            slot, w, _ = route_topk(logits, k)
            cap = 3 * t_r * k
            res = {"n_gpus": world, "tokens_per_rank": t_r, "top_k": k, "experts": E, "hidden": M}
            out = torch.empty_like(x)
            for mode, fused in (("gpu", False), ("remote", False), ("none", False),
                                ("gpu", True), ("remote", True)):
                ep = EPWorld(G, E, k, M, t_r, gpus=world, gpu_index=rank, n_cap_rows=cap)
                ep.set_fused(fused)

                def step():
                    ep.dispatch(x, slot, w, dedup=mode)
                    ep.combine(slot, w, dedup=mode, out=out)

                res[f"flat_{mode}{'_fused' if fused else ''}_ms"] = timed(step, world=world)
                if fused:
                    ep.close()
                    continue
                if mode == "gpu":
                    res["gpu_rows"] = int(ep.gpu_counts().sum())
                if mode == "remote":
                    cnt = ep.counts()
                    res["dedup_rows"] = int(cnt[:, :G].sum())
                    res["raw_rows"] = int(cnt[:, G:].sum())
                ep.check_status()
                ep.close()
            # the reference time model's transport choice on this mask with the
            # B200 runtime fits (transport.py), next to the measured best
            from paper_2508_09591_b200.transport import (choose_transport, default_params,
                                                         runtime_topology)
            rt = runtime_topology(G, world, E, M, 2)
            red = (lambda t_: dist.all_reduce(t_)) if world > 1 else None
            ch = choose_transport(hm.mask_from_ids(slot, E), rt, default_params(world, rt.num_levels),
                                  None, red)
            res["auto_mode"] = ch.mode
            res["auto_model_us"] = [round(v * 1e6, 1) for v in ch.times] + \
                [round(ch.time_without_dedup * 1e6, 1)]
            # the product runs dedup transports fused (row indices, no re-expansion)
            meas = {"gpu": res["flat_gpu_fused_ms"], "remote": res["flat_remote_fused_ms"],
                    "none": res["flat_none_ms"]}
            res["measured_best_mode"] = min(meas, key=meas.get)
            res["auto_over_best"] = round(meas[ch.mode] / min(meas.values()), 3)
            for fan in (((2, 4), (4, 2)) if args.hd2 else ()):
                tw = TwoLevelWorld(fan, E, k, M, t_r, gpus=world, gpu_index=rank,
                                   n_cap_rows=cap)

                def step2():
                    tw.dispatch(x, slot, w, dedup2="remote")
                    tw.combine(slot, w, dedup2="remote", out=out)

                res[f"hd2_{fan[0]}x{fan[1]}_ms"] = timed(step2, world=world)
                res[f"hd2_{fan[0]}x{fan[1]}_phase1_rows"] = int(tw.phase1.counts()[:, :G].sum())
                tw.phase1.check_status()
                tw.phase2.check_status()
                tw.close()
                # the reference cost model's choice for this mask (A6000 params)
                mask = hm.mask_from_ids(slot, E)
                topo = hm.build_topology(list(fan), E, M, 2)
                from paper_2508_09591_b200.traffic import _Model
                red = (lambda t: dist.all_reduce(t)) if world > 1 else None
                mdl = _Model(mask, topo, params, None, True, red).fetch()
                res[f"d_star_{fan[0]}x{fan[1]}"] = mdl.d_star
            if rank == 0:
                print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
