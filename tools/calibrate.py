"""B200 alpha/beta calibration of the executed exchange.

The reference fits seconds = alpha + beta * bytes per phase kind from
nccl-tests measurements on its cluster (cli.py:79-110, topology.py:256-276,
PAPER.md:545-558).  Here the phases are our own dispatch kernels on this box:

  std      flat dedup dispatch over G = 8 ranks (pack + barrier)
  inter.1  phase 1 of the two-level [2, 4] dispatch (relay world)
  intra.1  phase 2 of the two-level [2, 4] dispatch (re-dedup inside the group)

For each phase and token count, x = the model's volume for that phase
(participants * max group count * token bytes, traffic.py:93-120) and y =
the measured device time of the phase.  The series are fitted with the
package's fit_params (same OLS as the reference) and written as a params JSON
in the reference schema.  Launch with torchrun for N > 1.

    python tools/calibrate.py [--out profiles/params_b200.json]

``--runtime`` fits the RUNTIME hierarchy [P GPUs, L ranks per GPU] that the
layer's transport choice evaluates (paper_2508_09591_b200/transport.py):

  std      flat dispatch: "none" (one row per selection) and "remote" (one row
           per (token, remote rank), fused) -- pack + barrier + index, volume
           G * max rank count * token bytes (raw resp. dedup counts)
  inter.1  the GPU-level dedup push ("gpu", fused: pack + barrier), volume
           P * max per-GPU count * token bytes
  intra.1  its index step inside the GPU ("gpu": expand segment), volume
           L * max per-rank count * token bytes

    torchrun --nproc-per-node N tools/calibrate.py --runtime \
        --out paper_2508_09591_b200/params/b200_runtime_nN.json
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
from paper_2508_09591_b200 import _lib  # noqa: E402
from paper_2508_09591_b200.layer import EPWorld, TwoLevelWorld, route_topk  # noqa: E402

SEG_PACK = 2


def seg_ms(world: EPWorld, seg: int) -> float:
    import ctypes
    buf = (ctypes.c_float * 8)()
    _lib.call("hm_world_timings", world._h, buf, 8)
    return float(buf[seg]) + max(0.0, float(buf[3]))   # pack + barrier1


def seg_list(world: EPWorld) -> list[float]:
    import ctypes
    buf = (ctypes.c_float * 8)()
    _lib.call("hm_world_timings", world._h, buf, 8)
    return [max(0.0, float(v)) for v in buf]


def runtime_fit(args, world: int, rank: int) -> None:
    G, E, K, M = 8, args.experts, args.top_k, args.hidden
    if world < 2 or G % world or G // world < 2:
        raise SystemExit("--runtime needs 2..4 GPUs (a two-level [P, L] hierarchy)")
    L = G // world
    tb = M * 2
    series = {"std": [], "inter.1": [], "intra.1": []}
    for k in sorted({2, 4, K}):
        for t_r in (512, 1024, 2048, 4096):
            g = torch.Generator(device="cuda").manual_seed(t_r + k)
            logits = torch.randn(L * t_r, E, device="cuda", generator=g)
            x = torch.randn(L * t_r, M, device="cuda", generator=g).to(torch.bfloat16)
            slot, w, _ = route_topk(logits, k)
            from paper_2508_09591_b200.traffic import _device_counts
            dd, raw, _ = _device_counts(hm.mask_from_ids(slot, E), [world, G])
            if world > 1:
                dist.all_reduce(dd)
                dist.all_reduce(raw)
            c, r = dd.cpu().numpy(), raw.cpu().numpy()
            vol = {"none": G * int(r[world:].max()) * tb, "remote": G * int(c[world:].max()) * tb,
                   "inter": world * int(c[:world].max()) * tb,
                   "intra": L * int(c[world:].max()) * tb}
            ep = EPWorld(G, E, k, M, t_r, gpus=world, gpu_index=rank, n_cap_rows=3 * t_r * k)
            _lib.call("hm_world_set_timing", ep._h, 1)
            ms = {"none": [], "remote": [], "inter": [], "intra": []}
            for it in range(10):
                for mode in ("none", "remote", "gpu"):
                    # the dedup transports run fused, as in the layer (row
                    # indices instead of local copies and re-expansion)
                    ep.set_fused(mode != "none")
                    ep.dispatch(x, slot, w, dedup=mode)
                    torch.cuda.synchronize()
                    sg = seg_list(ep)
                    if mode == "gpu":
                        ms["inter"].append(sg[2] + sg[3])
                        ms["intra"].append(sg[4])
                    else:   # "none" has no expand launch (its event pair is stale)
                        ms[mode].append(sg[2] + sg[3] + (sg[4] if mode == "remote" else 0.0))
            keys = ("none", "remote", "inter", "intra")
            t = torch.tensor([np.median(ms[q][3:]) for q in keys], dtype=torch.float64,
                             device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = dict(zip(keys, (t / 1e3).tolist()))
            series["std"].append(hm.Measurement(vol["none"], sec["none"]))
            series["std"].append(hm.Measurement(vol["remote"], sec["remote"]))
            series["inter.1"].append(hm.Measurement(vol["inter"], sec["inter"]))
            series["intra.1"].append(hm.Measurement(vol["intra"], sec["intra"]))
            ep.close()
    fits = {q: hm.fit_params(v) for q, v in series.items()}
    params = hm.LevelParams((max(fits["inter.1"].alpha, 0.0),), (max(fits["inter.1"].beta, 1e-15),),
                            (max(fits["std"].alpha, 0.0), max(fits["intra.1"].alpha, 0.0)),
                            (max(fits["std"].beta, 1e-15), max(fits["intra.1"].beta, 1e-15)))
    if rank == 0:
        print(json.dumps({"gpus": world, "runtime_topology": [world, L],
                          "series": {q: [[m.bytes, m.seconds] for m in v] for q, v in series.items()},
                          "fits": {q: {"alpha": f.alpha, "beta": f.beta, "r2": f.r_squared}
                                   for q, f in fits.items()}}))
        if args.out:
            Path(args.out).parent.mkdir(parents=True, exist_ok=True)
            hm.save_params(params, args.out, {q: f.r_squared for q, f in fits.items()})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--runtime", action="store_true",
                    help="fit the runtime [P, L] transports (none/remote/gpu)")
    ap.add_argument("--experts", type=int, default=128)
    ap.add_argument("--hidden", type=int, default=2048)
    ap.add_argument("--top-k", type=int, default=8)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    if args.runtime:
        runtime_fit(args, world, rank)
        dist.destroy_process_group()
        return
    G, E, K, M = 8, args.experts, args.top_k, args.hidden
    L = G // world
    tb = M * 2
    series = {"std": [], "inter.1": [], "intra.1": []}
    topo1 = hm.build_topology([G], E, M, 2)
    topo2 = hm.build_topology([2, 4], E, M, 2)
    for t_r in (256, 512, 1024, 2048, 4096):
        g = torch.Generator(device="cuda").manual_seed(t_r)
        logits = torch.randn(L * t_r, E, device="cuda", generator=g)
        x = torch.randn(L * t_r, M, device="cuda", generator=g).to(torch.bfloat16)
        slot, w, _ = route_topk(logits, K)
        # model volumes from the global mask (token-sharded counts all-reduced)
        mask = hm.mask_from_ids(slot, E)
        from paper_2508_09591_b200.traffic import _device_counts
        dd, _, _ = _device_counts(mask, [2, G])
        if world > 1:
            dist.all_reduce(dd)
        c = dd.cpu().numpy()
        v_std = G * int(c[2:].max()) * tb
        v_inter = 2 * int(c[:2].max()) * tb
        v_intra = (G // 2) * int(c[2:].max()) * tb
        ep = EPWorld(G, E, K, M, t_r, gpus=world, gpu_index=rank)
        tw = TwoLevelWorld((2, 4), E, K, M, t_r, gpus=world, gpu_index=rank)
        for w_ in (ep, tw.phase1, tw.phase2):
            _lib.call("hm_world_set_timing", w_._h, 1)
        ms = {"std": [], "inter.1": [], "intra.1": []}
        for it in range(8):
            ep.dispatch(x, slot, w, dedup="all")
            torch.cuda.synchronize()
            ms["std"].append(seg_ms(ep, SEG_PACK))
            tw.dispatch(x, slot, w, dedup2="all")
            torch.cuda.synchronize()
            ms["inter.1"].append(seg_ms(tw.phase1, SEG_PACK))
            ms["intra.1"].append(seg_ms(tw.phase2, SEG_PACK))
        t = torch.tensor([np.median(ms[k][2:]) for k in ("std", "inter.1", "intra.1")],
                         dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        for k, v, sec in zip(("std", "inter.1", "intra.1"), (v_std, v_inter, v_intra),
                             (t / 1e3).tolist()):
            series[k].append(hm.Measurement(v, sec))
        ep.close()
        tw.close()
    fits = {k: hm.fit_params(v) for k, v in series.items()}
    params = hm.LevelParams((fits["inter.1"].alpha,), (max(fits["inter.1"].beta, 1e-15),),
                            (max(fits["std"].alpha, 0.0), max(fits["intra.1"].alpha, 0.0)),
                            (max(fits["std"].beta, 1e-15), max(fits["intra.1"].beta, 1e-15)))
    if rank == 0:
        out = {"gpus": world, "series": {k: [[m.bytes, m.seconds] for m in v]
                                         for k, v in series.items()},
               "fits": {k: {"alpha": f.alpha, "beta": f.beta, "r2": f.r_squared}
                        for k, f in fits.items()}}
        # d* under the B200 parameters for a uniform Qwen3-shaped step on [2, 4]
        gen = hm.generate_uniform(8 * 512, E, K, 1)
        d_star, rep = hm.optimal_dimension(gen, topo2, params)
        out["d_star_qwen3_2x4"] = d_star
        out["times_qwen3_2x4"] = list(rep.times)
        print(json.dumps(out))
        if args.out:
            hm.save_params(params, args.out, {k: f.r_squared for k, f in fits.items()})
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
