"""Layer forward / backward with the fused dispatch (GEMM1 gathers its A rows
by index) vs the copying dispatch (expert-major rows materialised, TMA
loads), interleaved, for the Qwen3 and DeepSeek-V3 shapes.  N = 1:
python tools/fused_layer_probe.py; N > 1 under torchrun (one rank per GPU)."""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_09591_b200.moe import HierMoELayer  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl")
    configs = [a.split("=")[1] for a in sys.argv if a.startswith("--config=")] or ["qwen3", "dsv3"]
    for cfg in configs:
        if cfg == "qwen3":
            G, E, K, M, I, T_r = 8, 128, 8, 2048, 768, 4096
            kw = {}
        else:
            G, E, K, M, I, T_r = 8, 256, 8, 7168, 2048, 4096
            kw = dict(router="dsv3", n_group=8, topk_group=4, route_scale=2.5, shared_inter=2048,
                      optimizer_state=False)
        L = G // world
        gen = torch.Generator(device="cuda").manual_seed(5 + rank)
        x = torch.randn(L * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
        g = torch.randn(L * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
        layers = {f: HierMoELayer(G, E, K, M, I, T_r, gpus=world, gpu_index=rank, dedup=True,
                                  grad=True, n_cap_rows=2 * T_r * K, fused_dispatch=f, **kw)
                  for f in (True, False)}
        out = torch.empty_like(x)
        res = {f: [0.0, 0.0] for f in layers}
        reps = 3 if cfg == "dsv3" else 10
        for rep in range(2 + reps):
            for f, layer in layers.items():
                if world > 1:
                    dist.barrier()
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record()
                layer(x, out=out)
                e[1].record()
                layer.backward(g)
                e[2].record()
                e[2].synchronize()
                if rep >= 2:
                    res[f][0] += e[0].elapsed_time(e[1]) / reps
                    res[f][1] += e[1].elapsed_time(e[2]) / reps
        for f, layer in layers.items():
            t = torch.tensor(res[f], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if rank == 0:
                print(json.dumps({"config": cfg, "n_gpus": world, "fused_dispatch": f,
                                  "fwd_ms": round(t[0].item(), 4),
                                  "bwd_ms": round(t[1].item(), 4)}), flush=True)
            layer.close()
        del layers
        torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
