"""NVLink hardware byte counters around the dispatch + combine step (N > 1).

Reads NVML's per-link NVLink data counters (NVML_FI_DEV_NVLINK_THROUGHPUT_
DATA_TX / _RX, KiB, summed over the GPU's links) before and after S steps of
each transport and reports, per GPU and step, the bytes the links actually
carried next to the algorithmic remote-row bytes (rows that cross to another
GPU x row bytes, dispatch + combine) and the device-timed link time.  This is
the NVLink counter evidence a multi-rank ncu run cannot give (ncu serialises
kernels, so the device barriers of a multi-GPU step would deadlock).

    torchrun --nproc-per-node N tools/nvlink_counters.py [--steps 20]
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

from paper_2508_09591_b200 import _lib  # noqa: E402
from paper_2508_09591_b200.layer import EPWorld, route_topk  # noqa: E402

# (tx, rx, unit bytes): NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/_RX (KiB) and
# NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES (bytes); per link, or all links
# (scope 0xFFFFFFFF) -- whichever the driver implements is reported
FIELDS = {"throughput_data": (138, 139, 1024), "count_bytes": (202, 204, 1)}
ALL = 0xFFFFFFFF


class Links:
    def __init__(self, index: int):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.links = []
        for link in range(18):
            try:
                if pynvml.nvmlDeviceGetNvLinkState(self.h, link) == pynvml.NVML_FEATURE_ENABLED:
                    self.links.append(link)
            except pynvml.NVMLError:
                pass

    def read(self) -> dict:
        """{counter: (tx bytes, rx bytes)} per counter family and scope."""
        out = {}
        for name, (tx_id, rx_id, unit) in FIELDS.items():
            for scope_name, scopes in (("per_link", self.links), ("all_links", [ALL])):
                ids = [(fid, sc) for sc in scopes for fid in (tx_id, rx_id)]
                try:
                    vals = self.nv.nvmlDeviceGetFieldValues(self.h, ids)
                except self.nv.NVMLError:
                    continue
                tx = rx = 0
                ok = False
                for (fid, _), f in zip(ids, vals):
                    if f.nvmlReturn != 0:
                        continue
                    ok = True
                    v = int(f.value.ullVal) * unit
                    if fid == tx_id:
                        tx += v
                    else:
                        rx += v
                if ok:
                    out[f"{name}.{scope_name}"] = (tx, rx)
        return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--tokens", type=int, default=4096)
    args = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    G, E, K, M, T_r = 8, 128, 8, 2048, args.tokens
    L = G // world
    T = L * T_r
    gen = torch.Generator(device="cuda").manual_seed(7 + rank)
    logits = torch.randn(T, E, device="cuda", generator=gen)
    x = torch.randn(T, M, device="cuda", generator=gen).to(torch.bfloat16)
    links = Links(local)
    rb = M * 2
    res = {"gpus": world, "rank": rank, "links": len(links.links), "tokens_per_rank": T_r}
    for mode in ("gpu", "none"):
        ep = EPWorld(G, E, K, M, T_r, gpus=world, gpu_index=rank, n_cap_rows=3 * T_r * K)
        slot, w, _ = route_topk(logits, K)
        for _ in range(3):
            ep.dispatch(x, slot, w, dedup=mode)
            ep.combine(slot, w, dedup=mode)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = links.read()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            ep.dispatch(x, slot, w, dedup=mode)
            ep.combine(slot, w, dedup=mode)
        e1.record()
        e1.synchronize()
        dist.barrier()
        t1 = links.read()
        ep.check_status()
        # algorithmic remote bytes of this GPU per step (dispatch + combine)
        cnt = ep.counts()
        mine = list(range(rank * L, (rank + 1) * L))
        slot_gpu = (np.arange(E) // (E // G)) // L
        if mode == "gpu":
            gc = ep.gpu_counts()[mine]
            sent = int(np.delete(gc, rank, axis=1).sum())           # rows pushed out
            recv = int(ep.rows_received_gpu())                      # rows pushed in
            tx_rows, rx_rows = sent + recv, recv + sent             # + the combine mirror
        else:
            sent = int(cnt[mine][:, G:][:, slot_gpu != rank].sum())
            src_gpu = np.arange(G) // L
            recv = int(cnt[src_gpu != rank][:, G:][:, slot_gpu == rank].sum())
            tx_rows, rx_rows = sent + recv, recv + sent
        ms = e0.elapsed_time(e1) / args.steps
        res[mode] = {"ms_per_step": ms,
                     "counters_bytes_per_step": {
                         k: [(t1[k][0] - t0[k][0]) / args.steps, (t1[k][1] - t0[k][1]) / args.steps]
                         for k in t1 if k in t0},
                     "algorithmic_tx_bytes_per_step": tx_rows * rb,
                     "algorithmic_rx_bytes_per_step": rx_rows * rb}
        ep.close()
    out = [None] * world
    dist.all_gather_object(out, res)
    if rank == 0:
        print(json.dumps({"tool": "nvlink_counters", "per_gpu": out}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
