"""Host<->device copy rates from pinned memory (the e2e leg's ceiling): one
direction alone and both at once, with the copy split over 1/2/4 streams.
python tools/pcie_probe.py"""
import json

import torch

N = 128 << 20   # bytes per direction


def rate(h2d_streams, d2h_streams, reps=10):
    h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(N, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
    si = [torch.cuda.Stream() for _ in range(max(h2d_streams, 1))]
    so = [torch.cuda.Stream() for _ in range(max(d2h_streams, 1))]

    def once():
        for k in range(h2d_streams):
            c = N // h2d_streams
            with torch.cuda.stream(si[k]):
                d_in[k * c:(k + 1) * c].copy_(h_in[k * c:(k + 1) * c], non_blocking=True)
        for k in range(d2h_streams):
            c = N // d2h_streams
            with torch.cuda.stream(so[k]):
                h_out[k * c:(k + 1) * c].copy_(d_out[k * c:(k + 1) * c], non_blocking=True)

    once()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    for s in si + so:
        s.wait_event(a)
    for _ in range(reps):
        once()
    for s in si + so:
        cur.wait_stream(s)
    b.record(cur)
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    moved = N * (int(h2d_streams > 0) + int(d2h_streams > 0))
    return {"h2d_streams": h2d_streams, "d2h_streams": d2h_streams, "ms": round(ms, 3),
            "GB_s_total": round(moved / ms / 1e6, 1)}


for cfg in [(1, 0), (2, 0), (4, 0), (0, 1), (0, 2), (0, 4), (1, 1), (2, 2), (4, 4)]:
    print(json.dumps(rate(*cfg)), flush=True)
