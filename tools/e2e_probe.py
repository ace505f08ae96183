"""Timeline of bench.py's end-to-end leg at N = 1 (Qwen3 step, pinned host
buffers, double-buffered copy-in / compute / copy-out streams): per-step event
times of H2D, compute and D2H, and the same pipeline without compute.
python tools/e2e_probe.py"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_09591_b200.layer import EPWorld, route_topk  # noqa: E402

G, E, K, M, T_r = 8, 128, 8, 2048, 4096
T = G * T_r
gen = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(T, M, device="cuda", generator=gen).to(torch.bfloat16)
logits = torch.randn(T, E, device="cuda", generator=gen)
ep = EPWorld(G, E, K, M, T_r, dtype=torch.bfloat16, n_cap_rows=3 * T_r * K)
ep.set_fused(True)
out = torch.empty(T, M, dtype=torch.bfloat16, device="cuda")
hx = [x.cpu().pin_memory() for _ in range(2)]
hl = [logits.cpu().pin_memory() for _ in range(2)]
ho = [torch.empty(T, M, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
dx = [torch.empty_like(x) for _ in range(2)]
dl = [torch.empty_like(logits) for _ in range(2)]
do = [torch.empty_like(out) for _ in range(2)]
comp = torch.cuda.current_stream()
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def ev():
    return torch.cuda.Event(enable_timing=True)


def run(n, compute=True, split_logits=False):
    h2d_done, comp_done, d2h_done = [ev(), ev()], [ev(), ev()], [ev(), ev()]
    for b in range(2):
        comp_done[b].record(comp)
        d2h_done[b].record(comp)
    marks = []
    t0 = ev()
    t0.record(comp)
    s_in.wait_event(t0)
    s_out.wait_event(t0)
    for i in range(n):
        b = i % 2
        m = [ev() for _ in range(6)]
        with torch.cuda.stream(s_in):
            s_in.wait_event(comp_done[b])
            m[0].record(s_in)
            dx[b].copy_(hx[b], non_blocking=True)
            dl[b].copy_(hl[b], non_blocking=True)
            m[1].record(s_in)
            h2d_done[b].record(s_in)
        comp.wait_event(h2d_done[b])
        comp.wait_event(d2h_done[b])
        m[2].record(comp)
        if compute:
            slot, wts, _ = route_topk(dl[b], K)
            ep.dispatch(dx[b], slot, wts, dedup="gpu")
            ep.combine(slot, wts, dedup="gpu", out=do[b])
        m[3].record(comp)
        comp_done[b].record(comp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(comp_done[b])
            m[4].record(s_out)
            ho[b].copy_(do[b], non_blocking=True)
            m[5].record(s_out)
            d2h_done[b].record(s_out)
        marks.append(m)
    torch.cuda.synchronize()
    rows = [[round(t0.elapsed_time(e), 3) for e in m] for m in marks]
    per = (rows[-1][5] - rows[2][5]) / (n - 3)
    return {"compute": compute, "ms_per_step": round(per, 3),
            "h2d_ms": round(sum(r[1] - r[0] for r in rows[2:]) / (n - 2), 3),
            "comp_ms": round(sum(r[3] - r[2] for r in rows[2:]) / (n - 2), 3),
            "d2h_ms": round(sum(r[5] - r[4] for r in rows[2:]) / (n - 2), 3),
            "timeline_last4": rows[-4:]}


for compute in (True, False, True):
    run(6, compute)
    print(json.dumps(run(24, compute)), flush=True)
