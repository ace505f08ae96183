"""Multi-GPU parity worker (one process per GPU, launched by torchrun from
tests/test_gpu_multi.py).  Every rank builds the same global inputs, runs its
slice through the CUDA-IPC/NVLink dispatch + combine and checks the bit-exact
receive order, counts and expert-major rows, plus the combined output, against
the CPU oracle."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import moe as OM  # noqa: E402
from paper_2508_09591_b200.layer import EPWorld, route_topk  # noqa: E402


def run_case(rank, world, G, E, K, M, T_r, dtype, dedup, seed):
    L = G // world
    g = torch.Generator().manual_seed(seed)
    logits = torch.randn(G * T_r, E, generator=g)
    x = torch.randn(G * T_r, M, generator=g).to(dtype)
    lo, hi = rank * L * T_r, (rank + 1) * L * T_r
    slot, w, _ = route_topk(logits[lo:hi].cuda(), K)
    ids_all, w_all, _ = OM.route_topk(logits.numpy(), K)
    assert np.array_equal(slot.cpu().numpy(), ids_all[lo:hi]), "router ids"
    plan = OM.DispatchPlan(ids_all, G, E, gpus=world)
    ep = EPWorld(G, E, K, M, T_r, dtype=dtype, gpus=world, gpu_index=rank)
    ep.dispatch(x[lo:hi].cuda(), slot, w, dedup=dedup)
    torch.cuda.synchronize()
    ep.check_status()
    cnt = ep.counts()
    assert np.array_equal(cnt[:, :G], plan.h), "dedup counts"
    # per-GPU dedup: rows per (source rank, GPU) == dedup counts of the [P, L]
    # hierarchy's level-1 cut restricted to each source (group_reduce at U[1]=P)
    gh = plan.hit.reshape(-1, world, L).any(axis=2)
    src_of = np.arange(G * T_r) // T_r
    want_g = np.stack([gh[src_of == s_].sum(axis=0) for s_ in range(G)])
    assert np.array_equal(ep.gpu_counts(), want_g), "gpu counts"
    if dedup == "gpu":   # one row per (token, other GPU hit), landed in its first pick's slot
        rows = np.nonzero(gh[:, rank] & ((src_of // L) != rank))[0]
        assert ep.rows_received_gpu() == rows.size
    assert np.array_equal(cnt[:, G:], plan.c), "slot counts"
    rows = ep.rows_received()
    e_loc = E // G
    xb = x.view(torch.int16) if dtype == torch.bfloat16 else x.view(torch.int32)
    for l in range(L):
        d = rank * L + l
        n = int(rows[l, 1])
        assert n == int(plan.n_e[d * e_loc:(d + 1) * e_loc].sum())
        xm = ep.read("xmaj", l, dtype, n * M).view(n, M).cpu()
        tt, kk = np.nonzero(ids_all // e_loc == d)
        assert torch.equal(xm.view(xb.dtype)[plan.epos[tt, kk]], xb[tt]), f"xmaj rank {d}"
        if dedup in ("all", "remote"):
            want = plan.recv_rows(d)
            if dedup == "remote":   # only rows from sources on other GPUs cross a link
                want = want[(want // T_r) // L != rank]
            r = int(rows[l, 0])
            assert r == want.size, (r, want.size)
            rx = ep.read("recv_x", l, dtype, r * M).view(r, M).cpu()
            assert torch.equal(rx.view(xb.dtype), xb[want]), f"recv rank {d}"
        # stand-in expert: y = x * (1 + slot / E)
        row_slot = np.repeat(np.arange(d * e_loc, (d + 1) * e_loc), plan.n_e[d * e_loc:(d + 1) * e_loc])
        s = torch.as_tensor(1.0 + row_slot / E, dtype=torch.float32).cuda()[:, None]
        ep.set_expert_outputs(l, (xm.cuda().float() * s).to(dtype))
    torch.cuda.synchronize()
    out = ep.combine(slot, w, dedup=dedup)
    torch.cuda.synchronize()
    ep.check_status()
    sc = 1.0 + np.arange(E) / E
    ref = (w_all[lo:hi] * sc[ids_all[lo:hi]]).sum(axis=1)[:, None] * x[lo:hi].double().numpy()
    rtol = 1e-5 if dtype == torch.float32 else 2e-2
    np.testing.assert_allclose(out.double().cpu().numpy(), ref, rtol=rtol, atol=rtol * np.abs(ref).max())
    # repeated steps reuse the buffers and barriers (epochs advance)
    for _ in range(3):
        ep.dispatch(x[lo:hi].cuda(), slot, w, dedup=dedup)
        out2 = ep.combine(slot, w, dedup=dedup)
    torch.cuda.synchronize()
    ep.check_status()
    assert torch.equal(out2, out)
    if dedup == "gpu":
        # the step replayed from a CUDA graph (device-side barrier epochs):
        # every rank captures and replays the same sequence
        xin = x[lo:hi].cuda()
        gout = torch.empty_like(out)
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            ep.dispatch(xin, slot, w, dedup=dedup)
            ep.combine(slot, w, dedup=dedup, out=gout)
        torch.cuda.current_stream().wait_stream(st)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            ep.dispatch(xin, slot, w, dedup=dedup)
            ep.combine(slot, w, dedup=dedup, out=gout)
        for _ in range(3):
            gout.zero_()
            graph.replay()
        torch.cuda.synchronize()
        ep.check_status()
        assert torch.equal(gout, out), "graph replay"
    ep.close()


def run_backward(rank, world, dedup):
    """Dispatch / combine backward across GPUs (K8) vs the analytic gradients
    of stand-in experts y = s_e x: dw_k = <g_t, y_k>, dx_t = sum_k w_k s_k g_t
    (every transport, incl. per-GPU dedup: gradient rows cross NVLink once per
    (token, GPU), gate grads and pre-reduced input grads come back)."""
    G, E, K, M, T_r, dtype = 8, 128, 8, 512, 64, torch.bfloat16
    L = G // world
    gen = torch.Generator().manual_seed(31)
    logits = torch.randn(G * T_r, E, generator=gen)
    x = torch.randn(G * T_r, M, generator=gen).to(dtype)
    g = torch.randn(G * T_r, M, generator=gen).to(dtype)
    lo, hi = rank * L * T_r, (rank + 1) * L * T_r
    slot, w, _ = route_topk(logits[lo:hi].cuda(), K)
    ep = EPWorld(G, E, K, M, T_r, dtype=dtype, gpus=world, gpu_index=rank, grad=True)
    ep.dispatch(x[lo:hi].cuda(), slot, w, dedup=dedup)
    torch.cuda.synchronize()
    rows = ep.rows_received()
    e_loc = E // G
    n_e = ep.counts()[:, G:].sum(axis=0)
    scales = []
    for l in range(L):
        d = rank * L + l
        n = int(rows[l, 1])
        xm = ep.read("xmaj", l, dtype, n * M).view(n, M)
        row_slot = np.repeat(np.arange(d * e_loc, (d + 1) * e_loc), n_e[d * e_loc:(d + 1) * e_loc])
        sc = torch.as_tensor(1.0 + row_slot / E, dtype=torch.float32).cuda()[:, None]
        scales.append(sc)
        ep.set_expert_outputs(l, (xm.float() * sc).to(dtype))
    ep.combine(slot, w, dedup=dedup)
    dw = ep.dispatch_grad(g[lo:hi].cuda(), slot, w, dedup=dedup)
    for l in range(L):
        n = scales[l].shape[0]
        gy = ep.read("gy", l, dtype, n * M).view(n, M)
        ep.write("gx", (gy.float() * scales[l]).to(dtype).contiguous(), l)
    dx = ep.combine_grad(slot, dw, dedup=dedup)
    torch.cuda.synchronize()
    ep.check_status()
    ids = slot.cpu().numpy()
    s = (1.0 + np.arange(E) / E)[ids]
    wn = w.cpu().numpy().astype(np.float64)
    xd, gd = x[lo:hi].double().numpy(), g[lo:hi].double().numpy()
    ydot = (gd * xd).sum(axis=1)[:, None] * s
    ref_dx = (wn * s).sum(axis=1)[:, None] * gd
    np.testing.assert_allclose(dw.double().cpu().numpy(), ydot, rtol=3e-2,
                               atol=3e-2 * np.abs(ydot).max(), err_msg=f"dw {dedup}")
    np.testing.assert_allclose(dx.double().cpu().numpy(), ref_dx, rtol=3e-2,
                               atol=3e-2 * np.abs(ref_dx).max(), err_msg=f"dx {dedup}")
    ep.close()


def run_planner(rank, world):
    """Token-sharded swap planning: all-reduced statistics give every rank the
    reference's decision on the concatenated global mask."""
    import paper_2508_09591_b200 as hm
    from oracle import hiera as O
    G, E, K, T_r = 8, 128, 8, 512
    L = G // world
    g = torch.Generator().manual_seed(77)
    logits = torch.randn(G * T_r, E, generator=g)
    logits += 3.0 * torch.log1p(torch.arange(E, dtype=torch.float32)).neg()[torch.randperm(E, generator=g)]
    ids_all, _, _ = OM.route_topk(logits.numpy(), K)
    lo, hi = rank * L * T_r, (rank + 1) * L * T_r
    local = hm.mask_from_ids(torch.as_tensor(ids_all[lo:hi]), E)
    topo = hm.build_topology([8], E, 2048, 2)
    params = hm.LevelParams((), (), (2.0e-5,), (1.3e-12,))
    plan = hm.select_swap(local, topo, params, 10.0, None, group=dist.group.WORLD)
    bits = OM.ids_to_bits(ids_all, E)
    pair, saving, d, no_swap, q = O.select_swap(bits, (8,), ((), (), (2.0e-5,), (1.3e-12,)), 4096, 10.0)
    assert plan.pair == pair and plan.predicted_saving == saving and plan.no_swap_time == no_swap
    assert np.array_equal(plan.cost_matrix, q)


def run_migrate(rank, world):
    """Cross-GPU and same-GPU slot swaps through the expert store, chained
    back to back with no host synchronisation: consecutive swaps share a GPU
    (0<->1 then 0<->2 ...), the sequence that needs one staging record per
    source GPU (a shared staging area let the second partner overwrite GPU 0's
    staging before it had committed the first partner's expert)."""
    from paper_2508_09591_b200.migrate import ExpertStore
    S = 8
    # ~1.3 MB per slot: large enough that pushes and commits overlap in time
    arrays = {"w": ((256, 1024), torch.bfloat16), "m": ((65536,), torch.float32)}
    st = ExpertStore(S, arrays, gpus=world, gpu_index=rank)
    for i, k in enumerate(arrays):
        v = st[k]
        glob = rank * S + torch.arange(S, device="cuda")
        # bf16 holds integers exactly only up to 256: slot ids there, 10*slot+1 in fp32
        val = glob if i == 0 else glob * 10 + 1
        v.copy_(val.view(-1, *([1] * (v.dim() - 1))).to(v.dtype).expand_as(v))
    torch.cuda.synchronize()
    dist.barrier()
    pairs = [(1, world * S - 2), (2, 5)]              # GPU 0 <-> last GPU; both on GPU 0
    for q in range(1, world):                         # GPU 0 <-> every other GPU, chained
        pairs.append((3, q * S + 4))
    if world >= 3:
        pairs += [(S + 1, 2 * S + 6), (0, S + 1), (2 * S + 6, 7)]
    content = list(range(world * S))                  # global slot -> original slot id
    for r, c in pairs:
        st.migrate(r, c)
        content[r], content[c] = content[c], content[r]
    torch.cuda.synchronize()
    st.check_status()
    for i, k in enumerate(arrays):
        v = st[k]
        for j in range(S):
            src = content[rank * S + j]
            want = float(src if i == 0 else src * 10 + 1)
            row = v[j].flatten()
            assert float(row[0]) == want and float(row[-1]) == want, (k, rank * S + j)
            assert bool((row == want).all()), (k, rank * S + j)
    st.close()


def run_layer_fused(rank, world):
    """Fused dispatch across GPUs: local picks gathered from x, rows that crossed
    NVLink gathered from the receive buffers (per-GPU dedup, mode 3, and
    per-rank dedup, mode 2, forward + backward) -- outputs and gradients
    bit-identical to the copying dispatch."""
    from paper_2508_09591_b200.moe import HierMoELayer
    G, E, K, M, I, T_r = 8, 64, 6, 512, 256, 96
    L = G // world
    gen = torch.Generator(device="cuda").manual_seed(40 + rank)
    x = torch.randn(L * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    gout = torch.randn(L * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    for dedup, grad in (("gpu", False), ("remote", True), ("gpu", True)):
        res = []
        # copying dispatch, fused dispatch, fused + exchange inside the GEMMs
        for fused, overlap in ((False, False), (True, False), (True, True)):
            layer = HierMoELayer(G, E, K, M, I, T_r, gpus=world, gpu_index=rank, dedup=dedup,
                                 seed=3, grad=grad, fused_dispatch=fused, optimizer_state=False,
                                 overlap=overlap)
            assert layer.overlap_now() == (overlap and dedup == "gpu")
            out = layer(x).clone()
            if not grad:   # a second step reuses the buffers, barriers and flags
                out = layer(x).clone()
            got = [out]
            if grad:
                got += [layer.backward(gout).clone(), layer.dw13.clone(), layer.dw2.clone(),
                        layer.dw_router.clone()]
            torch.cuda.synchronize()
            layer.check_status()
            for wd in layer.worlds:
                wd.check_status()
            res.append(got)
            layer.close()
            dist.barrier()
        for other in res[1:]:
            for a, b in zip(res[0], other):
                assert torch.equal(a, b), ("fused / overlapped", dedup, grad)


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    cases = [(8, 16, 2, 256, 256, torch.float32), (8, 128, 8, 2048, 128, torch.bfloat16),
             (8, 256, 8, 512, 96, torch.bfloat16),
             # one EP rank per GPU (the N = 8 bench layout at this world size)
             (world, 32 * world, 4, 1024, 128, torch.bfloat16)]
    for i, (G, E, K, M, T_r, dt) in enumerate(cases):
        for dedup in ("all", "remote", "gpu", "none"):
            run_case(rank, world, G, E, K, M, T_r, dt, dedup, seed=100 + i)
            dist.barrier()
    for dedup in ("all", "remote", "gpu", "none"):
        run_backward(rank, world, dedup)
        dist.barrier()
    run_migrate(rank, world)
    dist.barrier()
    run_layer_fused(rank, world)
    dist.barrier()
    run_planner(rank, world)
    dist.barrier()
    if rank == 0:
        print("MULTI-GPU PARITY OK", world)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
