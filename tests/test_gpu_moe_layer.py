"""Full MoE layer forward (gating -> dedup dispatch -> tcgen05 SwiGLU experts
-> dedup combine) vs the CPU restatement (oracle/moe.py) at bf16 tolerance.

Routing indices are compared bit-exactly on the same fp32 logits; the layer
values are parity-unpinned by the reference (no layer math there) and use
the BASELINE bf16 tolerance (rtol 2e-2)."""

import numpy as np
import pytest
import torch

from oracle import moe as OM

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dedup", ["all", "remote", "none"])
@pytest.mark.parametrize("shape", [(8, 16, 2, 256, 256, 64), (8, 64, 6, 512, 256, 40)])
def test_layer_forward_matches_oracle(hm, dedup, shape):
    from paper_2508_09591_b200.moe import HierMoELayer
    G, E, K, M, I, T_r = shape
    layer = HierMoELayer(G, E, K, M, I, T_r, dedup=dedup, seed=3)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(G * T_r, M, device="cuda", generator=g).to(torch.bfloat16)
    out = layer(x)
    torch.cuda.synchronize()
    layer.world.check_status()
    # the layer's router logits (tcgen05 GEMM, bf16 operands, fp32 accumulation)
    logits = layer.router_logits(x)
    ref_l = x.float() @ layer.w_router.to(torch.bfloat16).float().T
    torch.testing.assert_close(logits, ref_l, rtol=1e-4, atol=1e-4)
    logits = logits.cpu().numpy()
    slot, w, _ = OM.route_topk(logits, K, layer.expert_to_slot.cpu().numpy())
    # experts in slot space: local rank l holds slots [l*E_loc, (l+1)*E_loc)
    e_loc = E // G
    w13 = layer.w13.reshape(E, 2 * I, M).float().cpu().numpy()
    w2 = layer.w2.reshape(E, M, I).float().cpu().numpy()
    nb = I // 128
    gate = w13.reshape(E, nb, 2, 128, M)[:, :, 0].reshape(E, I, M)
    up = w13.reshape(E, nb, 2, 128, M)[:, :, 1].reshape(E, I, M)
    xs = x.float().cpu().numpy().astype(np.float64)

    def expert(rows, slots):
        outp = np.zeros((rows.shape[0], M))
        for e in np.unique(slots):
            sel = slots == e
            a = rows[sel] @ gate[e].T.astype(np.float64)
            b = rows[sel] @ up[e].T.astype(np.float64)
            h = a / (1.0 + np.exp(-a)) * b
            h = torch.tensor(h).to(torch.bfloat16).double().numpy()   # H is stored in bf16
            outp[sel] = h @ w2[e].T.astype(np.float64)
        return outp

    ref = OM.moe_forward(xs, slot.astype(np.int64), w, expert)
    got = out.double().cpu().numpy()
    np.testing.assert_allclose(got, ref, rtol=2e-2, atol=2e-2 * np.abs(ref).max())
    layer.close()


def test_layer_trace_and_placement_files(hm, tmp_path):
    """Routing trace CSV and placement JSON in the reference's formats: the
    recorded trace is the router's expert choice per token; adopting a
    planned placement file migrates the experts and leaves the layer's
    function bit-for-bit unchanged."""
    from paper_2508_09591_b200.moe import HierMoELayer
    G, E, K, M, I, T_r = 8, 16, 2, 256, 256, 64
    layer = HierMoELayer(G, E, K, M, I, T_r, dedup=True, seed=5, layer_index=3)
    g = torch.Generator(device="cuda").manual_seed(9)
    xs = [torch.randn(G * T_r, M, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2)]
    layer.record_trace()
    outs = [layer(x).clone() for x in xs]
    torch.cuda.synchronize()
    path = tmp_path / "trace.csv"
    layer.save_trace(path)
    entries = hm.load_trace(path, E)
    assert [(i, l) for i, l, _ in entries] == [(0, 3), (1, 3)]
    for (_, _, m), x in zip(entries, xs):
        _, _, ex = layer.route(x)
        want = np.zeros((G * T_r, E), dtype=bool)
        np.put_along_axis(want, ex.cpu().numpy().astype(np.int64), True, axis=1)
        assert np.array_equal(m.bits, want)
    # a planned placement (two swaps, one crossing local ranks) via the file
    perm = np.arange(E)
    perm[[1, 14]] = perm[[14, 1]]
    perm[[4, 5]] = perm[[5, 4]]
    hm.save_placements({3: hm.Placement(perm)}, E, tmp_path / "pl.json")
    layer.load_placement(tmp_path / "pl.json")
    assert np.array_equal(layer.placement.slot_to_expert, perm)
    layer.store.check_status()
    again = layer(xs[1])
    torch.cuda.synchronize()
    assert torch.equal(again, outs[1])
    layer.save_placement(tmp_path / "pl2.json")
    assert (tmp_path / "pl2.json").read_bytes() == (tmp_path / "pl.json").read_bytes()
    layer.close()


@pytest.mark.parametrize("dedup", [True, "none"])
def test_layer_dsv3_router_shared_expert(hm, dedup):
    """DeepSeek-V3-style layer: group-limited sigmoid gate (indices equal the
    oracle's on the layer's own logits) and a shared expert overlapped with
    the dispatch and summed into the combine."""
    from paper_2508_09591_b200.moe import HierMoELayer
    G, E, K, M, I, T_r, Is = 8, 64, 6, 512, 256, 40, 256
    layer = HierMoELayer(G, E, K, M, I, T_r, dedup=dedup, seed=11, router="dsv3", n_group=4,
                         topk_group=2, route_scale=2.5, shared_inter=Is, optimizer_state=False)
    g = torch.Generator(device="cuda").manual_seed(13)
    x = torch.randn(G * T_r, M, device="cuda", generator=g).to(torch.bfloat16)
    out = layer(x)
    torch.cuda.synchronize()
    layer.world.check_status()
    slot, w, ex = layer.route(x)
    logits = layer.router_logits(x).cpu().numpy()
    rs, rw, rex = OM.route_group_limited(logits, K, 4, 2, layer.score_bias.cpu().numpy(), 2.5,
                                         layer.expert_to_slot.cpu().numpy())
    assert np.array_equal(ex.cpu().numpy(), rex)
    np.testing.assert_allclose(w.cpu().numpy(), rw, rtol=1e-6, atol=1e-7)
    nb = I // 128
    w13 = layer.w13.reshape(E, 2 * I, M).float().cpu().numpy().reshape(E, nb, 2, 128, M)
    gate, up = w13[:, :, 0].reshape(E, I, M), w13[:, :, 1].reshape(E, I, M)
    w2 = layer.w2.reshape(E, M, I).float().cpu().numpy()
    xs = x.float().cpu().numpy().astype(np.float64)

    def ffn(rows, ga, u, d):
        a = rows @ ga.T.astype(np.float64)
        b = rows @ u.T.astype(np.float64)
        h = torch.tensor(a / (1.0 + np.exp(-a)) * b).to(torch.bfloat16).double().numpy()
        return h @ d.T.astype(np.float64)

    def expert(rows, slots):
        o = np.zeros((rows.shape[0], M))
        for e in np.unique(slots):
            sel = slots == e
            o[sel] = ffn(rows[sel], gate[e], up[e], w2[e])
        return o

    routed = OM.moe_forward(xs, slot.cpu().numpy().astype(np.int64), w.cpu().numpy(), expert)
    ws = layer.w13_shared.float().cpu().numpy().reshape(Is // 128, 2, 128, M)
    shared = ffn(xs, ws[:, 0].reshape(Is, M), ws[:, 1].reshape(Is, M),
                 layer.w2_shared.float().cpu().numpy())
    ref = routed + shared
    np.testing.assert_allclose(out.double().cpu().numpy(), ref, rtol=2e-2,
                               atol=2e-2 * np.abs(ref).max())
    layer.close()


@pytest.mark.parametrize("shape", [(4096, 2048), (3, 7), (1, 8), (0, 16)])
def test_widen_equals_float(shape):
    """hm_bf16_to_f32 (the router GEMM's fp32 operand) equals torch's cast bit
    for bit, including ragged tails and empty input."""
    from paper_2508_09591_b200.moe import HierMoELayer
    x = (torch.randn(shape, device="cuda") * 100).to(torch.bfloat16)
    xf = HierMoELayer.widen(x)
    torch.cuda.synchronize()
    assert xf.dtype == torch.float32 and torch.equal(xf, x.float())


@pytest.mark.parametrize("n", [4096 * 2048, 13, 8, 0])
@pytest.mark.parametrize("third", [False, True])
def test_sum_to_bf16(n, third):
    """hm_sum_to_bf16 = bf16((a + b) + c) with fp32 sums, bit for bit."""
    from paper_2508_09591_b200 import _lib
    from paper_2508_09591_b200._lib import ptr, stream_ptr
    a = torch.randn(n, device="cuda") * 3
    b = torch.randn(n, device="cuda").to(torch.bfloat16)
    c = torch.randn(n, device="cuda").to(torch.bfloat16) if third else None
    out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    _lib.call("hm_sum_to_bf16", ptr(a), ptr(b), ptr(c), ptr(out), n, stream_ptr())
    want = a + b.float()
    if third:
        want = want + c.float()
    torch.cuda.synchronize()
    assert torch.equal(out, want.to(torch.bfloat16))


def test_layer_auto_transport(hm):
    """dedup="auto": the layer takes the reference time model's choice on the
    step's mask (transport.choose_transport) and its output equals the layer
    run with that transport fixed."""
    from paper_2508_09591_b200.moe import HierMoELayer
    from paper_2508_09591_b200.routing import mask_from_ids
    from paper_2508_09591_b200.transport import choose_transport, runtime_topology
    G, E, K, M, I, T_r = 8, 64, 6, 512, 256, 64
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(G * T_r, M, device="cuda", generator=g).to(torch.bfloat16)
    # one GPU: flat [8] topology; dedup volumes are smaller -> d = 1 ("gpu" == "remote")
    for p, want in ((hm.LevelParams((), (), (1e-5,), (1e-12,)), "gpu"),):
        layer = HierMoELayer(G, E, K, M, I, T_r, dedup="auto", seed=3, transport_params=p,
                             transport_every=2)
        out = layer(x).clone()
        it, mode, ch = layer.transport_log[0]
        assert it == 0 and mode == ch.mode == want
        slot, _, _ = layer.route(x)
        ref = choose_transport(mask_from_ids(slot, E), runtime_topology(G, 1, E, M), p)
        assert ref == ch
        fixed = HierMoELayer(G, E, K, M, I, T_r, dedup=mode, seed=3)
        assert torch.equal(fixed(x), out)
        layer(x)
        layer(x)                       # iteration 2: re-evaluated
        assert [t[0] for t in layer.transport_log] == [0, 2]
        layer.close()
        fixed.close()
