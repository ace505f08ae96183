"""Full HierMoELayer backward (combine bwd -> tcgen05 FFN bwd -> dispatch bwd ->
softmax top-K bwd -> router) vs torch autograd in fp32 on the same bf16
inputs/weights and the same routing picks (bf16 tolerance)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dedup", ["all", "remote", "gpu", "none"])
def test_layer_backward_matches_autograd(hm, dedup):
    from paper_2508_09591_b200.moe import HierMoELayer
    G, E, K, M, I, T_r = 8, 16, 2, 256, 256, 32
    layer = HierMoELayer(G, E, K, M, I, T_r, dedup=dedup, seed=9, grad=True)
    gen = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(G * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    gout = torch.randn(G * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    out = layer(x)
    dx = layer.backward(gout)
    torch.cuda.synchronize()
    layer.world.check_status()
    slot, w, ex = layer._saved[-3:]
    # reference: same picks, fp32 autograd
    xr = x.float().requires_grad_(True)
    wr = layer.w_router.to(torch.bfloat16).float().requires_grad_(True)   # the GEMM's operand
    nb = I // 128
    w13 = layer.w13.reshape(E, nb, 2, 128, M).float()
    w1 = w13[:, :, 0].reshape(E, I, M).clone().requires_grad_(True)
    w3 = w13[:, :, 1].reshape(E, I, M).clone().requires_grad_(True)
    w2 = layer.w2.reshape(E, M, I).float().clone().requires_grad_(True)
    logits = xr @ wr.T
    picked = torch.gather(logits, 1, ex.long())
    gates = torch.softmax(picked, dim=1)
    slots = slot.long()
    y = torch.zeros_like(xr)
    for k in range(K):
        e = slots[:, k]
        a = torch.einsum("tm,tim->ti", xr, w1[e])
        b = torch.einsum("tm,tim->ti", xr, w3[e])
        hcur = torch.nn.functional.silu(a) * b
        y = y + gates[:, k:k + 1] * torch.einsum("ti,tmi->tm", hcur, w2[e])
    y.backward(gout.float())
    torch.testing.assert_close(out.float(), y.detach(), rtol=3e-2, atol=3e-2)
    torch.testing.assert_close(dx.float(), xr.grad, rtol=3e-2, atol=3e-2)
    torch.testing.assert_close(layer.dw_router, wr.grad, rtol=3e-2, atol=3e-2 * wr.grad.abs().max().item())
    d13 = torch.stack([w1.grad.view(E, nb, 128, M), w3.grad.view(E, nb, 128, M)], dim=2).reshape(E, 2 * I, M)
    got13 = layer.dw13.reshape(E, 2 * I, M).float()
    torch.testing.assert_close(got13, d13, rtol=3e-2, atol=3e-2 * d13.abs().max().item())
    got2 = layer.dw2.reshape(E, M, I).float()
    torch.testing.assert_close(got2, w2.grad, rtol=3e-2, atol=3e-2 * w2.grad.abs().max().item())
    layer.close()


def test_layer_backward_dsv3_shared_matches_autograd(hm):
    """DeepSeek-V3-style layer backward: normalised-sigmoid gate (group-limited
    picks), routed experts and the shared expert, vs fp32 autograd on the same
    picks (bf16 tolerance)."""
    from paper_2508_09591_b200.moe import HierMoELayer
    G, E, K, M, I, T_r, Is, c = 8, 32, 4, 256, 256, 32, 256, 2.5
    layer = HierMoELayer(G, E, K, M, I, T_r, dedup=True, seed=4, grad=True, router="dsv3",
                         n_group=4, topk_group=2, route_scale=c, shared_inter=Is,
                         optimizer_state=False)
    gen = torch.Generator(device="cuda").manual_seed(8)
    x = torch.randn(G * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    gout = torch.randn(G * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    out = layer(x)
    dx = layer.backward(gout)
    torch.cuda.synchronize()
    layer.world.check_status()
    slot, w, ex = layer._saved[-3:]
    xr = x.float().requires_grad_(True)
    wr = layer.w_router.to(torch.bfloat16).float().requires_grad_(True)   # the GEMM's operand

    def split13(w13, n, i):
        v = w13.reshape(n, i // 128, 2, 128, M).float()
        return (v[:, :, 0].reshape(n, i, M).clone().requires_grad_(True),
                v[:, :, 1].reshape(n, i, M).clone().requires_grad_(True))

    w1, w3 = split13(layer.w13, E, I)
    w2 = layer.w2.reshape(E, M, I).float().clone().requires_grad_(True)
    s1, s3 = split13(layer.w13_shared, 1, Is)
    s2 = layer.w2_shared.float().clone().requires_grad_(True)
    logits = xr @ wr.T
    sc = torch.sigmoid(torch.gather(logits, 1, ex.long()))
    gates = sc / sc.sum(dim=1, keepdim=True) * c
    slots = slot.long()
    y = torch.zeros_like(xr)
    for k in range(K):
        e = slots[:, k]
        a = torch.einsum("tm,tim->ti", xr, w1[e])
        b = torch.einsum("tm,tim->ti", xr, w3[e])
        y = y + gates[:, k:k + 1] * torch.einsum("ti,tmi->tm", torch.nn.functional.silu(a) * b,
                                                   w2[e])
    hs = torch.nn.functional.silu(xr @ s1[0].T) * (xr @ s3[0].T)
    y = y + hs @ s2.T
    y.backward(gout.float())
    torch.testing.assert_close(out.float(), y.detach(), rtol=3e-2, atol=3e-2)
    torch.testing.assert_close(dx.float(), xr.grad, rtol=3e-2, atol=3e-2 * xr.grad.abs().max().item())
    torch.testing.assert_close(layer.dw_router, wr.grad, rtol=3e-2,
                               atol=3e-2 * wr.grad.abs().max().item())
    nb = I // 128
    d13 = torch.stack([w1.grad.view(E, nb, 128, M), w3.grad.view(E, nb, 128, M)], dim=2).reshape(E, 2 * I, M)
    torch.testing.assert_close(layer.dw13.reshape(E, 2 * I, M).float(), d13, rtol=3e-2,
                               atol=3e-2 * d13.abs().max().item())
    torch.testing.assert_close(layer.dw2.reshape(E, M, I).float(), w2.grad, rtol=3e-2,
                               atol=3e-2 * w2.grad.abs().max().item())
    nbs = Is // 128
    ds13 = torch.stack([s1.grad.view(1, nbs, 128, M), s3.grad.view(1, nbs, 128, M)], dim=2).reshape(1, 2 * Is, M)
    torch.testing.assert_close(layer.dw13_shared.float(), ds13, rtol=3e-2,
                               atol=3e-2 * ds13.abs().max().item())
    torch.testing.assert_close(layer.dw2_shared[0].float(), s2.grad, rtol=3e-2,
                               atol=3e-2 * s2.grad.abs().max().item())
    layer.close()


@pytest.mark.parametrize("router", ["softmax", "dsv3"])
def test_micro_batched_layer_matches_single(hm, router):
    """Two micro-batches (separate EP worlds on two streams, exchange of one
    overlapping the other's experts) give the same outputs and input grads
    bit for bit, and the same weight grads up to the bf16 rounding of the
    per-micro-batch accumulation."""
    from paper_2508_09591_b200.moe import HierMoELayer
    G, E, K, M, I, T_r = 8, 32, 4, 256, 256, 64
    kw = dict(dedup=True, seed=21, grad=True, router=router, optimizer_state=False)
    if router == "dsv3":
        kw.update(n_group=4, topk_group=2, route_scale=2.5, shared_inter=256)
    one = HierMoELayer(G, E, K, M, I, T_r, **kw)
    two = HierMoELayer(G, E, K, M, I, T_r, micro_batches=2, **kw)
    gen = torch.Generator(device="cuda").manual_seed(22)
    x = torch.randn(G * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    gout = torch.randn(G * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    y1, y2 = one(x), two(x)
    d1, d2 = one.backward(gout), two.backward(gout)
    torch.cuda.synchronize()
    for wd in two.worlds:
        wd.check_status()
    assert torch.equal(y1, y2)
    assert torch.equal(d1, d2)
    torch.testing.assert_close(two.dw_router, one.dw_router, rtol=1e-5, atol=1e-5)
    for a, b in ((one.dw13, two.dw13), (one.dw2, two.dw2)):
        torch.testing.assert_close(b.float(), a.float(), rtol=2e-2,
                                   atol=2e-2 * a.float().abs().max().item())
    one.close()
    two.close()
