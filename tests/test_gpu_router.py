"""The router path on hand-written kernels (gating PAPER.md:112):
tcgen05 router GEMMs with fp32 results (hm_gemm_f32 / hm_wgrad_f32) and the
device gate backward (hm_gate_backward), vs torch fp32 on the same bf16
operands."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _call(name, *args):
    from paper_2508_09591_b200 import _lib
    _lib.call(name, *args)


@pytest.mark.parametrize("E,M,T", [(16, 256, 1000), (128, 2048, 4096), (256, 7168, 777)])
def test_router_logits_gemm(hm, E, M, T):
    from paper_2508_09591_b200._lib import ptr, stream_ptr
    g = torch.Generator(device="cuda").manual_seed(E)
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(E, M, device="cuda", generator=g) * M ** -0.5).to(torch.bfloat16)
    e256 = -(-E // 256) * 256
    wp = torch.zeros(e256, M, dtype=torch.bfloat16, device="cuda")
    wp[:E] = w
    out = torch.full((T, E), float("nan"), device="cuda")
    rows = torch.tensor([T], dtype=torch.int32, device="cuda")
    _call("hm_gemm_f32", ptr(x), T, ptr(rows), ptr(wp), e256, M, E, ptr(out), E, stream_ptr())
    torch.cuda.synchronize()
    ref = x.float() @ w.float().T
    torch.testing.assert_close(out, ref, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("E,K", [(16, 2), (128, 8), (256, 8)])
def test_gate_backward(hm, mode, E, K):
    from paper_2508_09591_b200._lib import ptr, stream_ptr
    T = 999
    g = torch.Generator(device="cuda").manual_seed(E + K + mode)
    logits = torch.randn(T, E, device="cuda", generator=g)
    ex = torch.argsort(torch.rand(T, E, device="cuda", generator=g), dim=1)[:, :K].to(torch.int32)
    c = 2.5
    if mode == 2:
        sk = torch.sigmoid(torch.gather(logits, 1, ex.long()))
        w = c * sk / sk.sum(dim=1, keepdim=True)
    else:
        p = torch.softmax(torch.gather(logits, 1, ex.long()), dim=1) if mode == 0 else \
            torch.gather(torch.softmax(logits, dim=1), 1, ex.long())
        w = p
    dw = torch.randn(T, K, device="cuda", generator=g)
    ld = -(-E // 128) * 128
    out = torch.full((T, ld), float("nan"), dtype=torch.bfloat16, device="cuda")
    _call("hm_gate_backward", ptr(logits), ptr(ex), ptr(w), ptr(dw), T, E, K, mode, c, ptr(out),
          ld, stream_ptr())
    torch.cuda.synchronize()
    # autograd reference of the same gate
    lg = logits.clone().requires_grad_(True)
    if mode == 0:
        wr = torch.softmax(torch.gather(lg, 1, ex.long()), dim=1)
    elif mode == 1:
        wr = torch.gather(torch.softmax(lg, dim=1), 1, ex.long())
    else:
        s = torch.sigmoid(torch.gather(lg, 1, ex.long()))
        wr = c * s / s.sum(dim=1, keepdim=True)
    wr.backward(dw)
    torch.testing.assert_close(out[:, :E].float(), lg.grad, rtol=1e-2, atol=1e-2 * lg.grad.abs().max().item())
    if ld > E:
        assert torch.count_nonzero(out[:, E:]) == 0


@pytest.mark.parametrize("E,M,T", [(16, 256, 1000), (128, 2048, 4096)])
def test_router_backward_gemms(hm, E, M, T):
    """dX_r = dlogits . Wr (fp32) and dWr += dlogits^T . x (fp32, accumulated)."""
    from paper_2508_09591_b200._lib import ptr, stream_ptr
    g = torch.Generator(device="cuda").manual_seed(3 * E)
    e128 = -(-E // 128) * 128
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(E, M, device="cuda", generator=g) * M ** -0.5).to(torch.bfloat16)
    dl = torch.zeros(T, e128, dtype=torch.bfloat16, device="cuda")
    dl[:, :E] = torch.randn(T, E, device="cuda", generator=g).to(torch.bfloat16)
    wt = torch.zeros(M, e128, dtype=torch.bfloat16, device="cuda")
    wt[:, :E] = w.T
    rows = torch.tensor([T], dtype=torch.int32, device="cuda")
    dx = torch.empty(T, M, device="cuda")
    _call("hm_gemm_f32", ptr(dl), T, ptr(rows), ptr(wt), M, e128, M, ptr(dx), M, stream_ptr())
    dwp = torch.ones(e128, M, device="cuda")          # accumulate onto 1.0
    _call("hm_wgrad_f32", ptr(dl), ptr(x), T, ptr(rows), e128, M, ptr(dwp), M, 1, stream_ptr())
    torch.cuda.synchronize()
    torch.testing.assert_close(dx, dl[:, :E].float() @ w.float(), rtol=1e-4, atol=1e-4)
    ref_w = 1.0 + dl[:, :E].float().T @ x.float()
    torch.testing.assert_close(dwp[:E], ref_w, rtol=1e-4, atol=1e-3)
    assert torch.equal(dwp[E:], torch.ones_like(dwp[E:]))


@pytest.mark.parametrize("valid", [4096, 3000, 200, 0])
def test_router_wgrad_split_k_device_count(hm, valid):
    """hm_wgrad_f32_split splits the token reduction into chunks sized on the device
    from the live row count: rows past the count (capacity 4096) never enter
    the gradient, empty chunks add zero, the accumulated value is kept."""
    from paper_2508_09591_b200._lib import ptr, stream_ptr
    g = torch.Generator(device="cuda").manual_seed(valid + 1)
    T, e128, M = 4096, 128, 2048
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    dl = torch.randn(T, e128, device="cuda", generator=g).to(torch.bfloat16)
    rows = torch.tensor([valid], dtype=torch.int32, device="cuda")
    dwp = torch.full((e128, M), 0.5, device="cuda")
    from paper_2508_09591_b200 import _lib
    need = int(_lib.load().hm_wgrad_f32_scratch_bytes(T, e128, M))
    assert need > 0
    with pytest.raises(ValueError):   # the split needs its scratch
        _call("hm_wgrad_f32_split", ptr(dl), ptr(x), T, ptr(rows), e128, M, ptr(dwp), M, 1,
              None, 0, stream_ptr())
    scratch = torch.empty(need, dtype=torch.uint8, device="cuda")
    _call("hm_wgrad_f32_split", ptr(dl), ptr(x), T, ptr(rows), e128, M, ptr(dwp), M, 1,
          ptr(scratch), need, stream_ptr())
    torch.cuda.synchronize()
    ref = 0.5 + dl[:valid].float().T @ x[:valid].float()
    torch.testing.assert_close(dwp, ref, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("T,shared", [(4096, True), (1000, False), (777, True)])
def test_router_dx_fused_sum_matches_separate(hm, T, shared):
    """hm_gemm_add_bf16 (router input gradient with the routed / shared dx
    added in the GEMM epilogue, one rounding) equals hm_gemm_f32 followed by
    hm_sum_to_bf16 bit for bit -- whole and partial 32-row blocks."""
    from paper_2508_09591_b200._lib import ptr, stream_ptr
    g = torch.Generator(device="cuda").manual_seed(T)
    E, M = 128, 2048
    dl = torch.randn(T, E, device="cuda", generator=g).to(torch.bfloat16)
    wt = (torch.randn(M, E, device="cuda", generator=g) * E ** -0.5).to(torch.bfloat16)
    dx = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    sdx = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16) if shared else None
    rows = torch.tensor([T], dtype=torch.int32, device="cuda")
    dxf = torch.empty(T, M, device="cuda")
    _call("hm_gemm_f32", ptr(dl), T, ptr(rows), ptr(wt), M, E, M, ptr(dxf), M, stream_ptr())
    ref = torch.empty(T, M, dtype=torch.bfloat16, device="cuda")
    _call("hm_sum_to_bf16", ptr(dxf), ptr(dx), ptr(sdx), ptr(ref), dx.numel(), stream_ptr())
    out = torch.empty(T, M, dtype=torch.bfloat16, device="cuda")
    _call("hm_gemm_add_bf16", ptr(dl), T, ptr(rows), ptr(wt), M, E, ptr(dx), ptr(sdx), ptr(out),
          M, stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
