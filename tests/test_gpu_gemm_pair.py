"""CTA-pair (tcgen05 cta_group::2, 256 x 256 tile) grouped GEMMs vs the
single-CTA kernels: identical bits (same per-element k order), and vs an fp32
reference; forward SwiGLU with the stored pre-activations included."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture
def pair():
    from paper_2508_09591_b200.ffn import set_gemm_pair
    yield set_gemm_pair
    set_gemm_pair(True)   # the library default


@pytest.mark.parametrize("n_rows,N,K", [
    ([128], 256, 64),
    ([300, 0, 77, 513], 512, 256),
    ([1, 129, 255, 256, 257], 256, 2048),
    ([2048] * 4, 2048, 768),
])
def test_pair_gemm_equals_single(hm, pair, n_rows, N, K):
    from paper_2508_09591_b200.ffn import grouped_gemm
    torch.manual_seed(0)
    G = len(n_rows)
    rows = sum(n_rows)
    a = torch.randn(max(rows, 1) + 300, K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(G, N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
    nr = torch.tensor(n_rows, dtype=torch.int32, device="cuda")
    pair(False)
    one = grouped_gemm(a, b, nr)
    pair(True)
    two = grouped_gemm(a, b, nr)
    torch.cuda.synchronize()
    assert torch.equal(one[:rows], two[:rows])
    r, refs = 0, []
    for g, n in enumerate(n_rows):
        refs.append(a[r:r + n].float() @ b[g].float().T)
        r += n
    torch.testing.assert_close(two[:rows].float(), torch.cat(refs), rtol=2e-2, atol=2e-2)


def test_pair_swiglu_ffn_equals_single(hm, pair):
    from paper_2508_09591_b200.ffn import expert_ffn_save_ptrs
    torch.manual_seed(2)
    G, M, I = 5, 512, 512
    n_rows = [700, 0, 129, 1000, 64]
    cap = sum(n_rows) + 256
    x = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    nr = torch.tensor(n_rows, dtype=torch.int32, device="cuda")
    res = []
    for on in (False, True):
        pair(on)
        h = torch.empty(cap, I, device="cuda", dtype=torch.bfloat16)
        y = torch.empty(cap, M, device="cuda", dtype=torch.bfloat16)
        g13 = torch.empty(cap, 2 * I, device="cuda", dtype=torch.bfloat16)
        expert_ffn_save_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h, y.data_ptr(),
                             g13.data_ptr())
        torch.cuda.synchronize()
        rows = sum(n_rows)
        res.append((h[:rows].clone(), y[:rows].clone(), g13[:rows].clone()))
    for a, b in zip(*res):
        assert torch.equal(a, b)


@pytest.mark.parametrize("shape", [(4, 2048, 768, [1000, 63, 0, 2049]), (3, 512, 256, [130, 0, 301])])
def test_wgrad_pair_equals_single(hm, shape):
    """Weight gradients from both CTA-pair MN-major GEMMs equal the single-CTA
    ones bit for bit (rows past the last group hold NaN: the tail zeroing /
    the per-group maps' zero fill must keep them out)."""
    from paper_2508_09591_b200.ffn import (FFNBackwardScratch, expert_ffn_backward_ptrs,
                                           expert_ffn_save_ptrs, set_wgrad_pair)
    G, M, I, n_rows = shape
    torch.manual_seed(7)
    rows = sum(n_rows)
    cap = rows + 100
    x = torch.full((cap, M), float("nan"), device="cuda", dtype=torch.bfloat16)
    x[:rows] = torch.randn(rows, M, device="cuda").to(torch.bfloat16)
    gy = torch.full((cap, M), float("nan"), device="cuda", dtype=torch.bfloat16)
    gy[:rows] = torch.randn(rows, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    w13t, w2t = w13.transpose(1, 2).contiguous(), w2.transpose(1, 2).contiguous()
    nr = torch.tensor(n_rows, dtype=torch.int32, device="cuda")
    h = torch.empty(cap, I, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(cap, M, device="cuda", dtype=torch.bfloat16)
    g13 = torch.empty(cap, 2 * I, device="cuda", dtype=torch.bfloat16)
    expert_ffn_save_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h, y.data_ptr(),
                         g13.data_ptr())
    res = []
    try:
        for on in (0, 1, 2):   # single CTA, pair with hand-off, pair with per-group maps
            set_wgrad_pair(on)
            sc = FFNBackwardScratch(cap, G, M, I)
            gx = torch.zeros(cap, M, device="cuda", dtype=torch.bfloat16)
            dw13 = torch.empty(G, 2 * I, M, device="cuda", dtype=torch.bfloat16)
            dw2 = torch.empty(G, M, I, device="cuda", dtype=torch.bfloat16)
            expert_ffn_backward_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w13t, w2t,
                                     gy.data_ptr(), M, I, sc, gx.data_ptr(), dw13, dw2,
                                     g13.data_ptr())
            torch.cuda.synchronize()
            res.append((dw13.clone(), dw2.clone()))
    finally:
        set_wgrad_pair(False)
    for other in res[1:]:
        assert not torch.isnan(other[0]).any() and not torch.isnan(other[1]).any()
        assert torch.equal(res[0][0], other[0])
        assert torch.equal(res[0][1], other[1])


@pytest.mark.parametrize("shape", [(4, 2048, 768, [1000, 63, 0, 2049]), (3, 512, 256, [130, 0, 301])])
def test_swiglu_bwd_vector_equals_scalar(hm, shape):
    """The 16-byte SwiGLU backward (default) and the 4-byte one give the same
    data and weight gradients bit for bit."""
    from paper_2508_09591_b200.ffn import (FFNBackwardScratch, expert_ffn_backward_ptrs,
                                           expert_ffn_save_ptrs, set_swiglu_scalar)
    G, M, I, n_rows = shape
    torch.manual_seed(11)
    rows = sum(n_rows)
    cap = rows + 100
    x = torch.zeros(cap, M, device="cuda", dtype=torch.bfloat16)
    x[:rows] = torch.randn(rows, M, device="cuda").to(torch.bfloat16)
    gy = torch.zeros(cap, M, device="cuda", dtype=torch.bfloat16)
    gy[:rows] = torch.randn(rows, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    w13t, w2t = w13.transpose(1, 2).contiguous(), w2.transpose(1, 2).contiguous()
    nr = torch.tensor(n_rows, dtype=torch.int32, device="cuda")
    h = torch.empty(cap, I, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(cap, M, device="cuda", dtype=torch.bfloat16)
    g13 = torch.empty(cap, 2 * I, device="cuda", dtype=torch.bfloat16)
    expert_ffn_save_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h, y.data_ptr(),
                         g13.data_ptr())
    res = []
    try:
        for scalar in (True, False):
            set_swiglu_scalar(scalar)
            sc = FFNBackwardScratch(cap, G, M, I)
            gx = torch.zeros(cap, M, device="cuda", dtype=torch.bfloat16)
            dw13 = torch.empty(G, 2 * I, M, device="cuda", dtype=torch.bfloat16)
            dw2 = torch.empty(G, M, I, device="cuda", dtype=torch.bfloat16)
            expert_ffn_backward_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w13t, w2t,
                                     gy.data_ptr(), M, I, sc, gx.data_ptr(), dw13, dw2,
                                     g13.data_ptr())
            torch.cuda.synchronize()
            res.append((gx[:rows].clone(), dw13.clone(), dw2.clone()))
    finally:
        set_swiglu_scalar(False)
    for a, b in zip(*res):
        assert torch.equal(a, b)
