"""tcgen05 grouped GEMM / expert SwiGLU FFN vs a plain PyTorch fp32 reference
(bf16 operands, fp32 accumulation; tolerance: bf16 output rounding)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref_gemm(a, b, n_rows):
    out, r = [], 0
    for g, n in enumerate(n_rows):
        out.append(a[r:r + n].float() @ b[g].float().T)
        r += n
    return torch.cat(out) if out else a.new_zeros((0, b.shape[1]), dtype=torch.float32)


@pytest.mark.parametrize("n_rows,N,K", [
    ([128], 256, 64),
    ([300, 0, 77, 513], 512, 256),
    ([1, 129, 255, 256, 257], 256, 2048),
    ([2048] * 4, 2048, 768),
])
def test_grouped_gemm_matches_fp32(hm, n_rows, N, K):
    from paper_2508_09591_b200.ffn import grouped_gemm
    torch.manual_seed(0)
    G = len(n_rows)
    rows = sum(n_rows)
    a = torch.randn(max(rows, 1), K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(G, N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
    nr = torch.tensor(n_rows, dtype=torch.int32, device="cuda")
    out = grouped_gemm(a, b, nr)
    torch.cuda.synchronize()
    ref = _ref_gemm(a, b, n_rows)
    torch.testing.assert_close(out[:rows].float(), ref, rtol=2e-2, atol=2e-2)


def test_swiglu_ffn_matches_fp32(hm):
    from paper_2508_09591_b200.ffn import expert_ffn_ptrs, pack_w13
    torch.manual_seed(1)
    G, M, I = 4, 2048, 768
    n_rows = [700, 0, 1500, 333]
    rows = sum(n_rows)
    x = torch.randn(rows, M, device="cuda").to(torch.bfloat16)
    w1 = (torch.randn(G, I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w3 = (torch.randn(G, I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    w13 = pack_w13(w1, w3)
    h = torch.empty(rows, I, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(rows, M, dtype=torch.bfloat16, device="cuda")
    nr = torch.tensor(n_rows, dtype=torch.int32, device="cuda")
    expert_ffn_ptrs(x.data_ptr(), rows, nr.data_ptr(), G, w13, w2, M, I, h, y.data_ptr())
    torch.cuda.synchronize()
    refs, r = [], 0
    for g, n in enumerate(n_rows):
        xs = x[r:r + n].float()
        hh = torch.nn.functional.silu(xs @ w1[g].float().T) * (xs @ w3[g].float().T)
        refs.append(hh.to(torch.bfloat16).float() @ w2[g].float().T)
        r += n
    ref = torch.cat(refs)
    torch.testing.assert_close(y.float(), ref, rtol=3e-2, atol=3e-2)


@pytest.mark.parametrize("G,M,I,n_rows", [(3, 256, 256, [100, 0, 257]),
                                          (4, 2048, 768, [1000, 63, 0, 2049])],
                         ids=["small", "qwen3_expert"])
def test_swiglu_ffn_backward_matches_autograd(hm, G, M, I, n_rows):
    """tcgen05 FFN backward (dgrad + MN-major weight grads) vs torch autograd
    in fp32.  Rows past the last group hold NaN: the weight-gradient GEMMs
    must not read past a group's own rows (zeroed tail k-block)."""
    from paper_2508_09591_b200.ffn import (FFNBackwardScratch, expert_ffn_backward_ptrs,
                                           pack_w13)
    torch.manual_seed(4)
    rows = sum(n_rows)
    cap = rows + 40
    x = torch.full((cap, M), float("nan"), device="cuda", dtype=torch.bfloat16)
    x[:rows] = torch.randn(rows, M, device="cuda").to(torch.bfloat16)
    gy = torch.full((cap, M), float("nan"), device="cuda", dtype=torch.bfloat16)
    gy[:rows] = torch.randn(rows, M, device="cuda").to(torch.bfloat16)
    w1 = (torch.randn(G, I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w3 = (torch.randn(G, I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    w13 = pack_w13(w1, w3)
    nr = torch.tensor(n_rows, dtype=torch.int32, device="cuda")
    sc = FFNBackwardScratch(cap, G, M, I)
    gx = torch.zeros(cap, M, device="cuda", dtype=torch.bfloat16)
    dw13 = torch.empty(G, 2 * I, M, device="cuda", dtype=torch.bfloat16)
    dw2 = torch.empty(G, M, I, device="cuda", dtype=torch.bfloat16)
    expert_ffn_backward_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, gy.data_ptr(),
                             M, I, sc, gx.data_ptr(), dw13, dw2)
    torch.cuda.synchronize()
    r = 0
    for g, n in enumerate(n_rows):
        xs = x[r:r + n].float().requires_grad_(True)
        a1 = w1[g].float().requires_grad_(True)
        a3 = w3[g].float().requires_grad_(True)
        b2 = w2[g].float().requires_grad_(True)
        y = (torch.nn.functional.silu(xs @ a1.T) * (xs @ a3.T)) @ b2.T
        y.backward(gy[r:r + n].float())
        torch.testing.assert_close(gx[r:r + n].float(), xs.grad, rtol=3e-2, atol=3e-2)
        d13 = pack_w13(a1.grad[None], a3.grad[None])[0]
        torch.testing.assert_close(dw13[g].float(), d13, rtol=3e-2, atol=3e-2 * max(1.0, d13.abs().max().item()))
        torch.testing.assert_close(dw2[g].float(), b2.grad, rtol=3e-2, atol=3e-2 * max(1.0, b2.grad.abs().max().item()))
        r += n


def test_saved_preactivations_match_recompute(hm):
    """Training forward's stored pre-activations + backward without recompute
    == backward with the GEMM1 recompute (bit for bit)."""
    from paper_2508_09591_b200.ffn import (FFNBackwardScratch, expert_ffn_backward_ptrs,
                                           expert_ffn_ptrs, expert_ffn_save_ptrs)
    torch.manual_seed(6)
    G, M, I = 3, 512, 256
    n_rows = [130, 0, 300]
    cap = sum(n_rows) + 20
    x = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    gy = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    nr = torch.tensor(n_rows, dtype=torch.int32, device="cuda")
    h = torch.empty(cap, I, device="cuda", dtype=torch.bfloat16)
    y0 = torch.empty(cap, M, device="cuda", dtype=torch.bfloat16)
    y1 = torch.empty_like(y0)
    g13 = torch.empty(cap, 2 * I, device="cuda", dtype=torch.bfloat16)
    expert_ffn_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h, y0.data_ptr())
    expert_ffn_save_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h, y1.data_ptr(),
                         g13.data_ptr())
    rows = sum(n_rows)
    assert torch.equal(y0[:rows], y1[:rows])
    res = []
    for saved in (0, g13.data_ptr()):
        sc = FFNBackwardScratch(cap, G, M, I)
        gx = torch.zeros(cap, M, device="cuda", dtype=torch.bfloat16)
        dw13 = torch.empty(G, 2 * I, M, device="cuda", dtype=torch.bfloat16)
        dw2 = torch.empty(G, M, I, device="cuda", dtype=torch.bfloat16)
        expert_ffn_backward_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2,
                                 gy.data_ptr(), M, I, sc, gx.data_ptr(), dw13, dw2, saved)
        torch.cuda.synchronize()
        res.append((gx[:rows].clone(), dw13.clone(), dw2.clone()))
    for a, b in zip(*res):
        assert torch.equal(a, b)


def test_multi_segment_ffn_equals_per_rank(hm):
    """One launch per GEMM over several EP ranks' expert groups (row segments
    [s * seg_rows, ...)) gives bit-identical forward outputs, pre-activations,
    input grads and weight grads to one launch per rank."""
    from paper_2508_09591_b200.ffn import (FFNBackwardScratch, expert_ffn_backward_multi_ptrs,
                                           expert_ffn_backward_ptrs, expert_ffn_multi_ptrs,
                                           expert_ffn_save_ptrs)
    torch.manual_seed(12)
    S, Gs, M, I, cap = 3, 4, 512, 256, 1500
    n = torch.randint(0, 350, (S * Gs,), dtype=torch.int32)
    n[5] = 0
    nr = n.cuda()
    x = torch.randn(S, cap, M, device="cuda").to(torch.bfloat16)
    gy = torch.randn(S, cap, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(S, Gs, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(S, Gs, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    outs = []
    for multi in (False, True):
        h = torch.zeros(S * cap, I, dtype=torch.bfloat16, device="cuda")
        y = torch.zeros(S, cap, M, dtype=torch.bfloat16, device="cuda")
        g13 = torch.zeros(S, cap, 2 * I, dtype=torch.bfloat16, device="cuda")
        gx = torch.zeros(S, cap, M, dtype=torch.bfloat16, device="cuda")
        dw13 = torch.zeros_like(w13)
        dw2 = torch.zeros_like(w2)
        if multi:
            sc = FFNBackwardScratch(S * cap, S * Gs, M, I)
            expert_ffn_multi_ptrs(x.data_ptr(), S * cap, 0, cap, S, nr.data_ptr(), Gs, w13, w2,
                                  M, I, h, y.data_ptr(), g13.data_ptr())
            expert_ffn_backward_multi_ptrs(x.data_ptr(), S * cap, 0, cap, S, nr.data_ptr(), Gs,
                                           w13, w2, gy.data_ptr(), M, I, sc, gx.data_ptr(),
                                           dw13, dw2, g13.data_ptr())
        else:
            for s in range(S):
                sc = FFNBackwardScratch(cap, Gs, M, I)
                hs = torch.zeros(cap, I, dtype=torch.bfloat16, device="cuda")
                np_ = nr[s * Gs:].data_ptr()
                expert_ffn_save_ptrs(x[s].data_ptr(), cap, np_, Gs, w13[s], w2[s], M, I, hs,
                                     y[s].data_ptr(), g13[s].data_ptr())
                expert_ffn_backward_ptrs(x[s].data_ptr(), cap, np_, Gs, w13[s], w2[s],
                                         gy[s].data_ptr(), M, I, sc, gx[s].data_ptr(), dw13[s],
                                         dw2[s], g13[s].data_ptr())
        torch.cuda.synchronize()
        used = [int(n[s * Gs:(s + 1) * Gs].sum()) for s in range(S)]
        outs.append([torch.cat([t[s, :used[s]] for s in range(S)]) for t in (y, g13, gx)]
                    + [dw13.clone(), dw2.clone()])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_ffn_explicit_groups_match_segments(hm):
    """hm_expert_ffn_groups (explicit row start / count / weight index per
    group, the overlapped forward's split) gives the rows the same bits as the
    segment-layout launch, with every expert split at an arbitrary row into
    two groups, and the groups listed out of order with empty ones."""
    from paper_2508_09591_b200 import _lib
    from paper_2508_09591_b200._lib import ptr, stream_ptr
    from paper_2508_09591_b200.ffn import expert_ffn_multi_ptrs
    torch.manual_seed(21)
    S, Gs, M, I, cap = 2, 4, 512, 256, 1400
    n = torch.randint(0, 330, (S * Gs,), dtype=torch.int32)
    n[3] = 0
    nr = n.cuda()
    x = torch.randn(S * cap, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(S * Gs, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(S * Gs, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    outs = []
    for explicit in (False, True):
        h = torch.zeros(S * cap, I, dtype=torch.bfloat16, device="cuda")
        y = torch.zeros(S * cap, M, dtype=torch.bfloat16, device="cuda")
        g13 = torch.zeros(S * cap, 2 * I, dtype=torch.bfloat16, device="cuda")
        if not explicit:
            expert_ffn_multi_ptrs(x.data_ptr(), S * cap, 0, cap, S, nr.data_ptr(), Gs, w13, w2,
                                  M, I, h, y.data_ptr(), g13.data_ptr())
        else:
            row0, rows, wsel = [], [], []
            for s in range(S):
                base = s * cap
                for j in range(Gs):
                    e = s * Gs + j
                    ne = int(n[e])
                    cut = ne // 3 if ne else 0
                    row0 += [base + cut, base]          # second part first
                    rows += [ne - cut, cut]
                    wsel += [e, e]
                    base += ne
            g = len(rows)
            t = lambda v: torch.tensor(v, dtype=torch.int32, device="cuda")  # noqa: E731
            r0, rc, ws = t(row0), t(rows), t(wsel)
            _lib.call("hm_expert_ffn_groups", ptr(x), S * cap, None, None, S * cap, g, ptr(r0),
                      ptr(rc), ptr(ws), S * Gs, ptr(w13), ptr(w2), M, I, ptr(h), ptr(y),
                      ptr(g13), 0, stream_ptr())
        torch.cuda.synchronize()
        used = [(s * cap, s * cap + int(n[s * Gs:(s + 1) * Gs].sum())) for s in range(S)]
        outs.append([torch.cat([v[a:b] for a, b in used]) for v in (h, y, g13)])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("gathered", [False, True])
def test_wgrad_pair_matches_single_cta(hm, gathered):
    """The CTA-pair weight-gradient kernel (256 x 256 tiles, both operands
    MN-major, tail tokens zeroed by the forwarder warp) gives dW13 / dW2 bit
    for bit equal to the single-CTA kernel -- ragged groups, an empty group,
    sizes off the 16-token MMA step -- with and without the gathered x rows."""
    from paper_2508_09591_b200 import _lib
    from paper_2508_09591_b200.ffn import (FFNBackwardScratch, expert_ffn_backward_gather_ptrs,
                                           expert_ffn_backward_ptrs, expert_ffn_save_ptrs)
    torch.manual_seed(33)
    G, M, I = 5, 512, 256
    n = torch.tensor([300, 0, 77, 513, 129], dtype=torch.int32)
    rows = int(n.sum())
    cap = rows + 64
    nr = n.cuda()
    x = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    gy = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    h = torch.zeros(cap, I, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(cap, M, dtype=torch.bfloat16, device="cuda")
    g13 = torch.zeros(cap, 2 * I, dtype=torch.bfloat16, device="cuda")
    expert_ffn_save_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h, y.data_ptr(),
                         g13.data_ptr())
    perm = torch.randperm(cap, device="cuda").to(torch.int32)   # gathered: x_src[perm[r]] = x[r]
    outs = []
    for pair in (0, 1):
        _lib.call("hm_ffn_set_option", 2, pair)
        sc = FFNBackwardScratch(cap, G, M, I)
        gx = torch.zeros(cap, M, dtype=torch.bfloat16, device="cuda")
        dw13, dw2 = torch.zeros_like(w13), torch.zeros_like(w2)
        if gathered:
            # x_src row perm[r] holds layout row r's activations
            x_src = torch.empty_like(x)
            x_src[perm.long()] = x
            expert_ffn_backward_gather_ptrs(x_src.data_ptr(), cap, perm.data_ptr(), cap,
                                            nr.data_ptr(), G, w13, w2, gy.data_ptr(), M, I, sc,
                                            gx.data_ptr(), dw13, dw2, g13.data_ptr())
        else:
            expert_ffn_backward_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, gy.data_ptr(),
                                     M, I, sc, gx.data_ptr(), dw13, dw2, g13.data_ptr())
        torch.cuda.synchronize()
        outs.append((dw13.clone(), dw2.clone(), gx.clone()))
    _lib.call("hm_ffn_set_option", 2, 1)
    assert torch.equal(outs[0][0], outs[1][0]), "dW13"
    assert torch.equal(outs[0][1], outs[1][1]), "dW2"
    assert torch.equal(outs[0][2], outs[1][2]), "gX"
    assert torch.count_nonzero(outs[1][0][1]) == 0      # empty group: zero gradient


@pytest.mark.parametrize("shape", [(5, 512, 256, [300, 0, 77, 513, 129]),
                                   (3, 512, 128, [1, 260, 511]),
                                   (4, 1024, 512, [700, 33, 0, 1030])])
def test_wide_tiles_match_256_tiles(hm, shape):
    """256 x 512 pair tiles (two accumulators sharing the A half, the epilogue
    releasing them one at a time, the next tile's first k-blocks run on
    accumulator 0 while accumulator 1 drains) give the forward (plain,
    SwiGLU with saved pre-activations, gathered A rows) and the backward bit
    for bit equal to 256 x 256 tiles -- ragged and empty groups, a
    single-k-block reduction (hidden 64), partial row tiles."""
    from paper_2508_09591_b200 import _lib
    from paper_2508_09591_b200.ffn import (FFNBackwardScratch, expert_ffn_backward_ptrs,
                                           expert_ffn_gather_ptrs, expert_ffn_save_ptrs)
    G, M, I, sizes = shape
    torch.manual_seed(44)
    n = torch.tensor(sizes, dtype=torch.int32)
    rows = int(n.sum())
    cap = rows + 64
    nr = n.cuda()
    x = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    gy = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    perm = torch.randperm(cap, device="cuda").to(torch.int32)
    x_src = torch.empty_like(x)
    x_src[perm.long()] = x
    outs = []
    try:
        for wide in (0, 2):   # 256 x 256 only / 256 x 512 wherever N allows
            _lib.call("hm_ffn_set_option", 5, wide)
            h = torch.zeros(cap, I, dtype=torch.bfloat16, device="cuda")
            y = torch.zeros(cap, M, dtype=torch.bfloat16, device="cuda")
            g13 = torch.zeros(cap, 2 * I, dtype=torch.bfloat16, device="cuda")
            expert_ffn_save_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h,
                                 y.data_ptr(), g13.data_ptr())
            hg = torch.zeros_like(h)
            yg = torch.zeros_like(y)
            expert_ffn_gather_ptrs(x_src.data_ptr(), cap, perm.data_ptr(), cap, nr.data_ptr(), G,
                                   w13, w2, M, I, hg, yg.data_ptr())
            gx = torch.zeros(cap, M, dtype=torch.bfloat16, device="cuda")
            dw13, dw2 = torch.zeros_like(w13), torch.zeros_like(w2)
            if I % 256 == 0:   # the backward's dH GEMM needs N = I in 256-column tiles
                sc = FFNBackwardScratch(cap, G, M, I)
                expert_ffn_backward_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2,
                                         gy.data_ptr(), M, I, sc, gx.data_ptr(), dw13, dw2,
                                         g13.data_ptr())
            torch.cuda.synchronize()
            outs.append([t[:rows].clone() for t in (h, y, g13, hg, yg, gx)] +
                        [dw13.clone(), dw2.clone()])
    finally:
        _lib.call("hm_ffn_set_option", 5, 1)
    names = ["h", "y", "g13", "h (gathered)", "y (gathered)", "gX", "dW13", "dW2"]
    for name, a, b in zip(names, outs[0], outs[1]):
        assert torch.equal(a, b), name
    # and the wide forward is right, not just self-consistent
    ref_rows = []
    r0 = 0
    for g in range(G):
        xs = x[r0:r0 + sizes[g]].float()
        a13 = xs @ w13[g].float().t()
        blk = a13.view(-1, I // 128, 2, 128)
        hh = torch.nn.functional.silu(blk[:, :, 0]) * blk[:, :, 1]
        ref_rows.append(hh.reshape(-1, I))
        r0 += sizes[g]
    torch.testing.assert_close(outs[1][0].float(), torch.cat(ref_rows), rtol=2e-2, atol=2e-2)



@pytest.mark.parametrize("shape", [(5, 512, 256, [300, 0, 77, 513, 129]),
                                   (3, 1024, 512, [31, 700, 96])])
def test_tma_store_epilogue_matches_lsu_stores(hm, shape):
    """GEMM2 / dH / gX epilogues with whole 32-row blocks leaving through TMA
    tensor stores (partial blocks at group ends through LSU stores) write the
    same rows bit for bit as the all-LSU epilogue -- and nothing past a group."""
    from paper_2508_09591_b200 import _lib
    from paper_2508_09591_b200.ffn import (FFNBackwardScratch, expert_ffn_backward_ptrs,
                                           expert_ffn_save_ptrs)
    G, M, I, sizes = shape
    torch.manual_seed(66)
    n = torch.tensor(sizes, dtype=torch.int32)
    rows = int(n.sum())
    cap = rows + 64
    nr = n.cuda()
    x = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    gy = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    outs = []
    try:
        for tma in (0, 1):
            _lib.call("hm_ffn_set_option", 6, tma)
            h = torch.zeros(cap, I, dtype=torch.bfloat16, device="cuda")
            y = torch.full((cap, M), 7.0, dtype=torch.bfloat16, device="cuda")
            g13 = torch.zeros(cap, 2 * I, dtype=torch.bfloat16, device="cuda")
            expert_ffn_save_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, M, I, h,
                                 y.data_ptr(), g13.data_ptr())
            sc = FFNBackwardScratch(cap, G, M, I)
            gx = torch.full((cap, M), 7.0, dtype=torch.bfloat16, device="cuda")
            dw13, dw2 = torch.zeros_like(w13), torch.zeros_like(w2)
            expert_ffn_backward_ptrs(x.data_ptr(), cap, nr.data_ptr(), G, w13, w2, gy.data_ptr(),
                                     M, I, sc, gx.data_ptr(), dw13, dw2, g13.data_ptr())
            torch.cuda.synchronize()
            outs.append((y.clone(), gx.clone(), dw13.clone(), dw2.clone(), sc.dh[:rows].clone()))
    finally:
        _lib.call("hm_ffn_set_option", 6, 1)
    for name, a, b in zip(["y", "gX", "dW13", "dW2", "dH"], outs[0], outs[1]):
        assert torch.equal(a, b), name
    # rows past the last group are never written
    assert torch.all(outs[1][0][rows:] == 7.0) and torch.all(outs[1][1][rows:] == 7.0)


def test_backward_with_forward_h_matches_recompute(hm):
    """Backward part bit 4 (h = the forward's H, not rewritten; dW2 from it)
    gives gX / dW13 / dW2 / dG13 bit for bit equal to the recomputing
    backward when handed the same H, and leaves that H untouched."""
    from paper_2508_09591_b200.ffn import FFNBackwardScratch, expert_ffn_backward_multi_ptrs
    from paper_2508_09591_b200.ffn import expert_ffn_multi_ptrs
    torch.manual_seed(77)
    G, M, I = 4, 512, 256
    n = torch.tensor([300, 0, 77, 257], dtype=torch.int32)
    cap = 704
    nr = n.cuda()
    x = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    gy = torch.randn(cap, M, device="cuda").to(torch.bfloat16)
    w13 = (torch.randn(G, 2 * I, M, device="cuda") * M ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(G, M, I, device="cuda") * I ** -0.5).to(torch.bfloat16)
    idx = torch.arange(cap, dtype=torch.int32, device="cuda")
    h = torch.zeros(cap, I, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(cap, M, dtype=torch.bfloat16, device="cuda")
    g13 = torch.zeros(cap, 2 * I, dtype=torch.bfloat16, device="cuda")
    expert_ffn_multi_ptrs(x.data_ptr(), cap, idx.data_ptr(), cap, 1, nr.data_ptr(), G, w13, w2,
                          M, I, h, y.data_ptr(), g13.data_ptr())
    outs = []
    h_given = None
    for use_fwd in (False, True):
        sc = FFNBackwardScratch(cap, G, M, I)
        gx = torch.zeros(cap, M, dtype=torch.bfloat16, device="cuda")
        dw13, dw2 = torch.zeros_like(w13), torch.zeros_like(w2)
        expert_ffn_backward_multi_ptrs(x.data_ptr(), cap, idx.data_ptr(), cap, 1, nr.data_ptr(),
                                       G, w13, w2, gy.data_ptr(), M, I, sc, gx.data_ptr(), dw13,
                                       dw2, g13.data_ptr(),
                                       h_fwd=h_given if use_fwd else None)
        torch.cuda.synchronize()
        outs.append((gx.clone(), dw13.clone(), dw2.clone(), sc.dg13[:int(n.sum())].clone()))
        if not use_fwd:
            h_given = sc.h.clone()          # the recomputed H, handed in as "the forward's"
            h_keep = h_given.clone()
    for name, a, b in zip(["gX", "dW13", "dW2", "dG13"], outs[0], outs[1]):
        assert torch.equal(a, b), name
    assert torch.equal(h_given, h_keep), "the forward's H is not rewritten"
