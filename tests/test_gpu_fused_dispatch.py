"""Fused one-GPU dispatch: the dispatch emits expert-major row indices and
GEMM1 gathers its rows from the tokens with TMA gather4 (hm_expert_ffn_gather;
the backward's dW13 gathers likewise).  Everything downstream must be bit-
identical to the copying dispatch: forward outputs, input and weight grads."""

import numpy as np
import pytest
import torch

from oracle import moe as OM

pytestmark = pytest.mark.gpu


def test_index_dispatch_matches_plan(hm):
    """xidx[rank][epos[t, k]] == t for every pick (the expert-major layout of
    the copying dispatch, DispatchPlan.epos), with ragged / dropped picks."""
    from paper_2508_09591_b200.layer import EPWorld, route_topk
    G, E, K, M, T_r = 8, 64, 6, 256, 200
    g = torch.Generator().manual_seed(11)
    logits = torch.randn(G * T_r, E, generator=g)
    x = torch.randn(G * T_r, M, generator=g).to(torch.bfloat16).cuda()
    slot, w, _ = route_topk(logits.cuda(), K)
    world = EPWorld(G, E, K, M, T_r)
    world.set_fused(True)
    world.dispatch(x, slot, w, dedup="gpu")
    torch.cuda.synchronize()
    world.check_status()
    ids = slot.cpu().numpy()
    plan = OM.DispatchPlan(ids, G, E)
    epos = world.read("epos", 0, torch.int32).cpu().numpy().reshape(-1, K)
    assert np.array_equal(epos, plan.epos)
    e_loc = E // G
    for d in range(G):
        n = int(plan.n_e[d * e_loc:(d + 1) * e_loc].sum())
        idx = world.read("xidx", d, torch.int32, n).cpu().numpy()
        tt, kk = np.nonzero(ids // e_loc == d)
        assert np.array_equal(idx[plan.epos[tt, kk]], tt)
    world.close()


def _grouped_gather_vs_copy(hm, groups, rows_per_group, M, I, seed):
    from paper_2508_09591_b200 import _lib
    from paper_2508_09591_b200.ffn import expert_ffn_gather_ptrs, expert_ffn_ptrs, pack_w13
    g = torch.Generator(device="cuda").manual_seed(seed)
    T = 3000
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    n = torch.tensor(rows_per_group, dtype=torch.int32, device="cuda")
    total = int(n.sum())
    cap = total + 300
    idx = torch.randint(0, T, (cap,), device="cuda", generator=g, dtype=torch.int32)
    xm = torch.zeros(cap, M, dtype=torch.bfloat16, device="cuda")
    xm[:total] = x[idx[:total].long()]
    w1 = torch.randn(groups, I, M, device="cuda", generator=g) * M ** -0.5
    w3 = torch.randn(groups, I, M, device="cuda", generator=g) * M ** -0.5
    w13 = pack_w13(w1.to(torch.bfloat16), w3.to(torch.bfloat16)).contiguous()
    w2 = (torch.randn(groups, M, I, device="cuda", generator=g) * I ** -0.5).to(torch.bfloat16)
    outs = []
    for fused in (False, True):
        h = torch.zeros(cap, I, dtype=torch.bfloat16, device="cuda")
        y = torch.zeros(cap, M, dtype=torch.bfloat16, device="cuda")
        if fused:
            expert_ffn_gather_ptrs(x.data_ptr(), T, idx.data_ptr(), cap, n.data_ptr(), groups,
                                   w13, w2, M, I, h, y.data_ptr())
        else:
            expert_ffn_ptrs(xm.data_ptr(), cap, n.data_ptr(), groups, w13, w2, M, I, h,
                            y.data_ptr())
        torch.cuda.synchronize()
        outs.append((h[:total].clone(), y[:total].clone()))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("rows", [[300, 1, 0, 517, 256, 255], [4096] * 4, [7, 9, 11]])
def test_gather_gemm_equals_copied_rows(hm, rows):
    _grouped_gather_vs_copy(hm, len(rows), rows, 512, 256, seed=len(rows))


@pytest.mark.parametrize("shape,mb", [((8, 64, 6, 512, 256, 64), 1), ((8, 64, 6, 512, 256, 64), 2),
                                      ((8, 16, 2, 256, 256, 96), 1)])
def test_fused_layer_bit_identical(hm, shape, mb):
    from paper_2508_09591_b200.moe import HierMoELayer
    G, E, K, M, I, T_r = shape
    gen = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(G * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    gout = torch.randn(G * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    res = []
    for fused in (False, True):
        layer = HierMoELayer(G, E, K, M, I, T_r, seed=3, grad=True, micro_batches=mb,
                             fused_dispatch=fused, optimizer_state=False)
        out = layer(x).clone()
        dx = layer.backward(gout).clone()
        torch.cuda.synchronize()
        layer.check_status()
        res.append((out, dx, layer.dw13.clone(), layer.dw2.clone(), layer.dw_router.clone()))
        layer.close()
    for a, b in zip(*res):
        assert torch.equal(a, b)


def test_fused_layer_bit_identical_qwen3_full_size(hm):
    """BASELINE configs[1] at the bench's size (8 ranks x 4096 tokens, E=128,
    top-8, hidden 2048, I=768): fused == copying dispatch, forward and backward."""
    from paper_2508_09591_b200.moe import HierMoELayer
    G, E, K, M, I, T_r = 8, 128, 8, 2048, 768, 4096
    gen = torch.Generator(device="cuda").manual_seed(6)
    x = torch.randn(G * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    gout = torch.randn(G * T_r, M, device="cuda", generator=gen).to(torch.bfloat16)
    res = []
    for fused in (False, True):
        layer = HierMoELayer(G, E, K, M, I, T_r, seed=3, grad=True, fused_dispatch=fused,
                             optimizer_state=False, n_cap_rows=3 * T_r * K)
        out = layer(x).clone()
        dx = layer.backward(gout).clone()
        torch.cuda.synchronize()
        layer.check_status()
        res.append((out, dx, layer.dw13.clone(), layer.dw2.clone()))
        layer.close()
        torch.cuda.empty_cache()
    for a, b in zip(*res):
        assert torch.equal(a, b)
