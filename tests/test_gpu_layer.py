"""GPU parity of the MoE-layer hot path (gating, dedup dispatch, combine)
against the CPU restatement in oracle/moe.py.

Bit-exact: routing indices, per-destination counts (== dedup_counts /
raw_counts at G, traffic.py:67-82), receive order (== propagate_level copy
order restricted to each destination, routing.py:204-215), every moved row.
Tolerances (BASELINE north star): fp32 rtol 1e-5, bf16 rtol 2e-2.
"""

import zlib

import numpy as np
import pytest
import torch

from oracle import moe as OM

pytestmark = pytest.mark.gpu

CONFIGS = {
    # name: (G, E, K, M, T_r, dtype)
    "configA_fp32": (8, 16, 2, 256, 512, torch.float32),
    "configA_bf16": (8, 16, 2, 256, 512, torch.bfloat16),
    "qwen3_small": (8, 128, 8, 2048, 256, torch.bfloat16),
    "dsv3_small": (8, 256, 8, 512, 128, torch.bfloat16),
    "ragged_tokens": (8, 64, 6, 128, 77, torch.float32),
}


def _inputs(G, E, K, M, T_r, dtype, seed=0, skew=0.0):
    g = torch.Generator().manual_seed(seed)
    T = G * T_r
    logits = torch.randn(T, E, generator=g, dtype=torch.float32)
    if skew:
        logits += skew * torch.linspace(2, -2, E)[torch.randperm(E, generator=g)]
    logits[::7, 3] = logits[::7, 5]          # exact ties exercise index-ascending order
    x = torch.randn(T, M, generator=g, dtype=torch.float32).to(dtype)
    return logits, x


def test_route_topk_matches_oracle(hm):
    from paper_2508_09591_b200.layer import route_topk
    for E, K in ((16, 2), (128, 8), (256, 8), (64, 6)):
        logits, _ = _inputs(1, E, K, 16, 1000, torch.float32, seed=E)
        perm = torch.randperm(E, generator=torch.Generator().manual_seed(1)).to(torch.int32)
        slot, w, ex = route_topk(logits.cuda(), K, perm.cuda())
        o_slot, o_w, o_ex = OM.route_topk(logits.numpy(), K, perm.numpy())
        assert np.array_equal(ex.cpu().numpy(), o_ex)
        assert np.array_equal(slot.cpu().numpy(), o_slot)
        np.testing.assert_allclose(w.cpu().numpy(), o_w, rtol=1e-5, atol=1e-7)
        slot2, w2, _ = route_topk(logits.cuda(), K, None, renormalize=False)
        _, o_w2, _ = OM.route_topk(logits.numpy(), K, None, renormalize=False)
        np.testing.assert_allclose(w2.cpu().numpy(), o_w2, rtol=1e-5, atol=1e-7)


def _world(hm, G, E, K, M, T_r, dtype):
    from paper_2508_09591_b200.layer import EPWorld
    return EPWorld(ranks=G, experts=E, top_k=K, hidden=M, tokens_per_rank=T_r, dtype=dtype)


def _scale(E):
    return 1.0 + torch.arange(E, dtype=torch.float64) / E


def _apply_experts(world, plan, E, dtype):
    """Stand-in expert: y = x * scale[slot] on every expert-major row."""
    e_loc = E // world.ranks
    sc = _scale(E)
    for d in range(world.ranks):
        n = int(plan.n_e[d * e_loc:(d + 1) * e_loc].sum())
        xm = world.read("xmaj", d, dtype, n * world.hidden).view(n, world.hidden)
        row_slot = np.repeat(np.arange(d * e_loc, (d + 1) * e_loc), plan.n_e[d * e_loc:(d + 1) * e_loc])
        s = sc[row_slot].to(torch.float32).cuda()[:, None]
        world.set_expert_outputs(d, (xm.float() * s).to(dtype))


@pytest.mark.parametrize("name", list(CONFIGS))
@pytest.mark.parametrize("dedup", ["all", "remote", "gpu", "none"])
def test_dispatch_combine_parity(hm, name, dedup):
    _parity(hm, name, CONFIGS[name], dedup)


# BASELINE configs[1] / configs[2] at the bench's full size: 8 ranks x 4096
# tokens, hidden 2048 (Qwen3) and 7168 (DeepSeek-V3)
FULL = {
    "qwen3_full": (8, 128, 8, 2048, 4096, torch.bfloat16),
    "dsv3_full": (8, 256, 8, 7168, 4096, torch.bfloat16),
}


@pytest.mark.parametrize("name,dedup", [("qwen3_full", "gpu"), ("qwen3_full", "none"),
                                        ("qwen3_full", "all"), ("dsv3_full", "gpu"),
                                        ("dsv3_full", "all")])
def test_dispatch_combine_parity_full_size(hm, name, dedup):
    _parity(hm, name, FULL[name], dedup)


def _parity(hm, name, cfg, dedup):
    from paper_2508_09591_b200.layer import route_topk
    G, E, K, M, T_r, dtype = cfg
    logits, x = _inputs(G, E, K, M, T_r, dtype, seed=zlib.crc32(name.encode()) % 1000)
    slot, w, _ = route_topk(logits.cuda(), K)
    world = _world(hm, G, E, K, M, T_r, dtype)
    xd = x.cuda()
    world.dispatch(xd, slot, w, dedup=dedup)
    torch.cuda.synchronize()
    world.check_status()
    ids = slot.cpu().numpy()
    plan = OM.DispatchPlan(ids, G, E)
    cnt = world.counts()
    assert np.array_equal(cnt[:, :G], plan.h)           # dedup rows per (src, dest)
    assert np.array_equal(cnt[:, G:], plan.c)           # selections per (src, slot)
    rn = world.rows_received()
    # one GPU: "remote" ships no dedup rows (every rank shares the GPU)
    assert np.array_equal(rn[:, 0], plan.h.sum(axis=0) if dedup == "all" else 0 * rn[:, 0])
    assert np.array_equal(rn[:, 1], plan.n_e.reshape(G, -1).sum(axis=1))
    # expert-major positions and contents (identical for dedup and raw)
    epos = world.read("epos", 0, torch.int32).cpu().numpy().reshape(-1, K)
    assert np.array_equal(epos, plan.epos)
    xb = x.view(torch.int16) if dtype == torch.bfloat16 else x.view(torch.int32)
    e_loc = E // G
    for d in range(G):
        n = int(rn[d, 1])
        xm = world.read("xmaj", d, dtype, n * M).view(n, M).cpu()
        tt, kk = np.nonzero(ids // e_loc == d)
        want = xb[tt]
        got = (xm.view(torch.int16) if dtype == torch.bfloat16 else xm.view(torch.int32))[
            plan.epos[tt, kk]]
        assert torch.equal(got, want)
    if dedup == "all":
        gpos = world.read("gpos", 0, torch.int32).cpu().numpy().reshape(-1, G)
        assert np.array_equal(gpos, np.where(plan.hit, plan.pos, -1))
        for d in range(G):
            r = int(rn[d, 0])
            rx = world.read("recv_x", d, dtype, r * M).view(r, M).cpu()
            assert torch.equal(rx.view(xb.dtype), xb[plan.recv_rows(d)])
    # combine with a stand-in expert y = x * scale[slot]
    _apply_experts(world, plan, E, dtype)
    out_reg = world.combine(slot, w, dedup=dedup).clone()
    # addend (e.g. a shared expert's output) summed last in fp32
    add = (x * 0.5).to(dtype).cuda()
    out_add = world.combine(slot, w, dedup=dedup, addend=add).clone()
    rtol_a = 1e-5 if dtype == torch.float32 else 2e-2
    torch.testing.assert_close(out_add.float(), out_reg.float() + add.float(), rtol=rtol_a,
                               atol=rtol_a * float(out_reg.float().abs().max()))
    out = world.combine(slot, w, dedup=dedup)
    torch.cuda.synchronize()
    assert torch.equal(out, out_reg)      # repeated combine -> identical bits
    torch.cuda.synchronize()
    world.check_status()
    sc = _scale(E).numpy()
    wts = w.cpu().numpy().astype(np.float64)
    ref = (wts * sc[ids]).sum(axis=1)[:, None] * x.double().numpy()
    rtol = 1e-5 if dtype == torch.float32 else 2e-2
    np.testing.assert_allclose(out.double().cpu().numpy(), ref, rtol=rtol,
                               atol=rtol * np.abs(ref).max())
    world.close()


def test_dedup_moves_fewer_rows(hm):
    """Dedup ships one row per (token, destination); raw ships K per token."""
    from paper_2508_09591_b200.layer import route_topk
    G, E, K, M, T_r, dtype = CONFIGS["qwen3_small"]
    logits, x = _inputs(G, E, K, M, T_r, dtype, seed=3)
    slot, w, _ = route_topk(logits.cuda(), K)
    world = _world(hm, G, E, K, M, T_r, dtype)
    world.dispatch(x.cuda(), slot, w, dedup="all")
    torch.cuda.synchronize()
    rows = world.rows_received()
    ratio = rows[:, 1].sum() / rows[:, 0].sum()
    assert 1.3 < ratio < 1.7        # uniform E=128, K=8, G=8: 8 / 5.34 = 1.498
    world.close()


@pytest.mark.parametrize("dedup", ["gpu", "remote", "all", "none"])
def test_ragged_picks_padding(hm, dedup):
    """Tokens with dropped picks (slot id -1, e.g. capacity-dropped) and one
    token with no picks at all: the padding moves no rows and contributes
    nothing to the combine."""
    from paper_2508_09591_b200.layer import route_topk
    G, E, K, M, T_r, dtype = 8, 64, 4, 512, 96, torch.bfloat16
    logits, x = _inputs(G, E, K, M, T_r, dtype, seed=31)
    slot, w, _ = route_topk(logits.cuda(), K)
    g = torch.Generator().manual_seed(5)
    drop = torch.rand(G * T_r, K, generator=g) < 0.25
    drop[17] = True                                  # a token with no picks left
    slot = slot.clone()
    slot[drop.cuda()] = -1
    world = _world(hm, G, E, K, M, T_r, dtype)
    world.dispatch(x.cuda(), slot, w, dedup=dedup)
    torch.cuda.synchronize()
    world.check_status()
    ids = slot.cpu().numpy()
    valid = ids >= 0
    e_loc = E // G
    rn = world.rows_received()
    sc = _scale(E)
    for d in range(G):
        n_want = int(((ids // e_loc == d) & valid).sum())
        assert int(rn[d, 1]) == n_want
        xm = world.read("xmaj", d, dtype, n_want * M).view(n_want, M)
        # stand-in expert on the rows actually received: y = x * scale[slot]
        tt, kk = np.nonzero((ids // e_loc == d) & valid)
        epos = world.read("epos", 0, torch.int32).cpu().numpy().reshape(-1, K)
        row_slot = np.zeros(n_want, dtype=np.int64)
        row_slot[epos[tt, kk]] = ids[tt, kk]
        world.set_expert_outputs(d, (xm.float() * sc[row_slot].float().cuda()[:, None]).to(dtype))
    out = world.combine(slot, w, dedup=dedup)
    torch.cuda.synchronize()
    world.check_status()
    wts = w.cpu().numpy().astype(np.float64) * valid
    ref = (wts * sc.numpy()[np.where(valid, ids, 0)]).sum(axis=1)[:, None] * x.double().numpy()
    np.testing.assert_allclose(out.double().cpu().numpy(), ref, rtol=2e-2,
                               atol=2e-2 * np.abs(ref).max())
    assert torch.count_nonzero(out[17]) == 0
    world.close()


@pytest.mark.parametrize("E,K", [(128, 8), (256, 8), (64, 4), (32, 2), (128, 1)])
@pytest.mark.parametrize("renorm", [True, False])
def test_route_quad_equals_lane(hm, E, K, renorm):
    """Four-lanes-per-token router == lane-per-token router, bit for bit
    (ties included)."""
    from paper_2508_09591_b200 import _lib
    from paper_2508_09591_b200.layer import route_topk
    g = torch.Generator().manual_seed(E + K)
    logits = torch.randn(3001, E, generator=g)
    logits[::5, 7] = logits[::5, 9]
    logits[::11, 3:12] = 0.25           # wide ties
    # the router's threshold pre-pass: the whole top K inside one lane of the
    # quad (lane 0 loads float4 columns 0, 4, 8, ... i.e. experts 16 i + 0..3),
    # rows with only 8 finite logits (two lanes all -inf), rows of one value
    lane0 = [16 * i + c for i in range(E // 16) for c in range(4)][:8]
    logits[1::17, lane0] = 10.0 + torch.arange(len(lane0), dtype=torch.float32)
    logits[2::19, 8:] = float("-inf")
    logits[3::23] = 0.5
    lg = logits.cuda()
    try:
        res = []
        for quad in (0, 1):
            _lib.call("hm_route_set_option", quad)
            res.append(route_topk(lg, K, renormalize=renorm))
    finally:
        _lib.call("hm_route_set_option", 1)     # the default
    for a, b in zip(*res):
        assert torch.equal(a, b)


@pytest.mark.parametrize("dedup", ["gpu", "all", "none"])
def test_dispatch_plan_then_push_equals_dispatch(hm, dedup):
    """hm_dispatch = hm_dispatch_plan + hm_dispatch_push: the counts are final
    after the plan, and the two phases move the same rows."""
    from paper_2508_09591_b200 import _lib
    from paper_2508_09591_b200._lib import ptr, stream_ptr
    from paper_2508_09591_b200.layer import route_topk, transport_mode
    G, E, K, M, T_r, dtype = CONFIGS["qwen3_small"]
    logits, x = _inputs(G, E, K, M, T_r, dtype, seed=77)
    slot, w, _ = route_topk(logits.cuda(), K)
    xd = x.cuda()
    world = _world(hm, G, E, K, M, T_r, dtype)
    world.dispatch(xd, slot, w, dedup=dedup)
    ref_counts = world.counts()
    ref = world.combine(slot, w, dedup=dedup).clone()
    mode = transport_mode(dedup)
    _lib.call("hm_dispatch_plan", world._h, ptr(slot), ptr(w), mode, stream_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(world.counts(), ref_counts)
    _lib.call("hm_dispatch_push", world._h, ptr(xd), ptr(slot), ptr(w), mode, stream_ptr())
    if mode:
        _lib.call("hm_expand", world._h, stream_ptr())
    out = world.combine(slot, w, dedup=dedup)
    torch.cuda.synchronize()
    world.check_status()
    assert torch.equal(out, ref)
    world.close()
