"""HD2 (two-level) dispatch/combine over virtual 2x4 and 4x2 groups on one GPU.

Phase 1 must ship exactly propagate_level's copies (routing.py:189-215,
pinned in oracle/hiera.py): one row per (token, level-1 group) to the rank
with the source's local index in that group, in row-major copy order, with
restricted selections; phase 2's per-destination counts are the intra-phase
counts (traffic.py:123-141); the combined output matches the oracle.
"""

import numpy as np
import pytest
import torch

from oracle import hiera as O
from oracle import moe as OM

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fanouts", [(2, 4), (4, 2)])
@pytest.mark.parametrize("E,K,M,T_r,dtype", [(256, 8, 512, 96, torch.bfloat16),
                                             (16, 2, 256, 128, torch.float32)])
@pytest.mark.parametrize("dedup2", ["all", "remote"])
def test_two_level_parity(hm, fanouts, E, K, M, T_r, dtype, dedup2):
    from paper_2508_09591_b200.layer import TwoLevelWorld, route_topk
    U1, F = fanouts
    G = U1 * F
    g = torch.Generator().manual_seed(11 + E + U1)
    logits = torch.randn(G * T_r, E, generator=g)
    x = torch.randn(G * T_r, M, generator=g).to(dtype)
    slot, w, _ = route_topk(logits.cuda(), K)
    ids = slot.cpu().numpy()
    tw = TwoLevelWorld(fanouts, E, K, M, T_r, dtype)
    tw.dispatch(x.cuda(), slot, w, dedup2=dedup2)
    torch.cuda.synchronize()
    tw.phase1.check_status()
    tw.phase2.check_status()
    # phase 1 == propagate_level copies, routed to the relay of (group, local index)
    bits = OM.ids_to_bits(ids, E)
    cbits, origin, parent = O.propagate(bits, U1)
    src = origin // T_r
    relay = parent * F + src % F
    h1 = tw.phase1.counts()[:, :G]
    want_h1 = np.zeros((G, G), dtype=np.int64)
    np.add.at(want_h1, (src, relay), 1)
    assert np.array_equal(h1, want_h1)
    assert np.array_equal(h1.sum(axis=0).reshape(U1, F).sum(axis=1), O.dedup_counts(bits, U1))
    xb = x.view(torch.int16) if dtype == torch.bfloat16 else x.view(torch.int32)
    r1 = tw.phase1.rows_received()[:, 0]
    ids2 = tw.ids2.cpu().numpy().reshape(G, U1 * T_r, K)
    for r in range(G):
        copies = np.nonzero(relay == r)[0]          # row-major copy order
        assert r1[r] == copies.size
        rx = tw.phase1.read("recv_x", r, dtype, copies.size * M).view(copies.size, M).cpu()
        assert torch.equal(rx.view(xb.dtype), xb[origin[copies]])
        got = np.zeros((copies.size, E), dtype=bool)
        for i in range(copies.size):
            sel = ids2[r, i][ids2[r, i] >= 0]
            got[i, sel] = True
        assert np.array_equal(got, cbits[copies])
        assert (ids2[r, copies.size:] == -1).all()
    # phase 2: per-GPU counts of the level-2 copy mask == dedup counts at G
    h2 = tw.phase2.counts()[:, :G]
    assert np.array_equal(h2.sum(axis=0), O.dedup_counts(cbits, G))
    assert np.array_equal(h2.sum(axis=0), O.dedup_counts(bits, G))
    # stand-in experts y = x * (1 + slot/E) on phase-2 expert-major rows, then combine
    e_loc = E // G
    c2 = tw.phase2.counts()[:, G:]
    n_e = c2.sum(axis=0)
    for d in range(G):
        n = int(n_e[d * e_loc:(d + 1) * e_loc].sum())
        xm = tw.phase2.read("xmaj", d, dtype, n * M).view(n, M)
        row_slot = np.repeat(np.arange(d * e_loc, (d + 1) * e_loc), n_e[d * e_loc:(d + 1) * e_loc])
        s = torch.as_tensor(1.0 + row_slot / E, dtype=torch.float32).cuda()[:, None]
        tw.phase2.set_expert_outputs(d, (xm.float() * s).to(dtype))
    out = tw.combine(slot, w, dedup2=dedup2)
    torch.cuda.synchronize()
    tw.phase1.check_status()
    sc = 1.0 + np.arange(E) / E
    ref = (w.cpu().numpy().astype(np.float64) * sc[ids]).sum(axis=1)[:, None] * x.double().numpy()
    rtol = 1e-5 if dtype == torch.float32 else 3e-2
    np.testing.assert_allclose(out.double().cpu().numpy(), ref, rtol=rtol, atol=rtol * np.abs(ref).max())
    tw.close()
