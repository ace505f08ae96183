"""Backward of dedup dispatch/combine (K8) vs analytic gradients.

Stand-in experts y = s_e * x (s_e = 1 + e/E) make the layer linear:
out_t = sum_k w_k s_{e_k} x_t, so for an output gradient g:
  d w_k = <g_t, y_k>,   d x_t = sum_k w_k s_{e_k} g_t.
The expert backward (gx = s_e * gy) is applied between the two calls.
"""

import zlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dedup", ["all", "remote", "gpu", "none"])
@pytest.mark.parametrize("shape", [(8, 16, 2, 256, 128, torch.float32),
                                   (8, 128, 8, 512, 64, torch.bfloat16)])
def test_dispatch_combine_backward(hm, dedup, shape):
    from paper_2508_09591_b200.layer import EPWorld, route_topk
    G, E, K, M, T_r, dtype = shape
    gen = torch.Generator().manual_seed(zlib.crc32(f"{dedup}{E}".encode()) % 10000)
    logits = torch.randn(G * T_r, E, generator=gen)
    x = torch.randn(G * T_r, M, generator=gen).to(dtype)
    g = torch.randn(G * T_r, M, generator=gen).to(dtype)
    slot, w, _ = route_topk(logits.cuda(), K)
    ep = EPWorld(G, E, K, M, T_r, dtype=dtype, grad=True)
    ep.dispatch(x.cuda(), slot, w, dedup=dedup)
    counts = ep.counts()[:, G:]
    n_e = counts.sum(axis=0)
    e_loc = E // G
    scale = 1.0 + torch.arange(E, dtype=torch.float32) / E
    row_scale = []
    for d in range(G):
        n = int(n_e[d * e_loc:(d + 1) * e_loc].sum())
        rs = torch.repeat_interleave(scale[d * e_loc:(d + 1) * e_loc],
                                     torch.as_tensor(n_e[d * e_loc:(d + 1) * e_loc])).cuda()[:, None]
        row_scale.append(rs)
        xm = ep.read("xmaj", d, dtype, n * M).view(n, M)
        ep.set_expert_outputs(d, (xm.float() * rs).to(dtype))
    ep.combine(slot, w, dedup=dedup)
    dw = ep.dispatch_grad(g.cuda(), slot, w, dedup=dedup)
    for d in range(G):
        n = row_scale[d].shape[0]
        gy = ep.read("gy", d, dtype, n * M).view(n, M)
        ep.write("gx", (gy.float() * row_scale[d]).to(dtype).contiguous(), d)
    dx = ep.combine_grad(slot, dw, dedup=dedup)
    torch.cuda.synchronize()
    ep.check_status()
    ids = slot.cpu().numpy()
    wn = w.cpu().numpy().astype(np.float64)
    s = scale.double().numpy()[ids]                               # [T, K]
    xd, gd = x.double().numpy(), g.double().numpy()
    y = xd if dtype == torch.float32 else None
    # gate grads: <g_t, y_k>, y_k = s_k x_t (as stored in the payload dtype)
    ydot = (gd * xd).sum(axis=1)[:, None] * s
    ref_dx = (wn * s).sum(axis=1)[:, None] * gd
    rtol = 1e-4 if dtype == torch.float32 else 3e-2
    np.testing.assert_allclose(dw.double().cpu().numpy(), ydot, rtol=rtol,
                               atol=rtol * np.abs(ydot).max())
    np.testing.assert_allclose(dx.double().cpu().numpy(), ref_dx, rtol=rtol,
                               atol=rtol * np.abs(ref_dx).max())
    ep.close()
