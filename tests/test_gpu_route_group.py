"""DeepSeek-V3 group-limited gate (hm_route_group) vs the CPU restatement
(oracle/moe.py route_group_limited): expert indices bit-exact, weights at
fp32 tolerance (rtol 1e-6)."""

import numpy as np
import pytest
import torch

from oracle import moe as OM

pytestmark = pytest.mark.gpu

CASES = [  # (T, E, K, n_group, topk_group, scale, bias)
    (4096, 256, 8, 8, 4, 2.5, True),      # DeepSeek-V3
    (1000, 64, 4, 4, 2, 1.0, True),
    (513, 16, 2, 1, 1, 1.0, False),       # no grouping: sigmoid top-K
    (300, 128, 6, 16, 3, 1.5, True),
    (64, 512, 8, 32, 4, 2.5, False),
]


@pytest.mark.parametrize("case", CASES, ids=[f"E{c[1]}g{c[3]}" for c in CASES])
def test_route_group_matches_oracle(hm, case):
    from paper_2508_09591_b200.layer import route_group_limited
    T, E, K, ng, tg, scale, use_bias = case
    g = torch.Generator().manual_seed(T + E)
    logits = torch.randn(T, E, generator=g) * 2.0
    bias = (torch.randn(E, generator=g) * 0.1) if use_bias else None
    perm = torch.randperm(E, generator=g).to(torch.int32)
    slot, w, ex = route_group_limited(logits.cuda(), K, ng, tg, None if bias is None else bias.cuda(),
                                      scale, perm.cuda())
    rs, rw, rex = OM.route_group_limited(logits.numpy(), K, ng, tg,
                                         None if bias is None else bias.numpy(), scale,
                                         perm.numpy())
    assert np.array_equal(ex.cpu().numpy(), rex)
    assert np.array_equal(slot.cpu().numpy(), rs)
    np.testing.assert_allclose(w.cpu().numpy(), rw, rtol=1e-6, atol=1e-7)


def test_route_group_rejects_bad_args(hm):
    from paper_2508_09591_b200.layer import route_group_limited
    x = torch.randn(8, 64, device="cuda")
    with pytest.raises(ValueError):
        route_group_limited(x, 8, 5, 2)        # 5 does not divide 64
    with pytest.raises(ValueError):
        route_group_limited(x, 8, 16, 1)       # 8 picks do not fit in one group of 4
