"""CTA-pair (tcgen05 cta_group::2, 256 x 256 tile) grouped GEMMs -- the
forward and data-gradient kernels -- vs an fp32 reference on ragged groups
(empty groups, single rows, tails of every size)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_rows,N,K", [
    ([128], 256, 64),
    ([300, 0, 77, 513], 512, 256),
    ([1, 129, 255, 256, 257], 256, 2048),
    ([2048] * 4, 2048, 768),
])
def test_pair_gemm_matches_fp32(hm, n_rows, N, K):
    from paper_2508_09591_b200.ffn import grouped_gemm
    torch.manual_seed(0)
    G = len(n_rows)
    rows = sum(n_rows)
    a = torch.randn(max(rows, 1) + 300, K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(G, N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
    nr = torch.tensor(n_rows, dtype=torch.int32, device="cuda")
    two = grouped_gemm(a, b, nr)
    torch.cuda.synchronize()
    r, refs = 0, []
    for g, n in enumerate(n_rows):
        refs.append(a[r:r + n].float() @ b[g].float().T)
        r += n
    torch.testing.assert_close(two[:rows].float(), torch.cat(refs), rtol=2e-2, atol=2e-2)
