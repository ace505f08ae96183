"""Expert migration (K11): ExpertStore swaps move every array's slot slices."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _fill(store, names, S):
    for i, k in enumerate(names):
        v = store[k]
        v.copy_((torch.arange(S, device="cuda").view(-1, *([1] * (v.dim() - 1))) * 10 + i)
                .to(v.dtype).expand_as(v))


def test_local_swap_moves_all_arrays(hm):
    from paper_2508_09591_b200.migrate import ExpertStore
    S = 16
    arrays = {"w13": ((256, 64), torch.bfloat16), "w2": ((64, 128), torch.bfloat16),
              "master": ((3 * 64 * 128,), torch.float32), "adam_m": ((3 * 64 * 128,), torch.float32),
              "adam_v": ((3 * 64 * 128,), torch.float32)}
    st = ExpertStore(S, arrays)
    _fill(st, list(arrays), S)
    before = {k: st[k].clone() for k in arrays}
    st.migrate(3, 11)
    st.migrate(5, 5)          # no-op
    torch.cuda.synchronize()
    st.check_status()
    for k in arrays:
        want = before[k].clone()
        want[[3, 11]] = want[[11, 3]]
        assert torch.equal(st[k], want), k
    st.close()


def test_layer_swap_moves_weights_with_placement(hm):
    """A planned swap applied to the layer: placement + physical weights move
    together, so the layer output is unchanged (same experts, new slots)."""
    from paper_2508_09591_b200.moe import HierMoELayer
    G, E, K, M, I, T_r = 8, 16, 2, 256, 256, 64
    layer = HierMoELayer(G, E, K, M, I, T_r, dedup="all", seed=5)
    x = torch.randn(G * T_r, M, device="cuda").to(torch.bfloat16)
    y0 = layer(x).clone()
    layer.apply_swap((1, 9))       # slots on different ranks
    layer.apply_swap((4, 5))       # same rank
    y1 = layer(x)
    torch.cuda.synchronize()
    layer.store.check_status()
    assert list(layer.placement.slot_to_expert[[1, 9, 4, 5]]) == [9, 1, 5, 4]
    # same experts compute every pick; only the dedup grouping (bf16 partial
    # rounding) may change with the new slot -> rank map
    torch.testing.assert_close(y1.float(), y0.float(), rtol=2e-2, atol=2e-2)
    layer.close()
