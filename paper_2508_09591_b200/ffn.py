"""Expert SwiGLU FFN on the dispatch's expert-major rows (tcgen05 grouped GEMM).

H = silu(X W1^T) * (X W3^T), Y = H W2^T per local expert, bf16 in/out with
fp32 accumulation in TMEM (csrc/gemm_sm100.cu).  Group sizes stay on the
device (the dispatch's per-slot counts), so the FFN needs no host sync.
"""

from __future__ import annotations

import torch

from . import _lib
from ._lib import ptr, stream_ptr

BLOCK = 128


def pack_w13(w1: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """[G, I, M] gate + up weights -> [G, 2I, M] with 128-row gate/up blocks
    interleaved (one 256-row GEMM tile = a gate block and its up block)."""
    g, inter, m = w1.shape
    if w3.shape != w1.shape or inter % BLOCK:
        raise ValueError("w1/w3 must be [G, I, M] with I a multiple of 128")
    nb = inter // BLOCK
    return torch.stack([w1.view(g, nb, BLOCK, m), w3.view(g, nb, BLOCK, m)], dim=2) \
        .reshape(g, 2 * inter, m).contiguous()


def grouped_gemm(a: torch.Tensor, b: torch.Tensor, n_rows: torch.Tensor, swiglu: bool = False,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """out[rows of g] = a[rows of g] @ b[g]^T (b: [G, N, K]); swiglu -> N/2 cols."""
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise ValueError("bf16 operands required")
    groups, n, k = b.shape
    cols = n // 2 if swiglu else n
    if out is None:
        out = torch.empty((a.shape[0], cols), dtype=torch.bfloat16, device=a.device)
    _lib.call("hm_grouped_gemm", ptr(a.contiguous()), a.shape[0], ptr(b.contiguous()), groups,
              ptr(n_rows), n, k, int(swiglu), ptr(out), out.stride(0), stream_ptr())
    return out


def expert_ffn_ptrs(x_ptr: int, a_rows: int, n_rows_ptr: int, groups: int, w13: torch.Tensor,
                    w2: torch.Tensor, hidden: int, inter: int, h: torch.Tensor, y_ptr: int) -> None:
    """FFN on raw device rows (e.g. an EPWorld's xmaj -> ymaj buffers)."""
    _lib.call("hm_expert_ffn", x_ptr, a_rows, n_rows_ptr, groups, ptr(w13), ptr(w2), hidden,
              inter, ptr(h), y_ptr, stream_ptr())


def expert_ffn_save_ptrs(x_ptr: int, a_rows: int, n_rows_ptr: int, groups: int,
                         w13: torch.Tensor, w2: torch.Tensor, hidden: int, inter: int,
                         h: torch.Tensor, y_ptr: int, g13_ptr: int) -> None:
    """Training forward: the FFN plus GEMM1's pre-activations into g13_ptr."""
    _lib.call("hm_expert_ffn_save", x_ptr, a_rows, n_rows_ptr, groups, ptr(w13), ptr(w2), hidden,
              inter, ptr(h), y_ptr, g13_ptr, stream_ptr())


def expert_ffn_gather_ptrs(x_ptr: int, x_rows: int, idx_ptr: int, a_rows: int, n_rows_ptr: int,
                           groups: int, w13: torch.Tensor, w2: torch.Tensor, hidden: int,
                           inter: int, h: torch.Tensor, y_ptr: int, g13_ptr: int = 0) -> None:
    """FFN with the fused dispatch: GEMM1 gathers its rows from the token-major
    x [x_rows, hidden] by the expert-major row indices idx (cp.async producer
    warps)."""
    _lib.call("hm_expert_ffn_gather", x_ptr, x_rows, idx_ptr, a_rows, n_rows_ptr, groups,
              ptr(w13), ptr(w2), hidden, inter, ptr(h), y_ptr, g13_ptr or None, stream_ptr())


def expert_ffn_backward_gather_ptrs(x_ptr: int, x_rows: int, idx_ptr: int, a_rows: int,
                                    n_rows_ptr: int, groups: int, w13: torch.Tensor,
                                    w2: torch.Tensor, gy_ptr: int, hidden: int, inter: int,
                                    sc: "FFNBackwardScratch", gx_ptr: int, dw13: torch.Tensor,
                                    dw2: torch.Tensor, g13_saved_ptr: int,
                                    accumulate: bool = False) -> None:
    """Backward of expert_ffn_gather_ptrs (saved pre-activations)."""
    _lib.call("hm_expert_ffn_backward_gather", x_ptr, x_rows, idx_ptr, a_rows, n_rows_ptr, groups,
              ptr(w13), ptr(w2), gy_ptr, hidden, inter, g13_saved_ptr, ptr(sc.dh),
              ptr(sc.dg13), ptr(sc.h), ptr(sc.layout), gx_ptr, ptr(dw13), ptr(dw2),
              int(bool(accumulate)), stream_ptr())


def expert_ffn_multi_ptrs(x_ptr: int, x_rows: int, idx_ptr: int, seg_rows: int, segs: int,
                          n_rows_ptr: int, groups_per_seg: int, w13: torch.Tensor,
                          w2: torch.Tensor, hidden: int, inter: int, h: torch.Tensor, y_ptr: int,
                          g13_ptr: int = 0, recv_ptr: int = 0) -> None:
    """All of a GPU's EP ranks' expert FFNs in one launch per GEMM (segments
    of ``groups_per_seg`` groups, rows at s * seg_rows); idx_ptr 0: x holds
    the expert-major rows, else the rows are gathered from x by index
    (negative index ~r: row r of the receive buffer at recv_ptr)."""
    _lib.call("hm_expert_ffn_multi", x_ptr, x_rows, idx_ptr or None, recv_ptr or None, seg_rows,
              segs, n_rows_ptr,
              groups_per_seg, ptr(w13), ptr(w2), hidden, inter, ptr(h), y_ptr, g13_ptr or None,
              stream_ptr())


def expert_ffn_backward_multi_ptrs(x_ptr: int, x_rows: int, idx_ptr: int, seg_rows: int,
                                   segs: int, n_rows_ptr: int, groups_per_seg: int,
                                   w13: torch.Tensor, w2: torch.Tensor, gy_ptr: int, hidden: int,
                                   inter: int, sc: "FFNBackwardScratch", gx_ptr: int,
                                   dw13: torch.Tensor, dw2: torch.Tensor, g13_ptr: int,
                                   accumulate: bool = False, recv_ptr: int = 0,
                                   parts: int = 3, h_fwd: torch.Tensor | None = None) -> None:
    """Backward of expert_ffn_multi_ptrs (saved pre-activations).  parts: 1 =
    data gradients (gx), 2 = weight gradients (from part 1's scratch), 3 = both.
    h_fwd: the forward's H (same row layout) -- dW2 uses it and the SwiGLU
    backward does not recompute it into the scratch."""
    h = sc.h if h_fwd is None else h_fwd
    _lib.call("hm_expert_ffn_backward_multi", x_ptr, x_rows, idx_ptr or None, recv_ptr or None,
              seg_rows, segs,
              n_rows_ptr, groups_per_seg, ptr(w13), ptr(w2), gy_ptr, hidden, inter, g13_ptr,
              ptr(sc.dh), ptr(sc.dg13), ptr(h), ptr(sc.layout), gx_ptr, ptr(dw13), ptr(dw2),
              int(bool(accumulate)), int(parts) | (4 if h_fwd is not None else 0), stream_ptr())


def set_gemm_ctas(n: int) -> None:
    """Cap the persistent grouped-GEMM grid at n CTAs (0: one per SM)."""
    _lib.call("hm_ffn_set_option", 1, int(n))


class FFNBackwardScratch:
    """Work buffers of one expert-FFN backward (capacity rows x widths)."""

    def __init__(self, rows: int, groups: int, hidden: int, inter: int):
        kw = dict(dtype=torch.bfloat16, device="cuda")
        self.rows, self.groups, self.hidden, self.inter = rows, groups, hidden, inter
        self.g13 = torch.empty(rows, 2 * inter, **kw)
        self.dg13 = torch.empty(rows, 2 * inter, **kw)
        self.dh = torch.empty(rows, inter, **kw)
        self.h = torch.empty(rows, inter, **kw)
        self.layout = torch.empty(2 * (groups + 1), dtype=torch.int32, device="cuda")


def expert_ffn_backward_ptrs(x_ptr: int, a_rows: int, n_rows_ptr: int, groups: int,
                             w13: torch.Tensor, w2: torch.Tensor, gy_ptr: int, hidden: int,
                             inter: int, sc: FFNBackwardScratch, gx_ptr: int, dw13: torch.Tensor,
                             dw2: torch.Tensor, g13_saved_ptr: int = 0,
                             accumulate: bool = False) -> None:
    """Grads of the SwiGLU experts: gx (rows), dW13 [g][2I][M], dW2 [g][M][I].
    The data-gradient GEMMs read w13 / w2 as stored (MN-major).
    ``g13_saved_ptr``: the forward's pre-activations (expert_ffn_save_ptrs);
    0 -> recomputed.  ``accumulate``: add the weight grads to dw13 / dw2
    (needs the saved pre-activations)."""
    if g13_saved_ptr:
        _lib.call("hm_expert_ffn_backward_saved", x_ptr, a_rows, n_rows_ptr, groups, ptr(w13),
                  ptr(w2), gy_ptr, hidden, inter, g13_saved_ptr, ptr(sc.dh), ptr(sc.dg13),
                  ptr(sc.h), ptr(sc.layout), gx_ptr, ptr(dw13), ptr(dw2), int(bool(accumulate)),
                  stream_ptr())
        return
    if accumulate:
        raise ValueError("accumulate needs the saved pre-activations")
    _lib.call("hm_expert_ffn_backward", x_ptr, a_rows, n_rows_ptr, groups, ptr(w13), ptr(w2),
              gy_ptr, hidden, inter, ptr(sc.g13), ptr(sc.dh), ptr(sc.dg13), ptr(sc.h),
              ptr(sc.layout), gx_ptr, ptr(dw13), ptr(dw2), stream_ptr())
