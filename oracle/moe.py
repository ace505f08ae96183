"""numpy restatement of the MoE layer hot path (TEST INFRASTRUCTURE ONLY).

The reference (``hiera2a``) models AlltoAll volumes but has no layer math;
``PAPER.md:110-117`` specifies it: softmax gating, top-K, E expert FFNs, a
gate-weighted sum, with expert parallelism (E/G experts per GPU, contiguous,
``topology.py:91-100``) and every GPU holding different tokens.  This module
restates that plus the per-rank dedup decomposition the product executes:

* a G-rank world holds ``T_r`` tokens per rank; the global token order is the
  rank-ordered concatenation (``SPEC.md:310``);
* slot ``s`` lives on rank ``s // (E/G)`` (``topology.py:99-100``);
* dispatch sends one row per (token, destination rank) hit -- the dedup mask
  is ``group_reduce(bits, G)`` (``traffic.py:58-64``) -- and the rows for
  destination ``d`` arrive in global token order, i.e. the row-major copy
  order of ``propagate_level`` (``routing.py:204-215``) restricted to ``d``;
* combine pre-reduces, on the expert side, every local expert's gate-weighted
  output into one row per (token, destination) and the source sums those rows
  over destinations in ascending rank order.

Parity for the layer values is **unpinned** by the reference (no code, no
tests); the dispatch/count decisions are pinned through :mod:`oracle.hiera`.
"""

from __future__ import annotations

import numpy as np


def route_topk(logits: np.ndarray, top_k: int, expert_to_slot=None,
               renormalize: bool = True):
    """Softmax top-K gating.

    Selection is on the logits, value descending then expert index ascending
    (a total order, so indices are bit-exact).  Weights are softmax
    probabilities of the chosen experts, renormalised over the K picks when
    ``renormalize`` (Qwen3 ``norm_topk_prob``).  Returns ``(slot_ids int32
    [T,K], weights float64 [T,K], expert_ids int32 [T,K])``.
    """
    logits = np.asarray(logits, dtype=np.float32)
    t, e = logits.shape
    order = np.lexsort((np.broadcast_to(np.arange(e), (t, e)), -logits), axis=1)
    experts = order[:, :top_k].astype(np.int32)
    l64 = logits.astype(np.float64)
    mx = l64.max(axis=1, keepdims=True)
    ex = np.exp(l64 - mx)
    chosen = np.take_along_axis(ex, experts, axis=1)
    denom = chosen.sum(axis=1, keepdims=True) if renormalize else ex.sum(axis=1, keepdims=True)
    weights = chosen / denom
    e2s = np.arange(e) if expert_to_slot is None else np.asarray(expert_to_slot)
    return e2s[experts].astype(np.int32), weights, experts


def route_group_limited(logits: np.ndarray, top_k: int, n_group: int, topk_group: int,
                        bias=None, route_scale: float = 1.0, expert_to_slot=None):
    """DeepSeek-V3 gate (the reference only specifies softmax
    top-K, so this follows DeepSeek-V3's published inference
    gate): scores = sigmoid(logits) (evaluated in float64, rounded to
    float32), choice = scores + bias (float32); group score = sum of the two
    largest choice values of each of ``n_group`` contiguous expert groups;
    keep the ``topk_group`` best groups; top-K of choice inside them; weights
    = scores of the picks / their sum * route_scale.  Every selection is
    value descending, index ascending.  Returns (slot ids int32 [T,K],
    weights float64 [T,K], expert ids int32 [T,K]).
    """
    logits = np.asarray(logits, dtype=np.float32)
    t, e = logits.shape
    gs = e // n_group
    sc = (1.0 / (1.0 + np.exp(-logits.astype(np.float64)))).astype(np.float32)
    b = np.zeros(e, np.float32) if bias is None else np.asarray(bias, np.float32)
    ch = (sc + b[None, :]).astype(np.float32)
    grp = ch.reshape(t, n_group, gs)
    top2 = -np.sort(-grp, axis=2)[:, :, :2]
    gscore = (top2[:, :, 0] + top2[:, :, 1]).astype(np.float32) if gs > 1 else top2[:, :, 0]
    gorder = np.lexsort((np.broadcast_to(np.arange(n_group), (t, n_group)), -gscore), axis=1)
    keep = np.zeros((t, n_group), dtype=bool)
    np.put_along_axis(keep, gorder[:, :topk_group], True, axis=1)
    masked = np.where(np.repeat(keep, gs, axis=1), ch, -np.inf).astype(np.float32)
    order = np.lexsort((np.broadcast_to(np.arange(e), (t, e)), -masked), axis=1)
    experts = order[:, :top_k].astype(np.int32)
    w = np.take_along_axis(sc, experts, axis=1).astype(np.float64)
    w = w / w.sum(axis=1, keepdims=True) * route_scale
    e2s = np.arange(e) if expert_to_slot is None else np.asarray(expert_to_slot)
    return e2s[experts].astype(np.int32), w, experts


def ids_to_bits(ids: np.ndarray, experts: int) -> np.ndarray:
    """K-per-row id lists -> T x E bool mask (RoutingMask.bits, routing.py:31-56)."""
    t = ids.shape[0]
    bits = np.zeros((t, experts), dtype=bool)
    bits[np.repeat(np.arange(t), ids.shape[1]), ids.reshape(-1)] = True
    return bits


class DispatchPlan:
    """Per-rank dedup dispatch plan of a G-rank world.

    Attributes (all integer numpy arrays):
      hit   [T, G]      dedup mask (token t sends one row to rank d)
      h     [G, G]      rows rank s sends to rank d (dedup)
      pos   [T, G]      receive-row index of (t, d) at rank d, -1 if not hit
      c     [G, E]      selections rank s sends to slot e (no dedup)
      epos  [T, K]      expert-major row of (t, k) at rank dest(e_k)
      n_e   [E]         rows per slot (expert GEMM group sizes)

    ``gpus``: the ranks' GPU count P.  A slot's rows are source-major starting
    with the sources on the destination's own GPU (ranks rotated by the GPU's
    first rank; the identity with one GPU), so the rows a GPU already holds
    form one block in front of the ones that cross NVLink.
    """

    def __init__(self, ids: np.ndarray, ranks: int, experts: int, gpus: int = 1):
        ids = np.asarray(ids, dtype=np.int64)
        t, k = ids.shape
        if t % ranks:
            raise ValueError("tokens must split evenly over ranks")
        self.ranks, self.experts, self.top_k = ranks, experts, k
        t_r = t // ranks
        e_loc = experts // ranks
        src = np.arange(t) // t_r
        dest = ids // e_loc
        hit = np.zeros((t, ranks), dtype=bool)
        hit[np.repeat(np.arange(t), k), dest.reshape(-1)] = True
        self.hit = hit
        self.h = np.stack([hit[src == s].sum(axis=0) for s in range(ranks)]).astype(np.int64)
        # receive order at d = global token order (source-major) of hitting tokens
        pos = np.full((t, ranks), -1, dtype=np.int64)
        for d in range(ranks):
            rows = np.nonzero(hit[:, d])[0]
            pos[rows, d] = np.arange(rows.size)
        self.pos = pos
        # expert-major layout at each rank: local slot blocks, each source-major
        c = np.zeros((ranks, experts), dtype=np.int64)
        for s in range(ranks):
            np.add.at(c[s], ids[src == s].reshape(-1), 1)
        self.c = c
        self.n_e = c.sum(axis=0)
        ebase = np.zeros(experts, dtype=np.int64)
        for e in range(experts):
            lo = (e // e_loc) * e_loc
            ebase[e] = self.n_e[lo:e].sum()
        epos = np.full((t, k), -1, dtype=np.int64)
        per_gpu = ranks // gpus
        for e in range(experts):
            tt, kk = np.nonzero(ids == e)          # row-major => token order
            q0 = (e // e_loc) // per_gpu * per_gpu
            order = np.argsort((src[tt] - q0) % ranks, kind="stable")
            tt, kk = tt[order], kk[order]
            epos[tt, kk] = ebase[e] + np.arange(tt.size)
        self.epos = epos
        self.ebase = ebase
        self.ids = ids

    def recv_rows(self, d: int) -> np.ndarray:
        """Global token index of every row rank d receives, in arrival order."""
        return np.nonzero(self.hit[:, d])[0]


def swiglu_experts(x_rows: np.ndarray, slot_of_row: np.ndarray, w1, w3, w2):
    """y = W2 (silu(W1 x) * (W3 x)) per row with its slot's weights (fp64).

    ``w1, w3``: [E, I, M]; ``w2``: [E, M, I].
    """
    x = np.asarray(x_rows, dtype=np.float64)
    out = np.zeros_like(x)
    for e in np.unique(slot_of_row):
        sel = slot_of_row == e
        a = x[sel] @ np.asarray(w1[e], np.float64).T
        b = x[sel] @ np.asarray(w3[e], np.float64).T
        hdn = a / (1.0 + np.exp(-a)) * b
        out[sel] = hdn @ np.asarray(w2[e], np.float64).T
    return out


def moe_forward(x, ids, weights, expert_fn):
    """out[t] = sum_k w[t,k] * expert_fn(x[t], ids[t,k]) in fp64."""
    x = np.asarray(x, dtype=np.float64)
    t, k = ids.shape
    rows = np.repeat(np.arange(t), k)
    y = expert_fn(x[rows], ids.reshape(-1)).reshape(t, k, -1)
    return (np.asarray(weights, np.float64)[:, :, None] * y).sum(axis=1)


def dedup_combine(plan: DispatchPlan, weights, y_expert_major, payload_round=None):
    """Expert-side pre-reduce + source-side sum, mirroring the product's order.

    ``y_expert_major[d]`` holds rank d's expert-major outputs (rows indexed by
    ``plan.epos``).  ``payload_round`` optionally rounds the pre-reduced
    partial rows (e.g. to bf16) as the wire format does.  Returns the
    combined [T, M] output in fp64.
    """
    t, k = plan.ids.shape
    e_loc = plan.experts // plan.ranks
    m = y_expert_major[0].shape[1]
    out = np.zeros((t, m))
    w = np.asarray(weights, np.float64)
    for tok in range(t):
        acc = np.zeros(m)
        for d in range(plan.ranks):
            if not plan.hit[tok, d]:
                continue
            part = np.zeros(m)
            for kk in range(k):
                if plan.ids[tok, kk] // e_loc == d:
                    part += w[tok, kk] * np.asarray(y_expert_major[d][plan.epos[tok, kk]], np.float64)
            if payload_round is not None:
                part = payload_round(part)
            acc += part
        out[tok] = acc
    return out


def cpu_dispatch_combine(logits, x, top_k: int, y_major=None, threads: int = 1,
                         chunk: int = 256):
    """torch-CPU port of one dispatch + combine step at full size (the timed
    CPU baseline; TEST/BENCH INFRASTRUCTURE ONLY).

    The same step the GPU times at N = 1, on host memory with ``threads``
    intra-op threads: softmax top-K gating (``torch.topk`` on the logits),
    the dispatch plan (stable sort of the picks by slot = the expert-major
    row order, source-major within a slot), the dispatch itself (one
    ``index_select`` of the token rows into expert-major order) and the
    combine (``index_select`` back to (token, pick) order and a gate-weighted
    fp32 sum per token, chunked so the fp32 temporaries stay in cache).  On
    one host every EP rank is local, so -- as on one GPU -- no dedup rows are
    exchanged.  ``x`` is bf16 (the GPU's storage format); ``y_major`` are the
    expert outputs in expert-major order (default: identity experts).
    Returns (out [T, M] bf16, y_major, order).
    """
    import torch
    torch.set_num_threads(max(1, threads))
    logits = torch.as_tensor(logits)
    x = torch.as_tensor(x)
    t = x.shape[0]
    # gating: top-K by value (ties by index via topk's sorted order), softmax
    # over the picks (renormalised, Qwen3 norm_topk_prob)
    val, ids = torch.topk(logits, top_k, dim=1, sorted=True)
    w = torch.softmax(val, dim=1)
    flat = ids.reshape(-1)
    order = torch.argsort(flat, stable=True)           # expert-major row -> (t, k) pick
    xm = x.index_select(0, order // top_k)               # dispatch
    ym = xm if y_major is None else y_major
    inv = torch.empty_like(order)
    inv[order] = torch.arange(order.numel())             # (t, k) pick -> expert-major row
    out = torch.empty_like(x)
    for lo in range(0, t, chunk):                        # combine
        hi = min(t, lo + chunk)
        yk = ym.index_select(0, inv[lo * top_k:hi * top_k]).view(hi - lo, top_k, -1)
        out[lo:hi] = torch.bmm(w[lo:hi, None, :], yk.float()).squeeze(1).to(x.dtype)
    return out, ym, order
