"""HierMoE layer hot path: gating, dedup dispatch, combine over an EP world.

The reference (hiera2a) only *models* this exchange -- per-destination dedup
counts (traffic.py:58-82) priced by an alpha-beta AlltoAll model
(traffic.py:93-170).  ``EPWorld`` executes it on B200s:

* G virtual expert-parallel ranks (``Topology.num_gpus``) are hosted on P
  physical GPUs, one process per GPU (P = 1: all G ranks on one GPU, the
  exchange runs through HBM; P > 1: CUDA-IPC peer mappings over NVLink 5);
* slot s lives on rank s // (E/G) (topology.py:99-100); tokens are rank-major
  (SPEC.md:310);
* ``dispatch(dedup=True)`` ships one row per (token, destination rank) -- the
  dedup mask is group_reduce(bits, G) (traffic.py:58-64) -- and re-expands it
  into expert-major rows at the destination; ``dedup=False`` is the
  non-deduplicated baseline (one row per selection, the reference's "std"
  strategy, engine.py:6-8);
* ``combine`` gate-weights and sums expert outputs back to the source:
  dedup pre-reduces per destination and the source sums in ascending rank
  order (deterministic, no float atomics).

All kernels are stream-ordered; a dispatch/combine step performs no host
synchronisation.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import ptr, stream_ptr

_KIND = {"recv_x": 0, "recv_meta": 1, "xmaj": 2, "ymaj": 3, "comb": 4, "counts": 5, "gpos": 6,
         "epos": 7, "hitmask": 8, "offsets": 9, "n_e": 10, "status": 11, "gy": 12, "gx": 13,
         "recv_g": 14, "gpos_g": 15, "rows_g": 16, "xidx": 17}

_STATUS = {2: "row capacity overflow", 3: "peer barrier timeout", 4: "slot id out of range"}

# transport modes: "none" one row per selection (no dedup, the reference's "std");
# "all" one row per (token, destination rank) for every destination, including
# ranks on the same GPU (the full dedup copy list); "remote" dedup rows only
# across GPUs -- ranks sharing a GPU exchange through HBM without a link to
# save bytes on, so their rows go straight to expert-major positions.
# "gpu" dedups per (token, destination GPU): one row crosses NVLink per
# remote GPU a token hits, and the receiving GPU re-expands it into its local
# ranks' expert rows -- the HierMoE principle (dedup at the level that owns a
# link) for ranks hosted several per GPU; with one rank per GPU it equals
# "remote".
MODES = {"none": 0, "all": 1, "remote": 2, "gpu": 3}


def transport_mode(dedup) -> int:
    if dedup is True:
        return MODES["gpu"]
    if dedup is False or dedup is None:
        return MODES["none"]
    if dedup not in MODES:
        raise ValueError(f"dedup must be a bool or one of {sorted(MODES)}")
    return MODES[dedup]


def route_topk(logits: torch.Tensor, top_k: int, expert_to_slot: torch.Tensor | None = None,
               renormalize: bool = True):
    """Softmax top-K gating on the GPU.

    Selection is value-descending, expert-index-ascending on ties (bit-exact
    indices); weights are softmax probabilities of the picks, renormalised
    over the K picks when ``renormalize``.  Returns (slot_ids int32 [T,K],
    weights fp32 [T,K], expert_ids int32 [T,K]).
    """
    if logits.dtype != torch.float32 or not logits.is_cuda or logits.ndim != 2:
        raise ValueError("logits must be a 2-D float32 CUDA tensor")
    logits = logits.contiguous()
    t, e = logits.shape
    slot = torch.empty((t, top_k), dtype=torch.int32, device=logits.device)
    w = torch.empty((t, top_k), dtype=torch.float32, device=logits.device)
    ex = torch.empty((t, top_k), dtype=torch.int32, device=logits.device)
    e2s = None if expert_to_slot is None else expert_to_slot.to(device=logits.device,
                                                               dtype=torch.int32).contiguous()
    _lib.call("hm_route_topk", ptr(logits), t, e, top_k, ptr(e2s), int(bool(renormalize)),
              ptr(slot), ptr(w), ptr(ex), stream_ptr())
    return slot, w, ex


def route_group_limited(logits: torch.Tensor, top_k: int, n_group: int, topk_group: int,
                        bias: torch.Tensor | None = None, route_scale: float = 1.0,
                        expert_to_slot: torch.Tensor | None = None):
    """DeepSeek-V3 group-limited gate on the GPU (sigmoid scores, bias-corrected
    choice, the ``topk_group`` best of ``n_group`` expert groups, top-K inside;
    weights = picked scores / their sum * ``route_scale``).  Returns (slot_ids
    int32 [T,K], weights fp32 [T,K], expert_ids int32 [T,K])."""
    if logits.dtype != torch.float32 or not logits.is_cuda or logits.ndim != 2:
        raise ValueError("logits must be a 2-D float32 CUDA tensor")
    logits = logits.contiguous()
    t, e = logits.shape
    slot = torch.empty((t, top_k), dtype=torch.int32, device=logits.device)
    w = torch.empty((t, top_k), dtype=torch.float32, device=logits.device)
    ex = torch.empty((t, top_k), dtype=torch.int32, device=logits.device)
    b = None if bias is None else bias.to(device=logits.device, dtype=torch.float32).contiguous()
    e2s = None if expert_to_slot is None else expert_to_slot.to(device=logits.device,
                                                               dtype=torch.int32).contiguous()
    _lib.call("hm_route_group", ptr(logits), t, e, top_k, n_group, topk_group, ptr(b),
              float(route_scale), ptr(e2s), ptr(slot), ptr(w), ptr(ex), stream_ptr())
    return slot, w, ex


def exchange_handles(mine: bytes, index: int, gpus: int, group=None) -> bytes:
    """All-gather one fixed-size IPC handle per GPU, ordered by GPU index.

    Works over NCCL (CUDA tensors) and gloo (CPU tensors); the GPU index of a
    process must equal its rank in ``group``.
    """
    import torch.distributed as dist
    if dist.get_world_size(group) != gpus or dist.get_rank(group) != index:
        raise ValueError("gpu_index/gpus must match the process group rank/size")
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    local = torch.tensor(bytearray(mine), dtype=torch.uint8, device=dev)
    parts = [torch.empty_like(local) for _ in range(gpus)]
    dist.all_gather(parts, local, group=group)
    return torch.cat(parts).cpu().numpy().tobytes()


def rank_placement(ranks: int, gpus: int, gpu_index: int) -> range:
    """Virtual EP ranks hosted on one GPU: contiguous blocks of L = G/P."""
    if gpus < 1 or ranks % gpus:
        raise ValueError(f"ranks ({ranks}) must be a multiple of gpus ({gpus})")
    per = ranks // gpus
    return range(gpu_index * per, (gpu_index + 1) * per)


class EPWorld:
    """G virtual EP ranks on P GPUs with symmetric dispatch/combine buffers.

    ``tokens_per_rank`` is the per-rank token capacity T_r; every call moves
    all L = G/P local ranks' tokens: x is [L*T_r, M], ids/weights [L*T_r, K].
    """

    def __init__(self, ranks: int, experts: int, top_k: int, hidden: int,
                 tokens_per_rank: int, dtype: torch.dtype = torch.bfloat16,
                 gpus: int = 1, gpu_index: int = 0, group=None, n_cap_rows: int = 0,
                 relay_groups: int = 0, grad: bool = False):
        lib = _lib.load()
        if dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("payload dtype must be bfloat16 or float32")
        self.ranks, self.experts, self.top_k, self.hidden = ranks, experts, top_k, hidden
        self.tokens_per_rank, self.dtype = tokens_per_rank, dtype
        self.gpus, self.gpu_index = gpus, gpu_index
        self.local = ranks // gpus
        self.elem = 2 if dtype == torch.bfloat16 else 4
        h = ctypes.c_void_p()
        _lib.check(lib.hm_world_create(ranks, gpus, gpu_index, experts, top_k, hidden, self.elem,
                                       tokens_per_rank, n_cap_rows, relay_groups, int(grad),
                                       ctypes.byref(h)),
                   "hm_world_create")
        self.relay_groups = relay_groups
        self._h = h
        info = (ctypes.c_int64 * 8)()
        _lib.check(lib.hm_world_info(h, info), "hm_world_info")
        self.r_cap, self.n_cap, self.row_bytes, self.sym_bytes = info[4], info[5], info[6], info[7]
        self.fused = False
        if gpus > 1:
            self._open_peers(group)

    def _open_peers(self, group) -> None:
        import torch.distributed as dist
        lib = _lib.load()
        n = int(lib.hm_world_ipc_handle_size())
        mine = (ctypes.c_uint8 * n)()
        _lib.check(lib.hm_world_ipc_handle(self._h, mine), "hm_world_ipc_handle")
        allh = exchange_handles(bytes(mine), self.gpu_index, self.gpus, group)
        buf = (ctypes.c_uint8 * len(allh)).from_buffer_copy(allh)
        _lib.check(lib.hm_world_open_peers(self._h, buf), "hm_world_open_peers")
        dist.barrier(group=group)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and _lib._lib is not None:
            _lib._lib.hm_world_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ step
    def dispatch(self, x: torch.Tensor, slot_ids: torch.Tensor, weights: torch.Tensor | None,
                 dedup=True) -> None:
        """Plan + exchange; afterwards each local rank's expert-major rows
        (``xmaj``) hold its experts' inputs.  ``dedup``: True (= "gpu": one
        row per (token, other GPU hit), re-expanded at the destination),
        "remote" (per remote rank), "all" (per rank, incl. this GPU's), or
        False (= "none"), see MODES."""
        self._check_rows(x, slot_ids)
        mode = transport_mode(dedup)
        s = stream_ptr()
        _lib.call("hm_dispatch", self._h, ptr(x), ptr(slot_ids), ptr(weights), mode, s)
        if mode:
            _lib.call("hm_expand", self._h, s)

    def dispatch_meta(self, slot_ids: torch.Tensor, weights: torch.Tensor) -> None:
        """Per-GPU dedup plan + every row's position and receive metadata,
        without moving rows (the overlapped forward: hm_experts_overlap moves
        them inside the expert GEMMs).  Fused dispatch across GPUs only."""
        s = stream_ptr()
        _lib.call("hm_dispatch_plan", self._h, ptr(slot_ids), ptr(weights), MODES["gpu"], s)
        _lib.call("hm_dispatch_meta", self._h, ptr(slot_ids), ptr(weights), s)

    def dispatch_ptr(self, x_ptr: int, slot_ids: torch.Tensor, weights: torch.Tensor,
                     dedup=True) -> None:
        """dispatch() with the payload given as a device pointer to
        [L*T_r, M] rows (e.g. a relay world's receive buffer)."""
        mode = transport_mode(dedup)
        s = stream_ptr()
        _lib.call("hm_dispatch", self._h, x_ptr, ptr(slot_ids), ptr(weights), mode, s)
        if mode:
            _lib.call("hm_expand", self._h, s)

    def combine_into(self, out_ptr: int, slot_ids: torch.Tensor, weights: torch.Tensor,
                     dedup=True) -> None:
        _lib.call("hm_combine", self._h, ptr(weights), ptr(slot_ids), transport_mode(dedup),
                  out_ptr, stream_ptr())

    def combine(self, slot_ids: torch.Tensor, weights: torch.Tensor, dedup=True,
                out: torch.Tensor | None = None,
                addend: torch.Tensor | None = None) -> torch.Tensor:
        """Gate-weighted sum of the expert outputs (``ymaj``) back at the source;
        ``addend`` ([L*T_r, M], payload dtype, e.g. a shared expert's output) is
        added in fp32 before the final rounding."""
        t = self.local * self.tokens_per_rank
        if out is None:
            out = torch.empty((t, self.hidden), dtype=self.dtype, device="cuda")
        if addend is None:
            _lib.call("hm_combine", self._h, ptr(weights), ptr(slot_ids), transport_mode(dedup),
                      ptr(out), stream_ptr())
        else:
            if addend.shape != (t, self.hidden) or addend.dtype != self.dtype \
                    or not addend.is_contiguous():
                raise ValueError(f"addend must be a contiguous [{t}, {self.hidden}] "
                                 f"{self.dtype} tensor")
            _lib.call("hm_combine_add", self._h, ptr(weights), ptr(slot_ids),
                      transport_mode(dedup), ptr(addend), ptr(out), stream_ptr())
        return out

    def dispatch_grad(self, grad_out: torch.Tensor, slot_ids: torch.Tensor,
                      weights: torch.Tensor, dedup=True) -> torch.Tensor:
        """Combine backward: d(out) -> expert-output grads (buffer "gy") and the
        gate grads of direct picks; returns the [T, K] gate-grad tensor (the
        dedup picks' entries are filled by combine_grad)."""
        self._check_rows(grad_out, slot_ids)
        dw = torch.zeros(slot_ids.shape, dtype=torch.float32, device="cuda")
        _lib.call("hm_dispatch_grad", self._h, ptr(grad_out), ptr(slot_ids), ptr(weights),
                  transport_mode(dedup), ptr(dw), stream_ptr())
        return dw

    def combine_grad(self, slot_ids: torch.Tensor, dw: torch.Tensor, dedup=True,
                     out: torch.Tensor | None = None) -> torch.Tensor:
        """Dispatch backward: expert-input grads (buffer "gx") -> token grads."""
        t = self.local * self.tokens_per_rank
        if out is None:
            out = torch.empty((t, self.hidden), dtype=self.dtype, device="cuda")
        _lib.call("hm_combine_grad", self._h, ptr(slot_ids), transport_mode(dedup), ptr(dw),
                  ptr(out), stream_ptr())
        return out

    def barrier(self) -> None:
        _lib.call("hm_world_barrier", self._h, stream_ptr())

    def set_fused(self, enabled: bool) -> None:
        """One GPU: dispatch emits expert-major row indices (buffer "xidx")
        instead of copying rows; the expert GEMM gathers the rows from x
        (ffn.expert_ffn_gather_ptrs).  "xmaj" is then not written."""
        _lib.call("hm_world_set_option", self._h, 10, int(bool(enabled)))
        self.fused = bool(enabled)

    def set_max_blocks(self, n: int) -> None:
        """Cap the exchange kernels' grid at n CTAs (0: 8 per SM)."""
        _lib.call("hm_world_set_option", self._h, 4, int(n))

    def _check_rows(self, x, ids):
        t = self.local * self.tokens_per_rank
        if x.shape != (t, self.hidden) or x.dtype != self.dtype or not x.is_contiguous():
            raise ValueError(f"x must be a contiguous [{t}, {self.hidden}] {self.dtype} tensor")
        if ids.shape != (t, self.top_k) or ids.dtype != torch.int32 or not ids.is_contiguous():
            raise ValueError(f"slot ids must be a contiguous [{t}, {self.top_k}] int32 tensor")

    # --------------------------------------------------------------- buffers
    def buffer(self, kind: str, local_rank: int = 0) -> tuple[int, int]:
        p = ctypes.c_void_p()
        n = ctypes.c_int64()
        _lib.call("hm_world_buffer", self._h, _KIND[kind], local_rank, ctypes.byref(p),
                  ctypes.byref(n))
        return int(p.value or 0), int(n.value)

    def read(self, kind: str, local_rank: int = 0, dtype=torch.uint8, count: int | None = None):
        """Copy (a prefix of) a world buffer into a new device tensor."""
        p, n = self.buffer(kind, local_rank)
        esz = torch.empty((), dtype=dtype).element_size()
        count = n // esz if count is None else count
        out = torch.empty(count, dtype=dtype, device="cuda")
        _lib.call("hm_memcpy", ptr(out), p, count * esz, stream_ptr())
        return out

    def write(self, kind: str, src: torch.Tensor, local_rank: int = 0, offset_bytes: int = 0):
        p, n = self.buffer(kind, local_rank)
        nbytes = src.numel() * src.element_size()
        if offset_bytes + nbytes > n:
            raise ValueError("write exceeds buffer")
        _lib.call("hm_memcpy", p + offset_bytes, ptr(src.contiguous()), nbytes, stream_ptr())

    def counts(self) -> np.ndarray:
        """[G, G+E] count matrix: h[s, d] dedup rows, then c[s, e] selections."""
        return self._count_matrix()[:, :self.ranks + self.experts]

    def gpu_counts(self) -> np.ndarray:
        """[G, P]: rows source rank s sends to GPU q under per-GPU dedup."""
        return self._count_matrix()[:, self.ranks + self.experts:]

    def rows_received_gpu(self) -> int:
        return int(self.read("rows_g", 0, torch.int32).cpu().numpy()[0])

    def _count_matrix(self) -> np.ndarray:
        c = self.read("counts", 0, torch.int32).cpu().numpy()
        return c.reshape(self.ranks, self.ranks + self.experts + self.gpus)

    def rows_received(self) -> np.ndarray:
        """Per local rank: (dedup rows received R, expert-major rows N)."""
        o = self.read("offsets", 0, torch.int32).cpu().numpy()
        return np.stack([o[:self.local], o[64:64 + self.local]], axis=1)

    def check_status(self) -> None:
        st = self.read("status", 0, torch.int32).cpu().numpy()
        if st[0]:
            raise RuntimeError(f"EPWorld: {_STATUS.get(int(st[0]), 'device error')} "
                               f"(status {int(st[0])})")

    def expert_rows(self, local_rank: int, dtype=None) -> torch.Tensor:
        """Copy of the expert-major inputs of a local rank ([N, M])."""
        n = int(self.rows_received()[local_rank, 1])
        dt = self.dtype if dtype is None else dtype
        return self.read("xmaj", local_rank, dt, n * self.hidden).view(n, self.hidden)

    def set_expert_outputs(self, local_rank: int, y: torch.Tensor) -> None:
        self.write("ymaj", y.to(self.dtype), local_rank)


class TwoLevelWorld:
    """HD2 dispatch/combine over a two-level hierarchy [U1, F] (the
    reference's d = 2 variant, traffic.py:144-152 / PAPER.md:238).

    Phase 1 (inter-level-1): one row per (token, level-1 group), sent to the
    rank with the source's local index in that group, carrying the token's
    picks restricted to the group -- exactly propagate_level's copies
    (routing.py:189-215).  Phase 2 (intra-level-1): each relay re-dedups its
    received copies to the ranks of its group.  Combine runs the mirror:
    phase-2 combine into the relay's per-copy rows, phase-1 gather at the
    source.  On one NVSwitch box the hierarchy is virtual (2x4, 4x2 groups).
    """

    def __init__(self, fanouts, experts: int, top_k: int, hidden: int, tokens_per_rank: int,
                 dtype=torch.bfloat16, gpus: int = 1, gpu_index: int = 0, group=None,
                 n_cap_rows: int = 0):
        u1, f = int(fanouts[0]), int(np.prod(fanouts[1:]))
        if len(fanouts) != 2:
            raise ValueError("TwoLevelWorld takes fan-outs [U1, F]")
        ranks = u1 * f
        self.u1, self.f, self.ranks = u1, f, ranks
        self.top_k, self.hidden = top_k, hidden
        self.phase1 = EPWorld(ranks, experts, top_k, hidden, tokens_per_rank, dtype, gpus,
                              gpu_index, group, relay_groups=u1)
        self.phase2 = EPWorld(ranks, experts, top_k, hidden, u1 * tokens_per_rank, dtype, gpus,
                              gpu_index, group, n_cap_rows=n_cap_rows)
        n2 = self.phase2.local * u1 * tokens_per_rank
        self.ids2 = torch.empty((n2, top_k), dtype=torch.int32, device="cuda")
        self.w2 = torch.empty((n2, top_k), dtype=torch.float32, device="cuda")

    def dispatch(self, x, slot_ids, weights, dedup2=True) -> None:
        self.phase1.dispatch(x, slot_ids, weights, dedup="all")
        _lib.call("hm_relay_ids", self.phase1._h, ptr(self.ids2), ptr(self.w2), stream_ptr())
        rx, _ = self.phase1.buffer("recv_x", 0)
        self.phase2.dispatch_ptr(rx, self.ids2, self.w2, dedup=dedup2)

    def combine(self, slot_ids, weights, dedup2=True, out=None):
        comb, _ = self.phase1.buffer("comb", 0)
        self.phase2.combine_into(comb, self.ids2, self.w2, dedup=dedup2)
        return self.phase1.combine(slot_ids, weights, dedup="all", out=out)

    def close(self) -> None:
        self.phase1.close()
        self.phase2.close()
