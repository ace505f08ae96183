"""HierMoELayer: the MoE layer the reference models, executed on B200s.

Forward: router logits -> softmax top-K (``hm_route_topk``,
slot ids through the current Placement) -> dedup dispatch over the EP world
(``hm_dispatch``/``hm_expand``) -> per-local-expert SwiGLU FFN on the
expert-major rows (tcgen05 grouped GEMM, ``hm_expert_ffn``) -> gate-weighted
dedup combine (``hm_combine``).  One process per GPU; the layer owns the
weights of the slots its local EP ranks host.
"""

from __future__ import annotations

import numpy as np
import torch

from .ffn import (FFNBackwardScratch, expert_ffn_backward_multi_ptrs, expert_ffn_backward_ptrs,
                  expert_ffn_multi_ptrs, expert_ffn_ptrs, expert_ffn_save_ptrs, pack_w13)
from . import _lib
from ._lib import ptr, stream_ptr
from .layer import EPWorld, route_group_limited, route_topk
from .migrate import ExpertStore
from .routing import Placement, RoutingMask, load_placements, save_placements, save_trace


class HierMoELayer:
    def __init__(self, ranks: int, experts: int, top_k: int, hidden: int, inter: int,
                 tokens_per_rank: int, gpus: int = 1, gpu_index: int = 0, group=None,
                 dedup=True, seed: int = 0, renormalize: bool = True, grad: bool = False,
                 n_cap_rows: int = 0, layer_index: int = 0, router: str = "softmax",
                 n_group: int = 1, topk_group: int = 1, route_scale: float = 1.0,
                 shared_inter: int = 0, optimizer_state: bool = True, micro_batches: int = 1,
                 transport_params=None, transport_every: int = 50, fused_dispatch=None,
                 overlap: bool = True):
        """``router``: "softmax" (softmax top-K; Qwen3) or "dsv3"
        (DeepSeek-V3 group-limited sigmoid gate: ``n_group`` / ``topk_group``
        / ``route_scale`` and a per-expert score bias).
        ``shared_inter`` > 0 adds a shared SwiGLU expert run on every local
        token on a side stream, overlapped with the dispatch, and summed into
        the combine.  ``optimizer_state`` keeps fp32 master weights and Adam
        moments in the expert store (moved with an expert on a swap).
        ``micro_batches`` > 1 splits every local rank's tokens into that many
        micro-batches, each with its own EP world, issued on separate streams
        so one micro-batch's exchange overlaps another's expert GEMMs (the
        expert weight grads are accumulated over micro-batches).
        ``dedup="auto"``: the transport of a step is chosen by the reference's
        time model on the step's (global) mask every ``transport_every``
        forwards (transport.choose_transport; ``transport_params`` a
        LevelParams or params-JSON path for the runtime [P, L] hierarchy,
        default the packaged B200 fits); the choices are logged in
        ``transport_log``.
        ``fused_dispatch`` (default: on unless ``dedup="all"``): the dispatch
        emits expert-major row indices instead of row copies and GEMM1 gathers
        its rows from x (or, across GPUs, from the receive buffer) by index
        (the backward's dW13 likewise); outputs and gradients are
        bit-identical to the copying dispatch.
        ``overlap`` (default on): with per-GPU dedup across GPUs the token
        rows cross NVLink from an idle warp of the local rows' GEMM1
        (hm_experts_overlap), and in the backward the dispatch backward runs
        on a side stream beside the weight-gradient GEMMs (``bwd_overlap``);
        bit-identical to the serial path."""
        if inter % 128 or hidden % 256 or shared_inter % 128:
            raise ValueError("hidden must be a multiple of 256 and inter / shared_inter of 128")
        if grad and (inter % 256 or shared_inter % 256):
            raise ValueError("backward needs inter / shared_inter multiples of 256 (GEMM tiles)")
        if router not in ("softmax", "dsv3"):
            raise ValueError(f"unknown router {router!r}")
        if micro_batches < 1 or tokens_per_rank % micro_batches:
            raise ValueError("micro_batches must divide tokens_per_rank")
        self.ranks, self.experts, self.top_k = ranks, experts, top_k
        self.hidden, self.inter = hidden, inter
        self.tokens_per_rank = tokens_per_rank
        self.gpus, self.gpu_index = gpus, gpu_index
        self.local = ranks // gpus
        self.e_loc = experts // ranks
        # True / "gpu": per-GPU dedup (forward and backward)
        self.auto_transport = dedup == "auto"
        if self.auto_transport:
            from .topology import load_params
            from .transport import default_params, runtime_topology
            dedup = True
            self.runtime_topo = runtime_topology(ranks, gpus, experts, hidden, 2)
            lv = self.runtime_topo.num_levels
            if transport_params is None:
                transport_params = default_params(gpus, lv)
            elif not hasattr(transport_params, "alpha_intra"):
                transport_params = load_params(transport_params)
            self.transport_params = transport_params
            self.transport_every = max(1, int(transport_every))
            self.transport_log = []
        self.dedup = "gpu" if dedup is True else dedup
        self.renormalize = renormalize
        self.micro_batches = micro_batches
        t_mb = tokens_per_rank // micro_batches
        # every micro-batch world gets the full expert-row capacity: under skewed
        # routing one micro-batch's hot rank can exceed a 1/m share of it
        self.worlds = [EPWorld(ranks, experts, top_k, hidden, t_mb, dtype=torch.bfloat16,
                               gpus=gpus, gpu_index=gpu_index, group=group, grad=grad,
                               n_cap_rows=n_cap_rows) for _ in range(micro_batches)]
        # device status words of every world (capacity overflow 2, barrier
        # timeout 3), copied to pinned host memory after each forward and
        # checked at the next call: no sync on the hot path, no silent drops
        from .migrate import _wrap
        self._status_dev = [_wrap(wd.buffer("status", 0)[0], (4,), torch.int32)
                            for wd in self.worlds]
        self._status_host = torch.zeros(len(self.worlds), 4, dtype=torch.int32).pin_memory()
        self._status_ev = None
        self.strict = False           # True: synchronise and check after every step
        self.world = self.worlds[0]
        # fused dispatch: expert-major row indices instead of row copies (one
        # GPU: into x; N > 1 with per-rank / per-GPU dedup: into x for local
        # picks, into the receive buffers for rows that crossed NVLink)
        self.fused = (self.dedup != "all") if fused_dispatch is None else bool(fused_dispatch)
        if self.fused and self.dedup == "all":
            raise ValueError("the fused dispatch needs a direct transport (not dedup='all')")
        self._x_cur = None
        # dispatch inside the expert GEMMs (hm_experts_overlap): per-GPU dedup
        # across GPUs with the fused dispatch, one micro-batch
        # (profiles/r02/overlap_rotated.jsonl)
        self.overlap = bool(overlap)
        self._cside = torch.cuda.Stream() if grad else None   # dispatch backward beside wgrads
        self.bwd_overlap = True
        self._streams = [None] + [torch.cuda.Stream() for _ in range(micro_batches - 1)]
        self.grad = grad
        # router replicated on every GPU (seeded identically); experts: the
        # slots of local ranks, seeded by global slot so any GPU count builds
        # the same model
        g = torch.Generator(device="cuda").manual_seed(seed)
        self.w_router = torch.randn(experts, hidden, device="cuda", generator=g) * hidden ** -0.5
        self.refresh_router()
        n_loc = self.local * self.e_loc
        n_par = 3 * hidden * inter
        # expert state in a symmetric store: bf16 weights (used by the FFN), fp32
        # master weights and Adam moments (moved with the expert on a swap)
        arrays = {"w13": ((2 * inter, hidden), torch.bfloat16),
                  "w2": ((hidden, inter), torch.bfloat16)}
        if optimizer_state:
            arrays.update({"master": ((n_par,), torch.float32),
                           "adam_m": ((n_par,), torch.float32),
                           "adam_v": ((n_par,), torch.float32)})
        self.store = ExpertStore(n_loc, arrays, gpus=gpus, gpu_index=gpu_index, group=group)
        first = gpu_index * n_loc
        for i in range(n_loc):
            gs = torch.Generator(device="cuda").manual_seed(seed * 100003 + first + i)
            w1 = torch.randn(1, inter, hidden, device="cuda", generator=gs) * hidden ** -0.5
            w3 = torch.randn(1, inter, hidden, device="cuda", generator=gs) * hidden ** -0.5
            w2 = torch.randn(hidden, inter, device="cuda", generator=gs) * inter ** -0.5
            self.store["w13"][i].copy_(pack_w13(w1.to(torch.bfloat16), w3.to(torch.bfloat16))[0])
            self.store["w2"][i].copy_(w2.to(torch.bfloat16))
            if optimizer_state:
                self.store["master"][i].copy_(torch.cat([w1.flatten(), w3.flatten(),
                                                         w2.flatten()]))
        if optimizer_state:
            self.store["adam_m"].zero_()
            self.store["adam_v"].zero_()
        self.router = router
        self.n_group, self.topk_group, self.route_scale = n_group, topk_group, route_scale
        self.score_bias = None
        if router == "dsv3":
            gb = torch.Generator(device="cuda").manual_seed(seed + 17)
            self.score_bias = torch.randn(experts, device="cuda", generator=gb) * 0.01
        self.shared_inter = shared_inter
        self.shared_overlap = True    # shared expert on a side stream beside the exchange
        if shared_inter:
            gsh = torch.Generator(device="cuda").manual_seed(seed * 7919 + 1)
            w1 = torch.randn(1, shared_inter, hidden, device="cuda", generator=gsh) * hidden ** -0.5
            w3 = torch.randn(1, shared_inter, hidden, device="cuda", generator=gsh) * hidden ** -0.5
            self.w13_shared = pack_w13(w1.to(torch.bfloat16), w3.to(torch.bfloat16))[0].contiguous()
            self.w2_shared = (torch.randn(hidden, shared_inter, device="cuda", generator=gsh)
                              * shared_inter ** -0.5).to(torch.bfloat16)
            t_loc = self.local * tokens_per_rank
            self._shared_rows = torch.tensor([t_loc], dtype=torch.int32, device="cuda")
            self._shared_h = torch.empty(t_loc, shared_inter, dtype=torch.bfloat16, device="cuda")
            self._shared_y = torch.empty(t_loc, hidden, dtype=torch.bfloat16, device="cuda")
            self._side = torch.cuda.Stream()
            self._shared_done = torch.cuda.Event()
            if grad:
                self.bwd_shared = FFNBackwardScratch(t_loc, 1, hidden, shared_inter)
                self.dw13_shared = torch.zeros(1, 2 * shared_inter, hidden, dtype=torch.bfloat16,
                                               device="cuda")
                self.dw2_shared = torch.zeros(1, hidden, shared_inter, dtype=torch.bfloat16,
                                              device="cuda")
                self._shared_dx = torch.empty(t_loc, hidden, dtype=torch.bfloat16, device="cuda")
                self._shared_g13 = torch.empty(t_loc, 2 * shared_inter, dtype=torch.bfloat16,
                                               device="cuda")
        self.w13 = self.store["w13"].view(self.local, self.e_loc, 2 * inter, hidden)
        self.w2 = self.store["w2"].view(self.local, self.e_loc, hidden, inter)
        # one launch per GEMM covers every local rank ([L][n_cap] row segments)
        self.hs = [torch.empty(self.local * wd.n_cap, inter, dtype=torch.bfloat16, device="cuda")
                   for wd in self.worlds]
        self.h = self.hs[0]
        self.set_placement(Placement.identity(experts))
        self._saved = None
        self.group = group
        self.layer_index = layer_index
        self.iteration = 0            # forward calls so far (trace "iter" column)
        self._trace = None            # [(iter, expert ids [T_local, K] on device)] when recording
        self.timeline = None          # [(label, event)] of the forward phases when a list
        if grad:
            self.bwd = FFNBackwardScratch(self.local * self.world.n_cap, self.local * self.e_loc,
                                          hidden, inter)
            # the forward keeps GEMM1's pre-activations per local rank (no recompute)
            self.g13s = [torch.empty(self.local, wd.n_cap, 2 * inter, dtype=torch.bfloat16,
                                     device="cuda") for wd in self.worlds]
            self.g13_saved = self.g13s[0]
            self.dw13 = torch.zeros_like(self.w13)
            self.dw2 = torch.zeros_like(self.w2)
            # fp32 router weight grad, padded to the wgrad GEMM's 128-row tiles
            self._dwr_pad = torch.zeros(self._e128, hidden, device="cuda")
            self._wgrad_scratch = None   # split-K partials of the router weight gradient
            self.dw_router = self._dwr_pad[:experts]

    def set_placement(self, placement: Placement) -> None:
        self.placement = placement
        self.expert_to_slot = torch.as_tensor(placement.expert_to_slot, dtype=torch.int32,
                                              device="cuda")

    def apply_swap(self, pair) -> None:
        """Apply a planned slot swap (swap.SwapPlan.pair): the placement and the
        physical expert state (weights + optimizer moments) move together, the
        bytes peer-to-peer when the slots live on different GPUs."""
        if pair is None:
            return
        r, c = int(pair[0]), int(pair[1])
        self.set_placement(self.placement.swapped(r, c))
        self.store.migrate(r, c)   # the backward reads the moved weights as stored

    @staticmethod
    def widen(x: torch.Tensor) -> torch.Tensor:
        """fp32 copy of bf16 activations (16-byte vectorised kernel,
        ``hm_bf16_to_f32``)."""
        if x.dtype != torch.bfloat16:
            return x.float()
        x = x.contiguous()
        xf = torch.empty(x.shape, dtype=torch.float32, device=x.device)
        _lib.call("hm_bf16_to_f32", ptr(x), ptr(xf), x.numel(), stream_ptr())
        return xf

    def refresh_router(self) -> None:
        """bf16 operands of the router GEMMs from the fp32 router weights
        (after a weight update): Wr [E_256][M] (expert rows zero-padded to the
        GEMM's 256-column tile) and Wr^T [M][E_128] (the data gradient's B,
        reduction zero-padded to 128)."""
        e, m = self.experts, self.hidden
        self._e256 = -(-e // 256) * 256
        self._e128 = -(-e // 128) * 128
        wb = self.w_router.to(torch.bfloat16)
        self._wr = torch.zeros(self._e256, m, dtype=torch.bfloat16, device="cuda")
        self._wr[:e] = wb
        self._wrt = torch.zeros(m, self._e128, dtype=torch.bfloat16, device="cuda")
        self._wrt[:, :e] = wb.T
        self._rows = {}

    def _rows_dev(self, t: int) -> torch.Tensor:
        r = self._rows.get(t)
        if r is None:
            r = self._rows[t] = torch.tensor([t], dtype=torch.int32, device="cuda")
        return r

    def router_logits(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """fp32 router logits x . Wr^T on the tcgen05 GEMM (bf16 operands,
        fp32 accumulation, hm_gemm_f32) -- no fp32 copy of x."""
        x = x.contiguous()
        t = x.shape[0]
        if out is None:
            out = torch.empty(t, self.experts, device="cuda")
        if t:
            _lib.call("hm_gemm_f32", ptr(x), t, ptr(self._rows_dev(t)), ptr(self._wr),
                      self._e256, self.hidden, self.experts, ptr(out), self.experts, stream_ptr())
        return out

    def route(self, x: torch.Tensor, logits: torch.Tensor | None = None):
        """Router logits (tcgen05 GEMM) -> top-K picks; ``logits``, if given,
        receives the logits (kept for the backward)."""
        logits = self.router_logits(x, logits)
        if self.router == "dsv3":
            return route_group_limited(logits, self.top_k, self.n_group, self.topk_group,
                                       self.score_bias, self.route_scale, self.expert_to_slot)
        return route_topk(logits, self.top_k, self.expert_to_slot, self.renormalize)

    def route_saved(self, x: torch.Tensor):
        """The forward's routing step: route x and, for a training layer, keep
        what the backward needs (x and the router logits)."""
        self._x_cur = x
        if not self.grad:
            return self.route(x)
        logits = torch.empty(x.shape[0], self.experts, device="cuda")
        slot, w, ex = self.route(x, logits)
        self._saved = (x, logits, slot, w, ex)
        return slot, w, ex

    def shared_forward(self, x: torch.Tensor) -> torch.Tensor:
        """The shared expert on every local token (one-group tcgen05 FFN)."""
        if self.grad:
            expert_ffn_save_ptrs(x.data_ptr(), x.shape[0], self._shared_rows.data_ptr(), 1,
                                 self.w13_shared[None], self.w2_shared[None], self.hidden,
                                 self.shared_inter, self._shared_h, self._shared_y.data_ptr(),
                                 self._shared_g13.data_ptr())
        else:
            expert_ffn_ptrs(x.data_ptr(), x.shape[0], self._shared_rows.data_ptr(), 1,
                            self.w13_shared[None], self.w2_shared[None], self.hidden,
                            self.shared_inter, self._shared_h, self._shared_y.data_ptr())
        return self._shared_y

    def fused_now(self) -> bool:
        """Whether this step's transport supports the fused dispatch (not the
        raw transport across GPUs, whose rows land expert-major on the peer)."""
        return self.fused and (self.gpus == 1 or self.dedup in (True, "gpu", "remote"))

    def overlap_now(self) -> bool:
        """Whether this step runs the exchange inside the expert GEMMs: the
        token rows cross NVLink beside the local rows' GEMM1 tiles and the
        received rows' pre-reduced outputs go back beside the local GEMM2
        (hm_dispatch_meta + hm_experts_overlap)."""
        return (self.overlap and self.gpus > 1 and self.micro_batches == 1
                and self.dedup in (True, "gpu") and self.fused_now()
                and self.local * self.e_loc <= 256)

    def _rows_source(self, wd, x_rows_t: torch.Tensor):
        """(x_ptr, x_rows, idx_ptr, recv_ptr) of the experts' A rows."""
        if not wd.fused:
            return wd.buffer("xmaj", 0)[0], self.local * wd.n_cap, 0, 0
        recv = 0
        if self.gpus > 1:   # rows that crossed NVLink: per-GPU (mode 3) / per-rank receive rows
            recv = wd.buffer("recv_g" if self.dedup in (True, "gpu") else "recv_x", 0)[0]
        return x_rows_t.data_ptr(), x_rows_t.shape[0], wd.buffer("xidx", 0)[0], recv

    def experts_forward(self, mb: int = 0) -> None:
        """SwiGLU FFN of every local rank's experts on its expert-major rows
        (of micro-batch ``mb``'s world), all ranks in one launch per GEMM."""
        wd, h = self.worlds[mb], self.hs[mb]
        p_ne, _ = wd.buffer("n_e", 0)
        first = self.gpu_index * self.local * self.e_loc   # this GPU's first slot
        x_ptr, x_rows, idx, recv = self._rows_source(wd, self._x_cur[self._mb_rows(mb)])
        expert_ffn_multi_ptrs(x_ptr, x_rows, idx, wd.n_cap, self.local, p_ne + 4 * first,
                              self.e_loc, self.w13, self.w2, self.hidden, self.inter, h,
                              wd.buffer("ymaj", 0)[0],
                              self.g13s[mb].data_ptr() if self.grad else 0, recv)

    def _mb_rows(self, mb: int) -> slice:
        n = self.local * self.tokens_per_rank // self.micro_batches
        return slice(mb * n, (mb + 1) * n)

    def _post_status(self) -> None:
        """Queue the copy of every world's status word to pinned host memory."""
        for i, st in enumerate(self._status_dev):
            self._status_host[i].copy_(st, non_blocking=True)
        self._status_ev = torch.cuda.Event()
        self._status_ev.record()
        if self.strict:
            self.check_status()

    def check_status(self) -> None:
        """Raise if the last step's kernels flagged an error: expert-row
        capacity overflow (picks would have been dropped) or a device barrier
        timeout (peer data stale).  Called at the start of every forward /
        backward for the previous step, and after every step when ``strict``."""
        if self._status_ev is None:
            return
        self._status_ev.synchronize()
        st = self._status_host[:, 0]
        if bool((st != 0).any()):
            from .layer import _STATUS
            code = int(st[st != 0][0])
            self._status_host.zero_()
            raise RuntimeError(f"HierMoELayer: {_STATUS.get(code, 'device error')} "
                               f"(status {code}); raise n_cap_rows or check the peers")

    def choose_transport(self, slot: torch.Tensor):
        """The reference's time-model choice (none / per-rank / per-GPU dedup)
        on this step's global mask; every GPU takes the same decision."""
        import torch.distributed as dist
        from .routing import mask_from_ids
        from .transport import choose_transport
        red = None
        if self.gpus > 1:
            red = lambda t: dist.all_reduce(t, group=self.group)  # noqa: E731
        ch = choose_transport(mask_from_ids(slot, self.experts), self.runtime_topo,
                              self.transport_params, None, red, allow_deep=not self.grad)
        self.dedup = ch.mode
        self.transport_log.append((self.iteration, self.dedup, ch))
        return ch

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        self.check_status()
        x = x.contiguous()
        slot, w, ex = self.route_saved(x)
        if self.auto_transport and self.iteration % self.transport_every == 0:
            self.choose_transport(slot)
        if self._trace is not None:
            self._trace.append((self.iteration, ex.clone()))
        self.iteration += 1
        shared = None
        cur = torch.cuda.current_stream()
        if self.shared_inter:   # tensor-bound shared expert beside the link-bound dispatch
            side = self._side if self.shared_overlap else cur
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                shared = self.shared_forward(x)
                self._shared_done.record(side)
        if out is None:
            out = torch.empty_like(x)
        # micro-batch m on stream m, pipelined: dispatch m follows dispatch m-1
        # and combine m follows combine m-1, so the exchange of one micro-batch
        # (NVLink, HBM) runs beside the expert GEMMs of its neighbour (tensor cores)
        prev_d = prev_c = None
        ready = torch.cuda.Event()   # routing done: the point every micro-batch starts from
        ready.record(cur)
        for m in range(self.micro_batches):
            st = self._streams[m]
            if st is not None:
                st.wait_event(ready)
            with torch.cuda.stream(st if st is not None else cur):
                s_m = torch.cuda.current_stream()
                rows = self._mb_rows(m)
                wd = self.worlds[m]
                if prev_d is not None:
                    s_m.wait_event(prev_d)
                self._mark(f"dispatch{m}")
                wd.set_fused(self.fused_now())
                if self.overlap_now():   # rows move inside the expert GEMMs
                    wd.dispatch_meta(slot, w)
                    prev_d = torch.cuda.Event()
                    prev_d.record(s_m)
                    self._mark(f"experts{m}")
                    _lib.call("hm_experts_overlap", wd._h, ptr(x), ptr(self.w13), ptr(self.w2),
                              self.hidden, self.inter, ptr(self.hs[m]),
                              self.g13s[m].data_ptr() if self.grad else None, stream_ptr())
                else:
                    wd.dispatch(x[rows], slot[rows], w[rows], dedup=self.dedup)
                    prev_d = torch.cuda.Event()
                    prev_d.record(s_m)
                    self._mark(f"experts{m}")
                    self.experts_forward(m)   # expert-major rows are local after the dispatch
                self._mark(f"experts{m}_end")
                if shared is not None:
                    s_m.wait_event(self._shared_done)
                if prev_c is not None:
                    s_m.wait_event(prev_c)
                self._mark(f"combine{m}")
                wd.combine(slot[rows], w[rows], dedup=self.dedup, out=out[rows],
                           addend=None if shared is None else shared[rows])
                self._mark(f"combine{m}_end")
                prev_c = torch.cuda.Event()
                prev_c.record(s_m)
        for st in self._streams[1:]:
            cur.wait_stream(st)
        self._post_status()
        return out

    __call__ = forward

    def _mark(self, label: str) -> None:
        if self.timeline is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.timeline.append((label, ev))

    def backward(self, grad_out: torch.Tensor) -> torch.Tensor:
        """Gradients of the last forward: returns dL/dx; accumulates expert
        weight grads (dw13, dw2, slot layout) and the router grad.

        combine bwd (dedup broadcast of dL/dout, replaying the forward plan)
        -> expert FFN bwd (tcgen05) -> dispatch bwd (dedup reduction) ->
        gate bwd (softmax top-K, or the DeepSeek-V3 normalised sigmoid) ->
        router GEMMs (tcgen05); the shared expert's FFN backward runs on a
        side stream beside the routed path, and the dispatch backward beside
        the weight-gradient GEMMs.
        """
        if not self.grad or self._saved is None:
            raise RuntimeError("HierMoELayer.backward needs grad=True and a forward first")
        self.check_status()
        x, logits, slot, w, ex = self._saved
        g = grad_out.contiguous()
        if self.shared_inter:   # shared expert backward beside the routed one
            cur = torch.cuda.current_stream()
            self._side.wait_stream(cur)
            with torch.cuda.stream(self._side):
                expert_ffn_backward_ptrs(x.data_ptr(), x.shape[0], self._shared_rows.data_ptr(),
                                         1, self.w13_shared[None], self.w2_shared[None],
                                         g.data_ptr(), self.hidden,
                                         self.shared_inter, self.bwd_shared,
                                         self._shared_dx.data_ptr(), self.dw13_shared,
                                         self.dw2_shared, self._shared_g13.data_ptr())
                self._shared_done.record(self._side)
        cur = torch.cuda.current_stream()
        dw = torch.empty(slot.shape, dtype=torch.float32, device="cuda")
        dx = torch.empty_like(x)
        ffn_done = None
        ready = torch.cuda.Event()
        ready.record(cur)
        for m in range(self.micro_batches):
            st = self._streams[m]
            if st is not None:
                st.wait_event(ready)
            with torch.cuda.stream(st if st is not None else cur):
                rows = self._mb_rows(m)
                wd = self.worlds[m]
                dw[rows] = wd.dispatch_grad(g[rows], slot[rows], w[rows], dedup=self.dedup)
                if ffn_done is not None:   # weight grads accumulate in micro-batch order
                    torch.cuda.current_stream().wait_event(ffn_done)
                p_ne, _ = wd.buffer("n_e", 0)
                first = self.gpu_index * self.local * self.e_loc
                x_ptr, x_rows, idx, recv = self._rows_source(wd, x[rows])
                args = (x_ptr, x_rows, idx, wd.n_cap, self.local, p_ne + 4 * first, self.e_loc,
                        self.w13, self.w2, wd.buffer("gy", 0)[0], self.hidden, self.inter,
                        self.bwd, wd.buffer("gx", 0)[0], self.dw13, self.dw2,
                        self.g13s[m].data_ptr())
                if self.micro_batches == 1 and self.bwd_overlap:
                    # data gradients, then the dispatch backward of gx (HBM /
                    # NVLink) on a side stream beside the weight-gradient GEMMs
                    # (tensor cores), which read only the FFN's own scratch
                    s_m = torch.cuda.current_stream()
                    expert_ffn_backward_multi_ptrs(*args, recv_ptr=recv, parts=1,
                                                   h_fwd=self.hs[m])
                    self._cside.wait_stream(s_m)
                    with torch.cuda.stream(self._cside):
                        wd.combine_grad(slot[rows], dw[rows], dedup=self.dedup, out=dx[rows])
                    expert_ffn_backward_multi_ptrs(*args, recv_ptr=recv, parts=2,
                                                   h_fwd=self.hs[m])
                    s_m.wait_stream(self._cside)
                    continue
                expert_ffn_backward_multi_ptrs(*args, accumulate=m > 0, recv_ptr=recv,
                                               h_fwd=self.hs[m])
                ffn_done = torch.cuda.Event()
                ffn_done.record()
                wd.combine_grad(slot[rows], dw[rows], dedup=self.dedup, out=dx[rows])
        for st in self._streams[1:]:
            cur.wait_stream(st)
        # gate backward on the device (dense bf16 dlogits, zero past E), then
        # the router GEMMs on the tcgen05 kernels: dX_r = dlogits . Wr (fp32)
        # and dWr += dlogits^T . x (fp32, accumulated)
        t = x.shape[0]
        mode = 2 if self.router == "dsv3" else (0 if self.renormalize else 1)
        dlogits = torch.empty(t, self._e128, dtype=torch.bfloat16, device="cuda")
        _lib.call("hm_gate_backward", ptr(logits), ptr(ex), ptr(w), ptr(dw), t, self.experts,
                  self.top_k, mode, float(self.route_scale), ptr(dlogits), self._e128,
                  stream_ptr())
        rows = self._rows_dev(t)
        # split over the token range (an E x M gradient is only a few output
        # tiles); the fp32 partials live in a layer-owned scratch
        need = int(_lib.load().hm_wgrad_f32_scratch_bytes(t, self._e128, self.hidden))
        if need and (self._wgrad_scratch is None or self._wgrad_scratch.numel() < need):
            self._wgrad_scratch = torch.empty(need, dtype=torch.uint8, device="cuda")
        _lib.call("hm_wgrad_f32_split", ptr(dlogits), ptr(x), t, ptr(rows), self._e128,
                  self.hidden, ptr(self._dwr_pad), self.hidden, 1,
                  ptr(self._wgrad_scratch) if need else None, need, stream_ptr())
        shared_dx = None
        if self.shared_inter:
            torch.cuda.current_stream().wait_event(self._shared_done)
            shared_dx = self._shared_dx
        if dx.dtype != torch.bfloat16:
            dxf = torch.empty(t, self.hidden, device="cuda")
            _lib.call("hm_gemm_f32", ptr(dlogits), t, ptr(rows), ptr(self._wrt), self.hidden,
                      self._e128, self.hidden, ptr(dxf), self.hidden, stream_ptr())
            out = dxf + dx
            return out if shared_dx is None else out + shared_dx
        # ((router term dlogits . Wr + dx) + shared dx) in fp32, rounded once
        # to bf16 in the router GEMM's epilogue
        out = torch.empty_like(dx)
        _lib.call("hm_gemm_add_bf16", ptr(dlogits), t, ptr(rows), ptr(self._wrt), self.hidden,
                  self._e128, ptr(dx), ptr(shared_dx), ptr(out), self.hidden, stream_ptr())
        return out

    # --- routing traces and placements in the reference's file formats ---
    def record_trace(self, enabled: bool = True) -> None:
        """Keep every forward's expert ids (device copies) for save_trace."""
        self._trace = [] if enabled else None

    def routing_masks(self) -> list:
        """(iteration, layer, RoutingMask) of the recorded forwards in expert
        space; the mask is the global one (all GPUs' tokens, rank order,
        SPEC.md:310) -- token shards are all-gathered over ``group``."""
        import torch.distributed as dist
        out = []
        for it, ex in self._trace or []:
            if self.gpus > 1:
                parts = [torch.empty_like(ex) for _ in range(self.gpus)]
                dist.all_gather(parts, ex, group=self.group)
                ex = torch.cat(parts)
            ids = ex.cpu().numpy()
            bits = np.zeros((ids.shape[0], self.experts), dtype=bool)
            np.put_along_axis(bits, ids.astype(np.int64), True, axis=1)
            out.append((it, self.layer_index, RoutingMask(bits, self.top_k)))
        return out

    def save_trace(self, path) -> None:
        """Recorded routing as the reference's trace CSV (routing.py:218-227),
        readable by its analyze / plan / simulate commands."""
        save_trace(self.routing_masks(), path)

    def save_placement(self, path) -> None:
        """This layer's placement as the reference's placement JSON (cli.py:193-198)."""
        save_placements({self.layer_index: self.placement}, self.experts, path)

    def load_placement(self, path) -> None:
        """Adopt a planned placement (the reference's `plan --out-placement`):
        every slot whose expert changes is migrated with its optimizer state."""
        target = load_placements(path, self.experts).get(self.layer_index)
        if target is None:
            return
        cur = np.asarray(self.placement.slot_to_expert).copy()
        want = np.asarray(target.slot_to_expert)
        for s in range(self.experts):        # selection sort by swaps
            if cur[s] == want[s]:
                continue
            t = int(np.flatnonzero(cur == want[s])[0])
            self.apply_swap((min(s, t), max(s, t)))
            cur[[s, t]] = cur[[t, s]]

    def flops_per_forward(self) -> int:
        """Expert FFN flops of this GPU's last forward (6 * rows * hidden * inter)."""
        rows = sum(int(wd.rows_received()[:, 1].sum()) for wd in self.worlds)
        return 6 * rows * self.hidden * self.inter

    def close(self) -> None:
        for wd in self.worlds:
            wd.close()
        self.store.close()
