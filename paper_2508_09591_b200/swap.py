"""Topology-aware expert-swap planning on the GPU (hiera2a ``swap.py`` 0.1.0).

``hm_swap_partials`` gathers, per group cut, the integer sufficient
statistics of the four-case swap analysis (swap.py:1-21, 81-118); the E x E x
g tensors follow elementwise (``hm_swap_tensor``).  The smooth-max cost
matrix and the argmin/exact-max decision run in one kernel each, in numpy's
floating-point operation order, so the chosen pair is the reference's.

``select_swap`` keeps everything on the device -- d* from the time model,
tensors for every level, cost, argmin -- and transfers the result once.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import ptr, stream_ptr
from .routing import DeviceMask, MaskLike, Placement, device_mask, propagate_device
from .topology import LevelParams, Topology
from .traffic import _device_counts, _Model


def smooth_max(x, gamma: float) -> float:
    """max(x) * (sum((x/max)^gamma))^(1/gamma) (swap.py:35-48), on the GPU.

    Limits of the device path (the reference has none): vectors of at most
    256 entries here; ``cost_matrix`` / ``select_swap`` support group cuts of
    at most 64 groups (topologies of up to 64 GPUs) and rows of at most 128
    selected slots (``ValueError`` beyond, never a silent wrong answer)."""
    x = np.asarray(x, dtype=float)
    if x.size == 0:
        raise ValueError("smooth_max of an empty vector")
    if np.any(x < 0):
        raise ValueError("smooth_max requires non-negative entries")
    if gamma < 1:
        raise ValueError(f"gamma must be >= 1, got {gamma}")
    if x.size > 256:
        raise ValueError("smooth_max: vectors longer than 256 are not supported")
    dx = torch.as_tensor(x.reshape(1, -1), device="cuda")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.call("hm_smooth_max_rows", ptr(dx), 1, x.size, float(gamma), ptr(out), stream_ptr())
    return float(out.item())


@dataclass(frozen=True)
class SwapTensors:
    """Per-pair dedup counts (swap.py:60-78): inter[i-1][r,c,k], intra[r,c,k]."""

    inter: tuple
    intra: object
    adjust_ops: int = 0
    dedup_calls: int = 0


class _Partials:
    """Device swap statistics of one group cut (``reduce`` sums them over a
    token-sharded mask before the tensor is built)."""

    def __init__(self, dev: DeviceMask, groups: int, reduce=None, defer: bool = False):
        e = dev.experts
        if groups < 1 or e % groups:
            raise ValueError(f"group count {groups} does not divide {e} experts")
        kw = dict(dtype=torch.int64, device="cuda")
        self.groups = groups
        self.base = torch.empty(groups, **kw)
        self.sel = torch.empty(e, **kw)
        self.hitsel = torch.empty(e * groups, **kw)
        self.lone = torch.empty(e, **kw)
        self.lonesel = torch.empty(e * e, **kw)
        self.flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("hm_swap_partials", ptr(dev.words), dev.num_tokens, e, groups, ptr(self.base),
                  ptr(self.sel), ptr(self.hitsel), ptr(self.lone), ptr(self.lonesel),
                  ptr(self.flag), stream_ptr())
        if reduce is not None:
            for t in (self.base, self.sel, self.hitsel, self.lone, self.lonesel):
                reduce(t)
        self.experts = e
        if not defer:
            self.finish()

    def stats(self):
        """The additive statistics (all-reduced over a token-sharded mask)."""
        return (self.base, self.sel, self.hitsel, self.lone, self.lonesel)

    def finish(self):
        e, groups = self.experts, self.groups
        self.z = torch.empty((e, e, groups), dtype=torch.int64, device="cuda")
        _lib.call("hm_swap_tensor", ptr(self.base), ptr(self.sel), ptr(self.hitsel),
                  ptr(self.lone), ptr(self.lonesel), e, groups, ptr(self.z), stream_ptr())
        return self

    def adjust_ops(self) -> torch.Tensor:
        """The reference's op counter (swap.py:117) as a device scalar."""
        e, g = self.experts, self.groups
        size = e // g
        raises = self.sel[:, None] - self.hitsel.view(e, g)
        grp = torch.arange(e, device="cuda") // size
        other = grp[:, None] != grp[None, :]
        drops = self.lone[:, None] - self.lonesel.view(e, e)
        return raises.sum() * size + (drops * other).sum()


def _build(dev: DeviceMask, topology: Topology, upto: int, reduce=None):
    u = topology.level_group_counts
    inter = [_Partials(dev, u[level], reduce) for level in range(1, upto)]
    intra = _Partials(dev, topology.num_gpus, reduce)
    return inter, intra


def _check_dense(parts) -> None:
    flags = torch.stack([p.flag[0] for p in parts]).cpu()
    if int(flags.max()) != 0:
        raise ValueError("swap planner: a row selects more than 128 slots")


def swap_tensors_incremental(mask: MaskLike, topology: Topology,
                             placement: Placement | None = None,
                             dim: int | None = None) -> SwapTensors:
    """All swap count tensors via the incremental case analysis (swap.py:121-138)."""
    dev = device_mask(mask, placement)
    upto = topology.num_levels if dim is None else dim
    inter, intra = _build(dev, topology, upto)
    parts = inter + [intra]
    _check_dense(parts)
    ops = int(torch.stack([p.adjust_ops() for p in parts]).sum().item())
    as_dev = isinstance(mask, DeviceMask)
    conv = (lambda z: z) if as_dev else (lambda z: z.cpu().numpy())
    return SwapTensors(inter=tuple(conv(p.z) for p in inter), intra=conv(intra.z),
                       adjust_ops=ops)


def swap_tensors_oracle(mask: MaskLike, topology: Topology,
                        placement: Placement | None = None) -> SwapTensors:
    """Brute-force builder (swap.py:141-177): recount every swapped mask on the
    GPU, re-propagating level by level with the per-GPU consistency check."""
    base = device_mask(mask, placement)
    u8 = base.to_bool()
    e = base.experts
    depth = topology.num_levels
    u = topology.level_group_counts
    g = topology.num_gpus
    inter = [np.zeros((e, e, u[i]), dtype=np.int64) for i in range(1, depth)]
    intra = np.zeros((e, e, g), dtype=np.int64)
    calls = 0
    for r in range(e):
        for c in range(r, e):
            perm = torch.arange(e, dtype=torch.int32)
            perm[r], perm[c] = c, r
            words = torch.empty_like(base.words)
            if base.num_tokens:
                _lib.call("hm_mask_pack", ptr(u8), base.num_tokens, e, ptr(perm.cuda()),
                          ptr(words), None, stream_ptr())
            cur = DeviceMask(words, e)
            per_gpu = _device_counts(cur, [g])[0].cpu().numpy()
            calls += 1
            for level in range(1, depth):
                counts = _device_counts(cur, [u[level]])[0].cpu().numpy()
                calls += 1
                inter[level - 1][r, c] = inter[level - 1][c, r] = counts
                cur = propagate_device(cur, u[level], level + 1)
                deeper = _device_counts(cur, [g])[0].cpu().numpy()
                calls += 1
                if not np.array_equal(deeper, per_gpu):
                    raise AssertionError("per-GPU counts changed across levels")
            intra[r, c] = intra[c, r] = per_gpu
    return SwapTensors(inter=tuple(inter), intra=intra, dedup_calls=calls)


def _z_dev(z) -> torch.Tensor:
    if isinstance(z, torch.Tensor):
        return z.to(device="cuda", dtype=torch.int64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(z), dtype=np.int64), device="cuda")


def _launch_cost(inter_z, intra_z, topology: Topology, params: LevelParams, dim_host: int,
                 dim_dev, gamma: float, want_q: bool, want_exact: bool):
    depth = topology.num_levels
    u = topology.level_group_counts
    g = topology.num_gpus
    e = int(intra_z.shape[0])
    n_inter = len(inter_z)
    # the library reads depth - 1 inter entries: cuts past the requested
    # dimension are passed as empty (null tensor, 0 groups)
    pad = max(depth - n_inter, 1)
    inter_ptrs = np.array([ptr(z) for z in inter_z] + [0] * pad, dtype=np.uint64)
    inter_groups = np.array([int(z.shape[2]) for z in inter_z] + [0] * pad, dtype=np.int32)
    inter_part = np.array([u[i] // u[i - 1] for i in range(1, n_inter + 1)] + [0] * pad,
                          dtype=np.int32)
    a_inter = np.array([params.inter(i)[0] for i in range(1, n_inter + 1)] + [0.0] * pad)
    b_inter = np.array([params.inter(i)[1] for i in range(1, n_inter + 1)] + [0.0] * pad)
    intra_ptrs = np.array([ptr(intra_z)] * depth, dtype=np.uint64)
    intra_groups = np.array([g] * depth, dtype=np.int32)
    intra_part = np.array([g // u[d - 1] for d in range(1, depth + 1)], dtype=np.int32)
    a_intra = np.array([params.intra(d - 1)[0] for d in range(1, depth + 1)])
    b_intra = np.array([params.intra(d - 1)[1] for d in range(1, depth + 1)])
    q = torch.empty((e, e), dtype=torch.float64, device="cuda") if want_q else None
    qx = torch.empty((e, e), dtype=torch.float64, device="cuda") if want_exact else None
    _lib.call("hm_swap_cost", inter_ptrs.ctypes.data, inter_groups.ctypes.data,
              inter_part.ctypes.data, a_inter.ctypes.data, b_inter.ctypes.data,
              intra_ptrs.ctypes.data, intra_groups.ctypes.data, intra_part.ctypes.data,
              a_intra.ctypes.data, b_intra.ctypes.data, depth, e, topology.token_bytes(),
              float(gamma), ptr(dim_dev), int(dim_host), ptr(q), ptr(qx), stream_ptr())
    return q, qx


def cost_matrix(tensors: SwapTensors, topology: Topology, params: LevelParams, dim: int,
                gamma: float) -> np.ndarray:
    """Predicted seconds of the dim-D dispatch per swap pair (swap.py:180-206)."""
    if not 1 <= dim <= topology.num_levels:
        raise ValueError(f"dimension {dim} out of range 1..{topology.num_levels}")
    if len(tensors.inter) < dim - 1:
        raise ValueError(f"tensors carry {len(tensors.inter)} inter levels, "
                         f"dimension {dim} needs {dim - 1}")
    inter = [_z_dev(z) for z in tensors.inter[:dim - 1]]
    intra = _z_dev(tensors.intra)
    q, _ = _launch_cost(inter, intra, topology, params, dim, None, gamma, True, False)
    if isinstance(tensors.intra, torch.Tensor):
        return q
    return q.cpu().numpy()


@dataclass(frozen=True)
class SwapPlan:
    """Outcome of one swap-selection step (swap.py:209-223)."""

    cost_matrix: np.ndarray
    pair: tuple[int, int] | None
    predicted_saving: float
    gamma: float
    d_star: int
    no_swap_time: float


def select_swap(mask: MaskLike, topology: Topology, params: LevelParams, gamma: float = 10.0,
                placement: Placement | None = None, group=None) -> SwapPlan:
    """Slot pair minimising the predicted dispatch time (swap.py:226-252).

    Device pipeline: counts -> d* (hm_time_model) -> swap tensors of every
    level -> cost at d* (read on the device) -> argmin + exact-max gate.

    ``group`` (extension): ``mask`` holds only this process's tokens; the
    counts and swap statistics, additive over tokens, are all-reduced over the
    process group (NCCL) and every rank then computes the identical decision
    -- the same result as the reference on the concatenated global mask.
    """
    sharded = False
    if group is not None:
        import torch.distributed as dist
        sharded = dist.get_world_size(group) > 1
    model = _Model(mask, topology, params, placement, True, defer=sharded)
    dev = model.dev
    if sharded:
        # every additive statistic in one flat buffer: one NCCL all-reduce
        # instead of two per count vector and five per cut
        u = topology.level_group_counts
        parts = [_Partials(dev, u[level], defer=True) for level in range(1, topology.num_levels)]
        parts.append(_Partials(dev, topology.num_gpus, defer=True))
        # the too-dense flags ride along, so every rank reaches the same
        # decision (raise or not) before the next collective
        flags = torch.cat([p.flag for p in parts]).to(torch.int64)
        bufs = [model.dedup_dev, model.raw_dev] + [t for p in parts for t in p.stats()] + [flags]
        flat = torch.cat([b.reshape(-1) for b in bufs])
        dist.all_reduce(flat, group=group)
        off = 0
        for b in bufs:
            b.view(-1).copy_(flat[off:off + b.numel()])
            off += b.numel()
        for i, p in enumerate(parts):
            p.flag.copy_(flags[i:i + 1].to(torch.int32))
        model.finish()
        for p in parts:
            p.finish()
        inter, intra = parts[:-1], parts[-1]
    else:
        inter, intra = _build(dev, topology, topology.num_levels, None)
    q, qx = _launch_cost([p.z for p in inter], intra.z, topology, params, topology.num_levels,
                         model.dstar_dev, gamma, True, True)
    out_i = torch.empty(4, dtype=torch.int64, device="cuda")
    out_f = torch.empty(2, dtype=torch.float64, device="cuda")
    _lib.call("hm_swap_select", ptr(q), ptr(qx), dev.experts, ptr(out_i), ptr(out_f), stream_ptr())
    host = torch.cat([out_i, out_f.view(torch.int64), model.dstar_dev.to(torch.int64)]).cpu()
    _check_dense(inter + [intra])
    r, c, chosen = int(host[1]), int(host[2]), int(host[3])
    no_swap = float(host[4:6].view(torch.float64)[0])
    saving = float(host[4:6].view(torch.float64)[1])
    d_star = int(host[6])
    q_out = q.cpu().numpy()
    if not chosen:
        return SwapPlan(q_out, None, 0.0, gamma, d_star, no_swap)
    return SwapPlan(q_out, (r, c), saving, gamma, d_star, no_swap)


def apply_swap(placement: Placement, pair: tuple[int, int] | None) -> Placement:
    """Apply a planned swap; None leaves the placement unchanged (swap.py:255-259)."""
    if pair is None:
        return placement
    return placement.swapped(*pair)
