"""Per-level dedup/raw counts, the alpha-beta time model and d* on the GPU.

Same names and results as hiera2a ``traffic.py`` (0.1.0).  One pass of
``hm_level_counts`` produces the dedup and raw histograms of every group cut
the model needs ([U[1..D-1], G]); ``hm_time_model`` evaluates the phase sums
and the two-branch d* rule on the device.

The reference obtains the level-l counts by explicitly propagating the copy
mask (traffic.py:123-141).  Counts of any cut that refines the copies' parent
groups are invariant under propagation -- a copy carries all of its origin
row's selections inside its parent group (routing.py:204-210), and the
reference asserts the per-GPU case itself (swap.py:172-175) -- so the device
counts the original mask directly.  tests/test_oracle.py pins the invariance
on the golden fixtures.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import ptr, stream_ptr
from .routing import DeviceMask, MaskLike, Placement, device_mask, mask_level
from .topology import LevelParams, Topology


@dataclass(frozen=True)
class GroupCounts:
    """Token counts per expert group for one dispatch phase (traffic.py:23-35)."""

    level: int
    group_count: int
    counts: np.ndarray

    def max(self) -> int:
        return int(self.counts.max()) if self.counts.size else 0

    def total(self) -> int:
        return int(self.counts.sum())


@dataclass(frozen=True)
class TrafficReport:
    """Predicted times per dimension + chosen d* (traffic.py:38-55)."""

    times: tuple[float, ...]
    inter_bytes: tuple[int, ...]
    intra_bytes: tuple[int, ...]
    d_star: int
    dup_rate_per_level: tuple[float, ...]

    @property
    def best_time(self) -> float:
        return self.times[self.d_star - 1]


def _check_groups(groups: int, experts: int) -> None:
    if groups < 1 or experts % groups:
        raise ValueError(f"group count {groups} does not divide {experts} experts")


def _device_counts(dev: DeviceMask, cuts: list[int], hit_cut: int | None = None):
    """dedup/raw int64 device vectors (concatenated over cuts) + optional T x g hit mask."""
    e = dev.experts
    for g in cuts:
        _check_groups(g, e)
    n = sum(cuts)
    dedup = torch.empty(n, dtype=torch.int64, device="cuda")
    raw = torch.empty(n, dtype=torch.int64, device="cuda")
    groups = torch.tensor(cuts, dtype=torch.int32)  # host array for the ABI
    hit = None
    if hit_cut is not None:
        hit = torch.empty((dev.num_tokens, cuts[hit_cut]), dtype=torch.uint8, device="cuda")
    _lib.call("hm_level_counts", ptr(dev.words), dev.num_tokens, e, groups.data_ptr(), len(cuts),
              ptr(dedup), ptr(raw), ptr(hit), -1 if hit_cut is None else hit_cut, stream_ptr())
    return dedup, raw, hit


def group_reduce(mask: MaskLike, groups: int, topology: Topology):
    """OR-reduce expert columns into `groups` contiguous groups (traffic.py:58-64)."""
    dev = device_mask(mask)
    _check_groups(groups, dev.experts)
    _, _, hit = _device_counts(dev, [groups], hit_cut=0)
    if isinstance(mask, DeviceMask):
        return hit.bool()
    return hit.cpu().numpy().astype(bool)


def dedup_counts(mask: MaskLike, groups: int, topology: Topology) -> GroupCounts:
    """Rows per group, once per row hitting it (traffic.py:67-71)."""
    dev = device_mask(mask)
    _check_groups(groups, dev.experts)
    dedup, _, _ = _device_counts(dev, [groups])
    return GroupCounts(level=mask_level(mask), group_count=groups, counts=dedup.cpu().numpy())


def raw_counts(mask: MaskLike, groups: int, topology: Topology) -> GroupCounts:
    """Selections per group (traffic.py:74-82)."""
    dev = device_mask(mask)
    _check_groups(groups, dev.experts)
    _, raw, _ = _device_counts(dev, [groups])
    return GroupCounts(level=mask_level(mask), group_count=groups, counts=raw.cpu().numpy())


def duplication_rate(mask: MaskLike, groups: int, topology: Topology) -> float:
    """1 - dedup/raw totals (traffic.py:85-90)."""
    dev = device_mask(mask)
    _check_groups(groups, dev.experts)
    dedup, raw, _ = _device_counts(dev, [groups])
    both = torch.stack([dedup.sum(), raw.sum()]).cpu().tolist()
    if both[1] == 0:
        return 0.0
    return 1.0 - both[0] / both[1]


def bytes_standard(counts: GroupCounts, topology: Topology) -> int:
    if counts.group_count != topology.num_gpus:
        raise ValueError("standard AlltoAll counts must use one group per GPU")
    return topology.num_gpus * counts.max() * topology.token_bytes()


def bytes_inter(level: int, counts: GroupCounts, topology: Topology) -> int:
    u = topology.level_group_counts
    if counts.group_count != u[level]:
        raise ValueError(f"inter-level-{level} counts must cover {u[level]} groups")
    return (u[level] // u[level - 1]) * counts.max() * topology.token_bytes()


def bytes_intra(dim: int, counts: GroupCounts, topology: Topology) -> int:
    if counts.group_count != topology.num_gpus:
        raise ValueError("intra-phase counts must use one group per GPU")
    return (topology.num_gpus // topology.level_group_counts[dim - 1]) * counts.max() \
        * topology.token_bytes()


def model_cuts(topology: Topology) -> list[int]:
    """Group cuts of the phase model: U[1..D-1] then G."""
    return list(topology.level_group_counts[1:]) + [topology.num_gpus]


def _param_arrays(topology: Topology, params: LevelParams):
    d = topology.num_levels
    a_i = [params.inter(i)[0] for i in range(1, d)]
    b_i = [params.inter(i)[1] for i in range(1, d)]
    a_a = [params.intra(i)[0] for i in range(0, d)]
    b_a = [params.intra(i)[1] for i in range(0, d)]
    return a_i, b_i, a_a, b_a


class _Model:
    """Device evaluation of counts + time model for one mask/placement."""

    def __init__(self, mask: MaskLike, topology: Topology, params: LevelParams,
                 placement: Placement | None, dedup: bool = True, reduce=None,
                 defer: bool = False):
        """``defer``: stop after the counts (the caller all-reduces them, e.g.
        batched with the swap statistics, then calls ``finish``)."""
        dev = device_mask(mask, placement)
        if dev.experts != topology.experts:
            # the reference indexes experts through the topology; keep its failure mode
            _check_groups(topology.num_gpus, dev.experts)
        self.dev = dev
        self.cuts = model_cuts(topology)
        dd, raw, _ = _device_counts(dev, self.cuts)
        if reduce is not None:      # token-sharded mask: counts are additive over tokens
            reduce(dd)
            reduce(raw)
        self.dedup_dev, self.raw_dev = dd, raw
        self._args = (topology, params, dedup)
        if not defer:
            self.finish()

    def finish(self):
        topology, params, dedup = self._args
        dd, raw = self.dedup_dev, self.raw_dev
        depth = topology.num_levels
        a_i, b_i, a_a, b_a = _param_arrays(topology, params)
        offs = np.cumsum([0] + self.cuts[:-1]).astype(np.int32)
        offs_dev = torch.as_tensor(offs, device="cuda")
        self.times_dev = torch.empty(depth, dtype=torch.float64, device="cuda")
        self.dstar_dev = torch.empty(1, dtype=torch.int32, device="cuda")
        self.max_dev = torch.empty(depth, dtype=torch.int64, device="cuda")
        u = np.asarray(topology.level_group_counts, dtype=np.int32)
        f64 = lambda v: np.asarray(v if v else [0.0], dtype=np.float64)  # noqa: E731
        ai, bi, aa, ba = f64(a_i), f64(b_i), f64(a_a), f64(b_a)
        _lib.call("hm_time_model", ptr(dd if dedup else raw), u.ctypes.data, depth,
                  topology.num_gpus, topology.token_bytes(), ai.ctypes.data, bi.ctypes.data,
                  aa.ctypes.data, ba.ctypes.data, ptr(offs_dev), ptr(self.times_dev),
                  ptr(self.dstar_dev), ptr(self.max_dev), stream_ptr())
        self.topology = topology
        return self

    def fetch(self):
        """One device->host transfer of everything the API returns."""
        host = torch.cat([self.times_dev.view(torch.int64), self.max_dev,
                          self.dstar_dev.to(torch.int64), self.dedup_dev, self.raw_dev]).cpu()
        d = self.topology.num_levels
        n = sum(self.cuts)
        self.times = tuple(float(x) for x in host[:d].view(torch.float64).tolist())
        self.maxima = [int(x) for x in host[d:2 * d].tolist()]
        self.d_star = int(host[2 * d])
        self.dedup = host[2 * d + 1:2 * d + 1 + n].numpy()
        self.raw = host[2 * d + 1 + n:].numpy()
        return self

    def byte_volumes(self):
        t = self.topology
        u, tb = t.level_group_counts, t.token_bytes()
        inter = tuple((u[i] // u[i - 1]) * self.maxima[i - 1] * tb for i in range(1, t.num_levels))
        intra = tuple((t.num_gpus // u[d - 1]) * self.maxima[-1] * tb
                      for d in range(1, t.num_levels + 1))
        return inter, intra

    def dup_rates(self):
        out, o = [], 0
        for g in self.cuts:
            dd = int(self.dedup[o:o + g].sum())
            rw = int(self.raw[o:o + g].sum())
            out.append(0.0 if rw == 0 else 1.0 - dd / rw)
            o += g
        return tuple(out)


def time_with_dedup(dim: int, mask: MaskLike, topology: Topology, params: LevelParams,
                    placement: Placement | None = None) -> float:
    if not 1 <= dim <= topology.num_levels:
        raise ValueError(f"dimension {dim} out of range 1..{topology.num_levels}")
    return _Model(mask, topology, params, placement, True).fetch().times[dim - 1]


def time_without_dedup(dim: int, mask: MaskLike, topology: Topology, params: LevelParams,
                       placement: Placement | None = None) -> float:
    if not 1 <= dim <= topology.num_levels:
        raise ValueError(f"dimension {dim} out of range 1..{topology.num_levels}")
    return _Model(mask, topology, params, placement, False).fetch().times[dim - 1]


def all_times(mask: MaskLike, topology: Topology, params: LevelParams,
              placement: Placement | None = None, dedup: bool = True):
    """(times, inter_bytes, intra_bytes) for d = 1..D (traffic.py:173-185)."""
    m = _Model(mask, topology, params, placement, dedup).fetch()
    inter, intra = m.byte_volumes()
    return m.times, inter, intra


def pick_dimension(times) -> int:
    """Flat wins only if strictly faster; deep ties -> smallest d (traffic.py:188-199)."""
    times = list(times)
    if len(times) == 1:
        return 1
    deep = min(range(2, len(times) + 1), key=lambda d: (times[d - 1], d))
    return 1 if times[0] < times[deep - 1] else deep


def optimal_dimension(mask: MaskLike, topology: Topology, params: LevelParams,
                      placement: Placement | None = None) -> tuple[int, TrafficReport]:
    """d* plus the traffic report (traffic.py:202-221), evaluated on the GPU."""
    m = _Model(mask, topology, params, placement, True).fetch()
    inter, intra = m.byte_volumes()
    report = TrafficReport(times=m.times, inter_bytes=inter, intra_bytes=intra,
                           d_star=m.d_star, dup_rate_per_level=m.dup_rates())
    return m.d_star, report
