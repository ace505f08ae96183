"""Routing masks, expert placement and hierarchical propagation on the GPU.

Same names and semantics as hiera2a ``routing.py`` (0.1.0):

* ``RoutingMask`` / ``PropagatedMask`` / ``Placement`` keep the reference's
  fields and validation (routing.py:31-133);
* masks live on the device as packed rows (:class:`DeviceMask`, W =
  ceil(E/32) uint32 words per row); numpy inputs are uploaded once and packed
  by ``hm_mask_pack`` (with the slot gather of ``slot_view``);
* ``propagate_level`` runs ``hm_propagate_count`` + scan + ``hm_propagate_emit``
  and returns the copies in the reference's row-major (row, group) order;
* ``generate_skewed`` / ``generate_uniform`` are the reference's input
  generator restated on numpy's PCG64 stream (the bit stream *is* numpy's, so
  this stays host-side; it is input synthesis, not the hot path);
* trace CSV I/O keeps the reference format (routing.py:218-284).
"""

from __future__ import annotations

import csv
import weakref
from dataclasses import dataclass
from typing import Union

import numpy as np
import torch

from . import _lib
from ._lib import ptr, stream_ptr
from .topology import Topology


class TraceFormatError(ValueError):
    """Malformed routing trace file."""


def layer_seed(base_seed: int, iteration: int, layer: int) -> int:
    """Per-(iteration, layer) seed schedule (routing.py:26-28)."""
    return base_seed + iteration * 65536 + layer


@dataclass(frozen=True)
class RoutingMask:
    """T x E bool selection matrix with exactly ``top_k`` picks per row."""

    bits: np.ndarray
    top_k: int

    def __post_init__(self):
        b = self.bits
        if b.ndim != 2 or b.dtype != np.bool_:
            raise ValueError("bits must be a 2-D boolean array")
        if not 1 <= self.top_k <= self.num_experts:
            raise ValueError(f"top_k={self.top_k} out of range for {self.num_experts} experts")
        counts = b.sum(axis=1)
        bad = np.flatnonzero(counts != self.top_k)
        if bad.size:
            raise ValueError(f"row {bad[0]} selects {counts[bad[0]]} experts, "
                             f"expected {self.top_k}")

    @property
    def num_tokens(self) -> int:
        return self.bits.shape[0]

    @property
    def num_experts(self) -> int:
        return self.bits.shape[1]


@dataclass(frozen=True)
class PropagatedMask:
    """Copies feeding the inter-level-``level`` dispatch (routing.py:59-78)."""

    level: int
    bits: np.ndarray
    origin_token: np.ndarray
    parent_group: np.ndarray

    @property
    def num_rows(self) -> int:
        return self.bits.shape[0]

    @property
    def num_experts(self) -> int:
        return self.bits.shape[1]


class DeviceMask:
    """Packed slot-space rows on the GPU: ``words`` int32 [T, ceil(E/32)].

    Duck-types as a mask for every traffic/swap function (``level``,
    ``num_experts``); ``origin_token`` / ``parent_group`` are device int64
    tensors for propagated masks.
    """

    def __init__(self, words: torch.Tensor, experts: int, level: int = 1,
                 origin_token: torch.Tensor | None = None,
                 parent_group: torch.Tensor | None = None):
        self.words = words
        self.experts = int(experts)
        self.level = int(level)
        self.origin_token = origin_token
        self.parent_group = parent_group

    @property
    def num_tokens(self) -> int:
        return int(self.words.shape[0])

    num_rows = num_tokens

    @property
    def num_experts(self) -> int:
        return self.experts

    def to_bool(self) -> torch.Tensor:
        """Unpack to a T x E uint8 device tensor."""
        t = self.num_tokens
        out = torch.empty((t, self.experts), dtype=torch.uint8, device=self.words.device)
        if t:
            _lib.call("hm_mask_unpack", ptr(self.words), t, self.experts, ptr(out), stream_ptr())
        return out

    def numpy_bits(self) -> np.ndarray:
        return self.to_bool().cpu().numpy().astype(bool)

    @property
    def bits(self) -> np.ndarray:  # reference-compatible view (host copy)
        return self.numpy_bits()


MaskLike = Union[RoutingMask, PropagatedMask, DeviceMask, np.ndarray, torch.Tensor]


def mask_bits(mask: MaskLike) -> np.ndarray:
    """Host bool matrix of any mask (routing.py:84-90)."""
    if isinstance(mask, DeviceMask):
        return mask.numpy_bits()
    bits = getattr(mask, "bits", mask)
    if isinstance(bits, torch.Tensor):
        bits = bits.detach().cpu().numpy()
    bits = np.asarray(bits)
    if bits.dtype != np.bool_:
        bits = bits.astype(bool)
    return bits


def mask_level(mask: MaskLike) -> int:
    return getattr(mask, "level", 1)


@dataclass(frozen=True)
class Placement:
    """slot_to_expert[s] = expert occupying slot s (routing.py:109-133)."""

    slot_to_expert: np.ndarray

    def __post_init__(self):
        perm = np.asarray(self.slot_to_expert)
        if not np.array_equal(np.sort(perm), np.arange(perm.size)):
            raise ValueError("slot_to_expert must be a permutation of 0..E-1")

    @staticmethod
    def identity(num_experts: int) -> "Placement":
        return Placement(np.arange(num_experts))

    @property
    def num_experts(self) -> int:
        return self.slot_to_expert.size

    @property
    def expert_to_slot(self) -> np.ndarray:
        inv = np.empty(self.num_experts, dtype=np.int64)
        inv[np.asarray(self.slot_to_expert)] = np.arange(self.num_experts)
        return inv

    def swapped(self, r: int, c: int) -> "Placement":
        perm = np.array(self.slot_to_expert, copy=True)
        perm[[r, c]] = perm[[c, r]]
        return Placement(perm)


# ---------------------------------------------------------------------------
# device upload with a per-object cache (masks are immutable by contract)

_upload_cache: dict[int, tuple[weakref.ref, torch.Tensor]] = {}


def _cache_get(obj):
    hit = _upload_cache.get(id(obj))
    if hit is not None and hit[0]() is obj:
        return hit[1]
    return None


def _cache_put(obj, tensor) -> None:
    try:
        key = id(obj)
        ref = weakref.ref(obj, lambda _r, k=key: _upload_cache.pop(k, None))
    except TypeError:  # plain ndarrays are not weak-referenceable: no caching
        return
    _upload_cache[key] = (ref, tensor)


def _device_u8(mask) -> tuple[torch.Tensor, int, int]:
    """T x E uint8 device copy of a host/torch mask (cached per mask object)."""
    if isinstance(mask, torch.Tensor):
        t = mask
    else:
        hit = _cache_get(mask) if not isinstance(mask, np.ndarray) else None
        if hit is not None:
            return hit, hit.shape[0], hit.shape[1]
        bits = getattr(mask, "bits", mask)
        if isinstance(bits, torch.Tensor):
            t = bits
        else:
            arr = np.ascontiguousarray(np.asarray(bits))
            if arr.ndim != 2:
                raise ValueError("bits must be a 2-D boolean array")
            if arr.dtype != np.bool_:
                arr = arr.astype(bool)
            t = torch.from_numpy(arr.view(np.uint8))
    if t.ndim != 2:
        raise ValueError("bits must be a 2-D boolean array")
    _lib.load()
    t = t.to(device="cuda", dtype=torch.uint8, non_blocking=True).contiguous()
    if not isinstance(mask, (torch.Tensor, np.ndarray)):
        _cache_put(mask, t)
    return t, t.shape[0], t.shape[1]


def _words(t: int, e: int, device="cuda") -> torch.Tensor:
    return torch.empty((t, (e + 31) // 32), dtype=torch.int32, device=device)


def device_mask(mask: MaskLike, placement: "Placement | None" = None) -> DeviceMask:
    """Slot-space packed device mask of ``mask`` under ``placement``."""
    if isinstance(mask, DeviceMask):
        if placement is None:
            return mask
        if placement.num_experts != mask.num_experts:
            raise ValueError(f"placement covers {placement.num_experts} experts, "
                             f"mask has {mask.num_experts}")
        u8 = mask.to_bool()
        t, e = u8.shape
        level, origin, parent = mask.level, mask.origin_token, mask.parent_group
    else:
        u8, t, e = _device_u8(mask)
        level = mask_level(mask)
        origin = getattr(mask, "origin_token", None)
        parent = getattr(mask, "parent_group", None)
        if origin is not None and not isinstance(origin, torch.Tensor):
            origin = torch.as_tensor(np.asarray(origin, dtype=np.int64), device="cuda")
        if parent is not None and not isinstance(parent, torch.Tensor):
            parent = torch.as_tensor(np.asarray(parent, dtype=np.int64), device="cuda")
    s2e = None
    if placement is not None:
        if placement.num_experts != e:
            raise ValueError(f"placement covers {placement.num_experts} experts, mask has {e}")
        s2e = torch.as_tensor(np.asarray(placement.slot_to_expert, dtype=np.int32), device="cuda")
    words = _words(t, e)
    if t:
        _lib.call("hm_mask_pack", ptr(u8), t, e, ptr(s2e), ptr(words), None, stream_ptr())
    return DeviceMask(words, e, level, origin, parent)


def mask_from_ids(slot_ids: torch.Tensor, experts: int) -> DeviceMask:
    """Packed slot-space mask of K-per-row slot ids (the router's output), on
    the GPU (hm_ids_to_bits); -1 entries are ignored."""
    ids = slot_ids.to(device="cuda", dtype=torch.int32).contiguous()
    t, k = ids.shape
    words = _words(t, experts)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    if t:
        _lib.call("hm_ids_to_bits", ptr(ids), t, k, experts, None, ptr(words), ptr(bad),
                  stream_ptr())
    return DeviceMask(words, experts)


def slot_view(mask: MaskLike, placement: "Placement | None") -> np.ndarray:
    """Host bool matrix re-indexed into slot space (routing.py:98-106)."""
    if placement is None:
        return mask_bits(mask)
    return device_mask(mask, placement).numpy_bits()


def apply_placement(mask: RoutingMask, placement: Placement) -> RoutingMask:
    """Expert-space -> slot-space mask (routing.py:177-186), gathered on the GPU."""
    if placement.num_experts != mask.num_experts:
        raise ValueError(f"placement covers {placement.num_experts} experts, "
                         f"mask has {mask.num_experts}")
    return RoutingMask(device_mask(mask, placement).numpy_bits(), mask.top_k)


def generate_uniform(num_tokens: int, num_experts: int, top_k: int, seed: int) -> RoutingMask:
    return generate_skewed(num_tokens, num_experts, top_k, 0.0, seed)


def generate_skewed(num_tokens: int, num_experts: int, top_k: int, zipf_s: float, seed: int,
                    ranking_seed: int | None = None) -> RoutingMask:
    """Zipf(s) popularity over a seeded ranking; K distinct experts per token by
    exponential race (routing.py:142-174), on numpy's PCG64 stream."""
    if top_k > num_experts:
        raise ValueError(f"top_k={top_k} exceeds expert count {num_experts}")
    if zipf_s < 0:
        raise ValueError(f"zipf_s must be >= 0, got {zipf_s}")
    rng = np.random.default_rng(seed)
    rank_rng = rng if ranking_seed is None else np.random.default_rng(ranking_seed)
    order = rank_rng.permutation(num_experts)
    popularity = np.empty(num_experts)
    popularity[order] = 1.0 / (np.arange(1, num_experts + 1) ** zipf_s)
    bits = np.zeros((num_tokens, num_experts), dtype=bool)
    step = max(1, min(num_tokens, 4_000_000 // max(num_experts, 1)))
    for lo in range(0, num_tokens, step):
        n = min(step, num_tokens - lo)
        race = rng.exponential(size=(n, num_experts)) / popularity
        winners = np.argpartition(race, top_k - 1, axis=1)[:, :top_k]
        bits[lo + np.arange(n)[:, None], winners] = True
    return RoutingMask(bits, top_k)


def _to_host_propagated(dev: DeviceMask) -> PropagatedMask:
    return PropagatedMask(level=dev.level, bits=dev.numpy_bits(),
                          origin_token=dev.origin_token.cpu().numpy(),
                          parent_group=dev.parent_group.cpu().numpy())


def propagate_device(dev: DeviceMask, groups: int, level_out: int) -> DeviceMask:
    """One copy per (row, group hit) with restricted selections, on the GPU."""
    t, e = dev.num_tokens, dev.experts
    dvc = dev.words.device
    copies = torch.empty(max(t, 1), dtype=torch.int64, device=dvc)
    first = torch.empty(max(t, 1), dtype=torch.int64, device=dvc)
    total = torch.zeros(1, dtype=torch.int64, device=dvc)
    s = stream_ptr()
    if t:
        _lib.call("hm_propagate_count", ptr(dev.words), t, e, groups, ptr(copies), s)
        ws = torch.empty(int(_lib.load().hm_scan_workspace(t)) // 8 + 1, dtype=torch.int64, device=dvc)
        _lib.call("hm_scan_i64", ptr(copies), t, ptr(first), ptr(total), ptr(ws), s)
    n = int(total.item())
    out_words = torch.zeros((n, (e + 31) // 32), dtype=torch.int32, device=dvc)
    origin = torch.empty(n, dtype=torch.int64, device=dvc)
    parent = torch.empty(n, dtype=torch.int64, device=dvc)
    if t and n:
        _lib.call("hm_propagate_emit", ptr(dev.words), t, e, groups, ptr(first),
                  ptr(dev.origin_token) if dev.origin_token is not None else None,
                  ptr(out_words), ptr(origin), ptr(parent), s)
    return DeviceMask(out_words, e, level_out, origin, parent)


def propagate_level(mask: MaskLike, topology: Topology):
    """Split every row by the level-l groups it selects (routing.py:189-215)."""
    level = mask_level(mask)
    if level >= topology.num_levels:
        raise ValueError(f"cannot propagate past level {topology.num_levels}")
    dev = device_mask(mask)
    groups = topology.level_group_counts[level]
    if dev.experts % groups:
        raise ValueError(f"group count {groups} does not divide {dev.experts} experts")
    out = propagate_device(dev, groups, level + 1)
    if isinstance(mask, DeviceMask):
        return out
    return _to_host_propagated(out)


def save_placements(placements: dict[int, Placement], experts: int, path) -> None:
    """Per-layer placements -> the reference's placement JSON
    (cli.py:193-198: {"experts": E, "layers": {"<layer>": slot_to_expert}})."""
    import json
    doc = {"experts": int(experts),
           "layers": {str(l): np.asarray(p.slot_to_expert).astype(int).tolist()
                      for l, p in sorted(placements.items())}}
    with open(path, "w") as fh:
        fh.write(json.dumps(doc, indent=2) + "\n")


def load_placements(path, experts: int) -> dict[int, Placement]:
    """Placement JSON -> per-layer placements (cli.py:183-190, same error)."""
    import json
    with open(path) as fh:
        raw = json.load(fh)
    if raw.get("experts") != experts:
        raise ValueError(f"placement file {path} is for {raw.get('experts')} "
                         f"experts, topology has {experts}")
    return {int(layer): Placement(np.array(perm, dtype=int))
            for layer, perm in raw["layers"].items()}


def save_trace(masks: list[tuple[int, int, RoutingMask]], path) -> None:
    """(iteration, layer, mask) triples -> trace CSV (routing.py:218-227)."""
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(["iter", "layer", "token", "experts"])
        for iteration, layer, mask in masks:
            bits = mask_bits(mask)
            for token, row in enumerate(bits):
                out.writerow([iteration, layer, token,
                              ";".join(str(e) for e in np.flatnonzero(row))])


def load_trace(path, num_experts: int) -> list[tuple[int, int, RoutingMask]]:
    """Trace CSV -> (iteration, layer, mask) triples (routing.py:230-284)."""
    entries: list[tuple[int, int, RoutingMask]] = []
    key, rows = None, []

    def flush():
        if key is None:
            return
        bits = np.vstack(rows)
        k = int(rows[0].sum())
        counts = bits.sum(axis=1)
        bad = np.flatnonzero(counts != k)
        if bad.size:
            raise TraceFormatError(f"{path}: iter {key[0]} layer {key[1]} token {bad[0]} "
                                   f"selects {counts[bad[0]]} experts, expected {k}")
        entries.append((key[0], key[1], RoutingMask(bits, k)))

    with open(path, newline="") as fh:
        reader = csv.DictReader(fh)
        want = ["iter", "layer", "token", "experts"]
        if reader.fieldnames is None or [f.strip() for f in reader.fieldnames] != want:
            raise TraceFormatError(f"{path}: expected header 'iter,layer,token,experts', "
                                   f"got {reader.fieldnames}")
        for lineno, row in enumerate(reader, start=2):
            try:
                k2 = (int(row["iter"]), int(row["layer"]))
                token = int(row["token"])
                ids = [int(x) for x in row["experts"].split(";") if x != ""]
            except (TypeError, ValueError, AttributeError) as exc:
                raise TraceFormatError(f"{path}:{lineno}: unparsable row") from exc
            if not ids:
                raise TraceFormatError(f"{path}:{lineno}: token {token} selects no experts")
            if max(ids) >= num_experts or min(ids) < 0:
                raise TraceFormatError(f"{path}:{lineno}: expert id {max(ids)} out of range "
                                       f"for {num_experts} experts")
            if len(set(ids)) != len(ids):
                raise TraceFormatError(f"{path}:{lineno}: duplicate expert ids")
            if k2 != key:
                flush()
                key, rows = k2, []
            if token != len(rows):
                raise TraceFormatError(f"{path}:{lineno}: token ids must be 0..T-1 in order, "
                                       f"got {token}")
            r = np.zeros(num_experts, dtype=bool)
            r[ids] = True
            rows.append(r)
        flush()
    return entries
