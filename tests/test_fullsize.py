"""Parity at the bench's FULL sizes (32,768-token steps; tests/golden/fullsize.json).

The fixtures were produced by running the reference hiera2a package on the
masks bench.py plans on (make_fullsize.py): Qwen3 [8] E=128, DSv3 [2,4] and
[4,2] E=256, and the config-D Zipf(1.2) mask.  Large arrays are compared
through SHA-256 digests of their canonical bytes, so equality is still bit
for bit.  CPU tests pin the mask generator and the oracle; GPU tests run the
product's device path.
"""

from __future__ import annotations

import hashlib
import json
import math
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

from oracle import hiera as O

FIX = json.loads((Path(__file__).resolve().parent / "golden" / "fullsize.json").read_text())
IDS = [c["name"] for c in FIX]


def _np(a):
    """Host numpy view of a result (device tensors are copied back)."""
    if hasattr(a, "detach"):
        return a.detach().cpu().numpy()
    return np.asarray(a)


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(_np(a)).tobytes()).hexdigest()


def _mask_sha(bits) -> str:
    return _sha(np.packbits(_np(bits).astype(bool), axis=1))


def _zsha(z) -> str:
    return _sha(_np(z).astype("<i8"))


def _qsha(q) -> str:
    return _sha(_np(q).astype("<f8"))


@lru_cache(maxsize=None)
def _bits(name: str) -> np.ndarray:
    """Regenerate the case's mask with the PRODUCT's generator (routing.py)."""
    from paper_2508_09591_b200 import routing as R
    c = next(c for c in FIX if c["name"] == name)
    t, e = c["tokens"], c["experts"]
    if "zipf" in name:
        ls = R.layer_seed(0, 0, 0)
        m = R.generate_skewed(t, e, 8, 1.2, ls, ranking_seed=2**48 + ls)
    else:
        m = R.generate_uniform(t, e, 8, 7)
    return m.bits


# ---------------------------------------------------------------- CPU (not gpu)

@pytest.mark.parametrize("case", FIX, ids=IDS)
def test_generator_matches_reference_stream(case):
    """The package's host generator reproduces the reference's PCG64 draw
    bit for bit at full size (routing.py:136-174): whole-mask digest plus the
    first 64 rows stored verbatim."""
    bits = _bits(case["name"])
    assert bits.shape == (case["tokens"], case["experts"])
    head = np.unpackbits(np.asarray(case["mask_head_packed"], np.uint8), axis=1,
                         count=case["experts"]).astype(bool)
    assert np.array_equal(bits[:64], head)
    assert _mask_sha(bits) == case["mask_sha256"]


@pytest.mark.parametrize("case", FIX, ids=IDS)
def test_oracle_counts_times_at_full_size(case):
    """The CPU oracle against the reference at full size: counts at every cut,
    the dedup mask, the copy list, times and d* (exact)."""
    bits, fan = _bits(case["name"]), tuple(case["fanouts"])
    u = O.level_group_counts(fan)
    for g in sorted(set(list(u[1:]) + [O.num_gpus(fan)])):
        assert O.dedup_counts(bits, g).tolist() == case[f"dedup_g{g}"]
        assert O.raw_counts(bits, g).tolist() == case[f"raw_g{g}"]
        assert O.duplication_rate(bits, g) == case[f"duprate_g{g}"]
    assert _mask_sha(O.group_hits(bits, O.num_gpus(fan))) == case["hitG_sha256"]
    p = tuple(tuple(x) for x in case["params"])
    tb = case["embed_dim"] * case["bytes_per_elem"]
    for dedup, tag in ((True, "dedup"), (False, "raw")):
        times, ib, ab = O.all_times(bits, fan, p, tb, dedup)
        assert list(times) == case[f"times_{tag}"]
        assert list(ib) == case[f"inter_bytes_{tag}"]
        assert list(ab) == case[f"intra_bytes_{tag}"]
    d, *_rest, rates = O.optimal_dimension(bits, fan, p, tb)
    assert d == case["d_star"] and list(rates) == case["dup_rate_per_level"]
    cur, origin = bits, None
    for level in range(1, len(fan)):
        cur, origin, parent = O.propagate(cur, u[level], origin)
        assert cur.shape[0] == case[f"prop{level}_rows"]
        assert _mask_sha(cur) == case[f"prop{level}_bits_sha256"]
        assert _zsha(origin) == case[f"prop{level}_origin_sha256"]
        assert _zsha(parent) == case[f"prop{level}_parent_sha256"]


# ---------------------------------------------------------------- GPU (product)

def _topo_params(hm, case):
    topo = hm.build_topology(case["fanouts"], case["experts"], case["embed_dim"],
                             case["bytes_per_elem"])
    a_i, b_i, a_a, b_a = (tuple(x) for x in case["params"])
    return topo, hm.LevelParams(a_i, b_i, a_a, b_a)


@pytest.mark.gpu
@pytest.mark.parametrize("case", FIX, ids=IDS)
def test_gpu_counts_copy_lists_times(hm, case):
    topo, params = _topo_params(hm, case)
    dev = hm.device_mask(_bits(case["name"]))
    u = topo.level_group_counts
    for g in sorted(set(list(u[1:]) + [topo.num_gpus])):
        assert hm.dedup_counts(dev, g, topo).counts.tolist() == case[f"dedup_g{g}"]
        assert hm.raw_counts(dev, g, topo).counts.tolist() == case[f"raw_g{g}"]
        assert hm.duplication_rate(dev, g, topo) == case[f"duprate_g{g}"]
    assert _mask_sha(hm.group_reduce(dev, topo.num_gpus, topo)) == case["hitG_sha256"]
    cur = dev
    for level in range(1, topo.num_levels):
        cur = hm.propagate_level(cur, topo)
        assert cur.num_rows == case[f"prop{level}_rows"]
        assert _mask_sha(cur.bits) == case[f"prop{level}_bits_sha256"]
        assert _zsha(cur.origin_token) == case[f"prop{level}_origin_sha256"]
        assert _zsha(cur.parent_group) == case[f"prop{level}_parent_sha256"]
    from paper_2508_09591_b200 import traffic
    for dedup, tag in ((True, "dedup"), (False, "raw")):
        times, ib, ab = traffic.all_times(dev, topo, params, None, dedup=dedup)
        assert list(times) == case[f"times_{tag}"]
        assert list(ib) == case[f"inter_bytes_{tag}"]
        assert list(ab) == case[f"intra_bytes_{tag}"]
    d, rep = hm.optimal_dimension(dev, topo, params)
    assert d == case["d_star"] and list(rep.dup_rate_per_level) == case["dup_rate_per_level"]
    assert [hm.time_without_dedup(k, dev, topo, params)
            for k in range(1, topo.num_levels + 1)] == case["time_without_dedup"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", FIX, ids=IDS)
def test_gpu_swap_tensors_cost_and_decision(hm, case):
    """Z tensors, every cost matrix (bitwise, numpy's SVML pow) and the swap
    decision at 32,768 tokens -- the decisions bench.py reports."""
    topo, params = _topo_params(hm, case)
    dev = hm.device_mask(_bits(case["name"]))
    st = hm.swap_tensors_incremental(dev, topo)
    assert _zsha(st.intra) == case["zintra_sha256"]
    assert [_zsha(z) for z in st.inter] == case["zinter_sha256"]
    assert st.adjust_ops == case["adjust_ops"]
    for dim in range(1, topo.num_levels + 1):
        for gname, gm in (("g", case["gamma"]), ("inf", math.inf)):
            assert _qsha(hm.cost_matrix(st, topo, params, dim, gm)) == \
                case[f"q_d{dim}_{gname}_sha256"], (dim, gname)
    plan = hm.select_swap(dev, topo, params, case["gamma"])
    assert (list(plan.pair) if plan.pair else None) == case["plan_pair"]
    assert plan.d_star == case["plan_d_star"]
    assert plan.no_swap_time == case["plan_no_swap"]
    assert plan.predicted_saving == case["plan_saving"]
    assert _qsha(plan.cost_matrix) == case["plan_q_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", FIX, ids=IDS)
def test_gpu_transport_choice_follows_reference_rule(hm, case):
    """choose_transport on the full-size mask = the reference's rule on the
    reference's own numbers: d* = pick_dimension(times), and the
    non-deduplicated AlltoAll (time_without_dedup(1)) only when strictly
    faster (traffic.py:188-221, engine.py:159-163)."""
    from paper_2508_09591_b200.transport import choose_transport
    topo, params = _topo_params(hm, case)
    ch = choose_transport(hm.device_mask(_bits(case["name"])), topo, params)
    assert list(ch.times) == case["times_dedup"]
    assert ch.time_without_dedup == case["time_without_dedup"][0]
    assert ch.d_star == case["d_star"]
    best = case["times_dedup"][case["d_star"] - 1]
    want = "none" if case["time_without_dedup"][0] < best else \
        ({1: "remote", 2: "gpu"}[case["d_star"]] if len(case["fanouts"]) > 1 else "gpu")
    assert ch.mode == want
