"""GPU parity of the decision path against the reference's golden vectors.

Every comparison is exact: integer counts, copy lists, swap tensors and
decisions bit for bit; times, dup rates and savings as identical doubles.
"""

import math

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu

CASES = G.cases()


def _topo(hm, case):
    return hm.build_topology(case["fanouts"], case["experts"], case["embed_dim"],
                             case["bytes_per_elem"])


def _params(hm, case):
    a_i, b_i, a_a, b_a = G.params(case)
    return hm.LevelParams(tuple(a_i), tuple(b_i), tuple(a_a), tuple(b_a))


def _placement(hm, case):
    p = G.perm(case)
    return None if p is None else hm.Placement(p)


def _slot_bits(case):
    b = G.bits(case)
    p = G.perm(case)
    return b if p is None else b[:, p]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_counts_dedup_mask(hm, case):
    topo = _topo(hm, case)
    sv = _slot_bits(case)
    u = G.level_groups(case)
    for g in sorted(set(list(u[1:]) + [G.gpus(case)])):
        assert np.array_equal(hm.dedup_counts(sv, g, topo).counts, G.arr(case, f"dedup_g{g}"))
        assert np.array_equal(hm.raw_counts(sv, g, topo).counts, G.arr(case, f"raw_g{g}"))
        assert hm.duplication_rate(sv, g, topo) == case[f"duprate_g{g}"]
    hit = hm.group_reduce(sv, G.gpus(case), topo)
    assert np.array_equal(hit, G.unpack(case, "hitG", G.gpus(case)))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_propagation_copy_lists(hm, case):
    topo = _topo(hm, case)
    cur = _slot_bits(case)
    for level in range(1, topo.num_levels):
        cur = hm.propagate_level(cur, topo)
        assert cur.level == level + 1
        assert np.array_equal(cur.bits, G.unpack(case, f"prop{level}_bits", case["experts"]))
        assert np.array_equal(cur.origin_token, G.arr(case, f"prop{level}_origin"))
        assert np.array_equal(cur.parent_group, G.arr(case, f"prop{level}_parent"))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_times_and_dimension(hm, case):
    from paper_2508_09591_b200 import traffic
    topo, params = _topo(hm, case), _params(hm, case)
    mask = G.bits(case)
    pl = _placement(hm, case)
    for dedup, tag in ((True, "dedup"), (False, "raw")):
        times, ib, ab = traffic.all_times(mask, topo, params, pl, dedup=dedup)
        assert list(times) == case[f"times_{tag}"]
        assert list(ib) == case[f"inter_bytes_{tag}"]
        assert list(ab) == case[f"intra_bytes_{tag}"]
    d, rep = hm.optimal_dimension(mask, topo, params, pl)
    assert d == case["d_star"] == rep.d_star
    assert list(rep.dup_rate_per_level) == case["dup_rate_per_level"]


FULL = [c for c in CASES if G.arr(c, "zintra") is not None]


@pytest.mark.parametrize("case", FULL, ids=[c["name"] for c in FULL])
def test_swap_tensors(hm, case):
    topo = _topo(hm, case)
    st = hm.swap_tensors_incremental(G.bits(case), topo, _placement(hm, case))
    assert np.array_equal(st.intra, G.arr(case, "zintra"))
    for li, z in enumerate(st.inter):
        assert np.array_equal(z, G.arr(case, f"zinter{li + 1}"))
    assert st.adjust_ops == case["adjust_ops"]


@pytest.mark.parametrize("case", FULL, ids=[c["name"] for c in FULL])
def test_cost_matrix(hm, case):
    topo, params = _topo(hm, case), _params(hm, case)
    st = hm.swap_tensors_incremental(G.bits(case), topo, _placement(hm, case))
    for dim in range(1, topo.num_levels + 1):
        for gname, gm in (("g", case["gamma"]), ("inf", math.inf)):
            ref = G.arr(case, f"q_d{dim}_{gname}")
            if ref is None:
                continue
            q = hm.cost_matrix(st, topo, params, dim, gm)
            assert np.array_equal(q, ref)              # bitwise, incl. numpy's SVML pow


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_select_swap_decision(hm, case):
    topo, params = _topo(hm, case), _params(hm, case)
    plan = hm.select_swap(G.bits(case), topo, params, case["gamma"], _placement(hm, case))
    assert (list(plan.pair) if plan.pair else None) == case["plan_pair"]
    assert plan.d_star == case["plan_d_star"]
    assert plan.no_swap_time == case["plan_no_swap"]
    assert plan.predicted_saving == case["plan_saving"]


def test_known_answers(hm):
    topo4x2 = hm.build_topology([4, 2], 16, 4, 2)
    b = np.zeros((3, 4), bool)
    for t, s in enumerate([{0, 1}, {0, 2}, {2, 3}]):
        b[t, list(s)] = True
    topo = hm.build_topology([2], 4, 4, 2)
    assert hm.dedup_counts(b, 2, topo).counts.tolist() == [2, 2]
    assert hm.raw_counts(b, 2, topo).counts.tolist() == [3, 3]
    with pytest.raises(ValueError):
        hm.group_reduce(b, 3, topo)
    out = hm.propagate_level(np.eye(16, dtype=bool)[[0]] | np.eye(16, dtype=bool)[[5]], topo4x2)
    assert out.num_rows == 2 and sorted(out.parent_group.tolist()) == [0, 1]
    # walkthrough (test_swap.py:65-103)
    wb = np.zeros((5, 4), bool)
    for t, s in enumerate([{0}, {1}, {0, 2}, {0, 2}, {1, 3}]):
        wb[t, list(s)] = True
    wt = hm.build_topology([2], 4, 1, 1)
    z = hm.swap_tensors_incremental(wb, wt).intra
    assert z[1, 2].tolist() == [3, 2] and z[0, 3].tolist() == [2, 3]
    plan = hm.select_swap(wb, wt, hm.LevelParams((), (), (0.0,), (1.0,)), gamma=10.0)
    assert plan.pair == (0, 3) and plan.no_swap_time == 10.0
    assert hm.smooth_max([5.0], 10) == 5.0
    assert hm.smooth_max([3.0, 1.0, 2.99], math.inf) == 3.0
    assert hm.smooth_max([0.0, 0.0], 10) == 0.0
    # empty mask: times are the alphas, tie goes deep (test_traffic.py:295-304)
    t22 = hm.build_topology([2, 2], 8, 4, 2)
    d, rep = hm.optimal_dimension(np.zeros((0, 8), bool), t22,
                                  hm.LevelParams((0.25,), (1e-7,), (0.75, 0.5), (1e-7, 1e-7)))
    assert rep.times == (0.75, 0.75) and d == 2


def test_bruteforce_builder_matches(hm):
    small = [c for c in FULL if c["experts"] <= 8 and 0 < c["tokens"] <= 40][:6]
    for case in small:
        topo = _topo(hm, case)
        fast = hm.swap_tensors_incremental(G.bits(case), topo, _placement(hm, case))
        slow = hm.swap_tensors_oracle(G.bits(case), topo, _placement(hm, case))
        assert np.array_equal(fast.intra, slow.intra)
        for a, b in zip(fast.inter, slow.inter):
            assert np.array_equal(a, b)
        assert slow.dedup_calls > 0


def test_generator_matches_reference_draw(hm):
    """The package's generate_uniform reproduces the reference's draw
    (tests/golden/fullsize.json; the full 32,768-token masks are checked by
    tests/test_fullsize.py)."""
    import json
    from pathlib import Path
    fx = json.loads((Path(__file__).resolve().parent / "golden" / "fullsize.json").read_text())
    case = fx[0]
    m = hm.generate_uniform(64, case["experts"], 8, 7)
    head = np.unpackbits(np.asarray(case["mask_head_packed"], np.uint8), axis=1,
                         count=case["experts"]).astype(bool)
    # generate_uniform draws in chunks, so the first 64 rows of a 64-token
    # draw are not the head of a 32768-token draw; compare the full draw
    full = hm.generate_uniform(case["tokens"], case["experts"], 8, 7)
    assert np.array_equal(full.bits[:64], head)
    assert m.bits.sum(axis=1).tolist() == [8] * 64


def _svml_numpy() -> bool:
    try:
        from numpy._core._multiarray_umath import __cpu_features__ as f
        return bool(f.get("AVX512_SKX"))
    except Exception:
        return False


@pytest.mark.skipif(not _svml_numpy(), reason="host numpy does not use SVML pow")
def test_device_np_pow_bitwise(hm):
    """The device restatement of numpy's pow equals the host's np.power bit
    for bit (numpy's AVX512_SKX SVML path, numpy_pow.cuh)."""
    import torch
    from paper_2508_09591_b200 import _lib
    rng = np.random.default_rng(21)
    z = rng.integers(0, 1 << 20, 500000)
    m = z + rng.integers(0, 1 << 20, 500000) + 1
    xs = [z / m, rng.uniform(1, 64, 500000), np.exp(rng.uniform(-60, 60, 500000))]
    ys = [np.full(500000, 10.0), np.full(500000, 0.1), rng.uniform(0.02, 30, 500000)]
    for x, y in zip(xs, ys):
        dx, dy = torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda")
        out = torch.empty_like(dx)
        _lib.call("hm_np_pow", dx.data_ptr(), dy.data_ptr(), x.size, out.data_ptr(),
                  _lib.stream_ptr())
        with np.errstate(over="ignore", under="ignore"):
            ref = np.power(x, y)
        assert np.array_equal(out.cpu().numpy(), ref)
