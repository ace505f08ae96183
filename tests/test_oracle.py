"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The oracle (oracle/hiera.py) is only trusted as a checker after it reproduces,
bit for bit, what the reference hiera2a package produced on the same inputs
(tests/golden/make_golden.py) and the reference's own known-answer tests.
"""

import math

import numpy as np
import pytest

import golden_io as G
from oracle import hiera as O
from oracle import moe as OM

CASES = G.cases()


def _sv(case):
    return O.slot_view(G.bits(case), G.perm(case))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_counts_and_masks(case):
    sv = _sv(case)
    u = G.level_groups(case)
    for g in sorted(set(list(u[1:]) + [G.gpus(case)])):
        assert np.array_equal(O.dedup_counts(sv, g), G.arr(case, f"dedup_g{g}"))
        assert np.array_equal(O.raw_counts(sv, g), G.arr(case, f"raw_g{g}"))
        assert O.duplication_rate(sv, g) == case[f"duprate_g{g}"]
    assert np.array_equal(O.group_hits(sv, G.gpus(case)), G.unpack(case, "hitG", G.gpus(case)))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_propagation_copy_lists(case):
    cur, origin = _sv(case), None
    u = G.level_groups(case)
    for level in range(1, len(case["fanouts"])):
        cur, origin, parent = O.propagate(cur, u[level], origin)
        assert np.array_equal(cur, G.unpack(case, f"prop{level}_bits", case["experts"]))
        assert np.array_equal(origin, G.arr(case, f"prop{level}_origin"))
        assert np.array_equal(parent, G.arr(case, f"prop{level}_parent"))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_time_model_and_dimension(case):
    sv, p, tb = _sv(case), G.params(case), G.token_bytes(case)
    for dedup, tag in ((True, "dedup"), (False, "raw")):
        times, ib, ab = O.all_times(sv, tuple(case["fanouts"]), p, tb, dedup)
        assert list(times) == case[f"times_{tag}"]          # exact float equality
        assert list(ib) == case[f"inter_bytes_{tag}"]
        assert list(ab) == case[f"intra_bytes_{tag}"]
    d, *_rest, rates = O.optimal_dimension(sv, tuple(case["fanouts"]), p, tb)
    assert d == case["d_star"]
    assert list(rates) == case["dup_rate_per_level"]


FULL = [c for c in CASES if G.arr(c, "zintra") is not None]


@pytest.mark.parametrize("case", FULL, ids=[c["name"] for c in FULL])
def test_swap_tensors_and_cost(case):
    sv, fan = _sv(case), tuple(case["fanouts"])
    inter, intra = O.swap_tensors(sv, fan)
    assert np.array_equal(intra, G.arr(case, "zintra"))
    for li, z in enumerate(inter):
        assert np.array_equal(z, G.arr(case, f"zinter{li + 1}"))
    p, tb = G.params(case), G.token_bytes(case)
    for dim in range(1, len(fan) + 1):
        for gname, gm in (("g", case["gamma"]), ("inf", math.inf)):
            q_ref = G.arr(case, f"q_d{dim}_{gname}")
            if q_ref is None:
                continue
            q = O.cost_matrix(inter, intra, fan, p, tb, dim, gm)
            assert np.array_equal(q, q_ref)                  # bitwise


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_select_swap(case):
    pair, saving, d, no_swap, q = O.select_swap(_sv(case), tuple(case["fanouts"]),
                                                G.params(case), G.token_bytes(case),
                                                case["gamma"])
    assert (list(pair) if pair else None) == case["plan_pair"]
    assert saving == case["plan_saving"]
    assert d == case["plan_d_star"]
    assert no_swap == case["plan_no_swap"]


def test_bruteforce_equals_incremental_small():
    for case in [c for c in FULL if c["experts"] <= 12 and c["tokens"] <= 60][:15]:
        sv, fan = _sv(case), tuple(case["fanouts"])
        a_inter, a_intra = O.swap_tensors(sv, fan)
        b_inter, b_intra = O.swap_tensors_bruteforce(sv, fan)
        assert np.array_equal(a_intra, b_intra)
        for x, y in zip(a_inter, b_inter):
            assert np.array_equal(x, y)


# ---- reference known-answer tests (cited) ---------------------------------

def _rows(rows, e):
    b = np.zeros((len(rows), e), dtype=bool)
    for t, s in enumerate(rows):
        b[t, list(s)] = True
    return b


def test_known_answers():
    # topology U vectors (test_topology.py:15-20)
    assert O.level_group_counts((4, 2, 2, 2)) == (1, 4, 8, 16)
    # hand counts (test_traffic.py:56-64, 72-74)
    b = _rows([{0, 1}, {0, 2}, {2, 3}], 4)
    assert O.dedup_counts(b, 2).tolist() == [2, 2]
    assert O.raw_counts(b, 2).tolist() == [3, 3]
    assert O.dedup_counts(np.ones((7, 4), bool), 2).tolist() == [7, 7]
    # two-node fixture (test_traffic.py:222-238)
    b = _rows([{16, 17, 18, 19}, {20, 21, 22, 23}], 32)
    assert O.dedup_counts(b, 2).tolist() == [0, 2]
    gc = O.dedup_counts(b, 16)
    assert gc.sum() == 4 and gc[8:12].tolist() == [1, 1, 1, 1]
    p = ((0.0,), (1e-6,), (0.0, 0.0), (1e-6, 1e-9))
    assert O.time_with_dedup(2, b, (2, 8), p, 8) < O.time_with_dedup(1, b, (2, 8), p, 8)
    # d* tie rules (test_traffic.py:295-312)
    assert O.pick_dimension([1.0]) == 1
    assert O.pick_dimension([1.0, 2.0, 3.0]) == 1
    assert O.pick_dimension([2.0, 2.0, 3.0]) == 2
    assert O.pick_dimension([5.0, 3.0, 3.0]) == 2
    assert O.pick_dimension([5.0, 4.0, 3.0]) == 3
    empty = np.zeros((0, 8), bool)
    d, times, *_ = O.optimal_dimension(empty, (2, 2), ((0.25,), (1e-7,), (0.75, 0.5), (1e-7, 1e-7)), 8)
    assert times == (0.75, 0.75) and d == 2
    # propagation {0,5} on [4,2] E=16 (test_routing.py:135-141)
    out, org, par = O.propagate(_rows([{0, 5}], 16), 4)
    assert out.shape[0] == 2 and sorted(par.tolist()) == [0, 1] and org.tolist() == [0, 0]
    # swap walkthrough (test_swap.py:65-103)
    wb = _rows([{0}, {1}, {0, 2}, {0, 2}, {1, 3}], 4)
    _, z = O.swap_tensors(wb, (2,))
    assert z[0, 2].tolist() == [4, 4] and z[1, 3].tolist() == [4, 4]
    assert z[1, 2].tolist() == [3, 2] and z[0, 3].tolist() == [2, 3]
    assert all(z[r, r].tolist() == [5, 3] for r in range(4))
    pair, saving, _, no_swap, _ = O.select_swap(wb, (2,), ((), (), (0.0,), (1.0,)), 1)
    assert pair == (0, 3) and no_swap == 10.0 and saving == 4.0
    # smooth max (test_swap.py:23-59)
    sm = lambda x, g: float(O.smooth_max_lastaxis(np.asarray(x, float)[None], g)[0])
    assert sm([5.0], 10) == 5.0
    assert sm([1.0, 1.0], 10) == pytest.approx(2 ** 0.1)
    assert sm([3.0, 1.0, 2.99], math.inf) == 3.0
    assert sm([0.0, 0.0], 10) == 0.0


def test_moe_plan_matches_reference_counts():
    """The dispatch plan's per-destination histogram is dedup_counts at G and
    its receive order is the row-major copy order (pinned fixture case)."""
    case = next(c for c in CASES if c["name"] == "qwen3_e128_k8")
    bits = G.bits(case)
    ids = np.stack([np.nonzero(r)[0] for r in bits]).astype(np.int32)
    plan = OM.DispatchPlan(ids, 8, 128)
    assert np.array_equal(plan.h.sum(axis=0), G.arr(case, "dedup_g8"))
    assert np.array_equal(plan.c.sum(axis=0).reshape(8, 16).sum(axis=1), G.arr(case, "raw_g8"))
    hit = G.unpack(case, "hitG", 8)
    assert np.array_equal(plan.hit, hit)
    for d in range(8):
        assert np.array_equal(plan.recv_rows(d), np.nonzero(hit[:, d])[0])


def test_route_topk_tie_order():
    logits = np.array([[1.0, 3.0, 3.0, 0.5], [2.0, 2.0, 2.0, 2.0]], np.float32)
    slots, w, ex = OM.route_topk(logits, 2)
    assert ex.tolist() == [[1, 2], [0, 1]]
    assert np.allclose(w.sum(axis=1), 1.0)


def test_cpu_port_step_matches_layer_math():
    """The timed CPU port (bench.py cpu_baseline / --impl reference) computes
    the MoE dispatch+combine step: with identity experts out = sum_k w_k x."""
    import torch
    g = torch.Generator().manual_seed(3)
    T, E, K, M = 700, 64, 6, 96
    logits = torch.randn(T, E, generator=g)
    x = torch.randn(T, M, generator=g).to(torch.bfloat16)
    out, ym, order = OM.cpu_dispatch_combine(logits, x, K, threads=2)
    ids, w, _ = OM.route_topk(logits.numpy(), K)
    # expert-major rows are the picks sorted by slot, source-major inside a slot
    flat = ids.reshape(-1)
    assert np.array_equal(np.sort(flat, kind="stable"), flat[order.numpy()])
    ref = w.sum(axis=1)[:, None] * x.double().numpy()
    np.testing.assert_allclose(out.double().numpy(), ref, rtol=2e-2, atol=2e-2)
    # with non-identity experts: y = 2 x on every expert-major row
    out2, _, _ = OM.cpu_dispatch_combine(logits, x, K, y_major=(ym.float() * 2).to(ym.dtype))
    np.testing.assert_allclose(out2.double().numpy(), 2 * ref, rtol=2e-2, atol=4e-2)
