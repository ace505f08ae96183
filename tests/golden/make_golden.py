"""Generate golden vectors by running the REFERENCE ``hiera2a`` package.

Run in the build container only (it reads /root/reference, which does not
exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed, small):
  tests/golden/cases.npz       seeded masks + reference outputs per case
  tests/golden/cases.json      per-case scalars (d*, times, pairs, savings ...)
  tests/golden/sims.json       engine aggregates (smoke_sim, criterion-6 run)

Masks are stored as packed bits (``np.packbits`` along the expert axis).
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import hiera2a as H  # noqa: E402
from hiera2a import routing as HR  # noqa: E402
from hiera2a import traffic as HT  # noqa: E402
from hiera2a import swap as HS  # noqa: E402
from hiera2a.engine import SimConfig, run_simulation  # noqa: E402

OUT = Path(__file__).resolve().parent


def rparams(rng, depth):
    return H.LevelParams(
        alpha_inter=tuple(float(rng.uniform(0.0, 1e-4)) for _ in range(depth - 1)),
        beta_inter=tuple(float(rng.uniform(1e-8, 1e-6)) for _ in range(depth - 1)),
        alpha_intra=tuple(float(rng.uniform(0.0, 1e-4)) for _ in range(depth)),
        beta_intra=tuple(float(rng.uniform(1e-9, 1e-7)) for _ in range(depth)),
    )


def ptuple(p):
    return [list(p.alpha_inter), list(p.beta_inter), list(p.alpha_intra), list(p.beta_intra)]


def main():
    arrays: dict[str, np.ndarray] = {}
    meta: list[dict] = []

    def add_case(name, fanouts, experts, bits, params, placement=None,
                 gamma=10.0, embed=8, bpe=2, full=True, store_q=True):
        topo = H.build_topology(list(fanouts), experts, embed, bpe)
        i = len(meta)
        key = f"c{i}"
        arrays[f"{key}_bits"] = np.packbits(bits, axis=1)
        perm = None
        if placement is not None:
            perm = np.asarray(placement.slot_to_expert)
            arrays[f"{key}_perm"] = perm
        sv = HR.slot_view(bits, placement)
        u = topo.level_group_counts
        rec = {"name": name, "key": key, "fanouts": list(fanouts), "experts": experts,
               "tokens": int(bits.shape[0]), "embed_dim": embed, "bytes_per_elem": bpe,
               "params": ptuple(params), "gamma": gamma, "has_perm": perm is not None}
        # counting at every level cut and per GPU (traffic.py:58-90)
        for g in sorted(set(list(u[1:]) + [topo.num_gpus])):
            arrays[f"{key}_dedup_g{g}"] = HT.dedup_counts(sv, g, topo).counts
            arrays[f"{key}_raw_g{g}"] = HT.raw_counts(sv, g, topo).counts
            rec[f"duprate_g{g}"] = HT.duplication_rate(sv, g, topo)
        arrays[f"{key}_hitG"] = np.packbits(HT.group_reduce(sv, topo.num_gpus, topo), axis=1)
        # propagation chain (routing.py:189-215)
        cur = sv
        for level in range(1, topo.num_levels):
            cur = HR.propagate_level(cur, topo)
            arrays[f"{key}_prop{level}_bits"] = np.packbits(cur.bits, axis=1)
            arrays[f"{key}_prop{level}_origin"] = cur.origin_token.astype(np.int64)
            arrays[f"{key}_prop{level}_parent"] = cur.parent_group.astype(np.int64)
        # time model (traffic.py:155-221)
        for dedup in (True, False):
            times, ib, ab = HT.all_times(bits, topo, params, placement, dedup=dedup)
            tag = "dedup" if dedup else "raw"
            rec[f"times_{tag}"] = list(times)
            rec[f"inter_bytes_{tag}"] = list(ib)
            rec[f"intra_bytes_{tag}"] = list(ab)
        d_star, rep = HT.optimal_dimension(bits, topo, params, placement)
        rec["d_star"] = d_star
        rec["dup_rate_per_level"] = list(rep.dup_rate_per_level)
        if full:
            st = HS.swap_tensors_incremental(bits, topo, placement)
            arrays[f"{key}_zintra"] = st.intra.astype(np.int32)
            for li, z in enumerate(st.inter):
                arrays[f"{key}_zinter{li + 1}"] = z.astype(np.int32)
            rec["adjust_ops"] = st.adjust_ops
            for dim in range(1, topo.num_levels + 1):
                for gname, gm in (("g", gamma), ("inf", math.inf)):
                    q = HS.cost_matrix(st, topo, params, dim, gm)
                    if store_q:
                        arrays[f"{key}_q_d{dim}_{gname}"] = q
        plan = HS.select_swap(bits, topo, params, gamma, placement)
        rec["plan_pair"] = list(plan.pair) if plan.pair else None
        rec["plan_saving"] = plan.predicted_saving
        rec["plan_d_star"] = plan.d_star
        rec["plan_no_swap"] = plan.no_swap_time
        if store_q:
            arrays[f"{key}_plan_q"] = plan.cost_matrix
        meta.append(rec)

    rng = np.random.default_rng(20261018)

    # 1) config-shaped masks: uniform + zipf, GPU level and 2x4/4x2
    shaped = [
        ("configA_e16_k2", (8,), 16, 2, 4096, 0.0),
        ("qwen3_e128_k8", (8,), 128, 8, 8 * 256, 0.0),
        ("qwen3_zipf12", (8,), 128, 8, 8 * 256, 1.2),
        ("dsv3_2x4", (2, 4), 256, 8, 8 * 128, 0.0),
        ("dsv3_4x2", (4, 2), 256, 8, 8 * 128, 0.0),
    ]
    for name, fan, e, k, t, s in shaped:
        mask = H.generate_skewed(t, e, k, s, int(rng.integers(0, 2**31)),
                                 ranking_seed=(2**48 + 3) if s > 0 else None)
        params = rparams(rng, len(fan))
        placement = H.Placement(rng.permutation(e)) if "zipf" in name else None
        add_case(name, fan, e, mask.bits, params, placement,
                 embed=2048 if e == 128 else (7168 if e == 256 else 256),
                 store_q=(e <= 128))

    # 2) small random instances over the reference test pools
    pools = [(2,), (4,), (8,), (2, 2), (2, 1), (4, 2), (2, 4), (2, 2, 2), (4, 2, 2), (2, 2, 1)]
    for i in range(120):
        fan = pools[int(rng.integers(0, len(pools)))]
        g = int(np.prod(fan))
        e = g * int(rng.integers(1, 5))
        if e < 2:
            e = 2 * g
        k = int(rng.integers(1, min(e, 6) + 1))
        t = int(rng.integers(0, 120))
        s = float(rng.choice([0.0, 1.0, 1.5]))
        mask = H.generate_skewed(t, e, k, s, int(rng.integers(0, 2**31)))
        bits = mask.bits
        if i % 7 == 3 and t > 0:   # variable-popcount rows (helpers.random_mask_bits)
            bits = rng.random((t, e)) < rng.uniform(0.1, 0.6)
            empty = ~bits.any(axis=1)
            bits[empty, rng.integers(0, e, size=int(empty.sum()))] = True
        placement = H.Placement(rng.permutation(e)) if rng.random() < 0.5 else None
        add_case(f"rand{i}", fan, e, bits, rparams(rng, len(fan)), placement,
                 gamma=float(rng.choice([10.0, 10.0, 3.0, 17.5])))

    # 3) walkthrough fixture (test_swap.py:62-103)
    rows = [{0}, {1}, {0, 2}, {0, 2}, {1, 3}]
    wb = np.zeros((5, 4), dtype=bool)
    for t, sel in enumerate(rows):
        wb[t, list(sel)] = True
    add_case("walkthrough", (2,), 4, wb, H.LevelParams((), (), (0.0,), (1.0,)), embed=1, bpe=1)

    np.savez_compressed(OUT / "cases.npz", **arrays)
    (OUT / "cases.json").write_text(json.dumps(meta, indent=1) + "\n")

    # 4) engine aggregates that run through the hot-path functions
    cfgdir = Path("/root/reference/pkg/configs")
    topo = H.load_topology(cfgdir / "topology_4x8.json")
    params = H.load_params(cfgdir / "params_4x8.json", topo.num_levels)
    sims = {}
    smoke = SimConfig(topology=topo, params=params, iterations=3, layers=2, tokens=512,
                      routing="uniform", top_k=8, swap_frequency=1, gamma=10.0, base_seed=0)
    c6 = SimConfig(topology=topo, params=params, iterations=6, layers=2, tokens=8192,
                   routing="uniform", top_k=8, swap_frequency=1, gamma=10.0, base_seed=7,
                   strategies=("std", "h2", "hd2", "hd", "hier"))
    zipf = SimConfig(topology=H.build_topology([8], 128, 2048, 2),
                     params=H.LevelParams((), (), (2.0e-5,), (1.3e-12,)),
                     iterations=4, layers=1, tokens=4096, routing="zipf", zipf_s=1.2,
                     top_k=8, swap_frequency=2, gamma=10.0, base_seed=11)
    for name, cfg in (("smoke_sim", smoke), ("criterion6", c6), ("zipf_qwen3", zipf)):
        rep = run_simulation(cfg, threads=1)
        sims[name] = {
            "aggregate": {s: rep.aggregate(s) for s in rep.strategies},
            "cells": [[i, l, s, v] for (i, l, s), v in sorted(rep.seconds.items())],
            "d_star": [[i, l, d] for (i, l), d in sorted(rep.d_star.items())],
            "swap_log": rep.swap_log,
        }
    (OUT / "sims.json").write_text(json.dumps(sims, indent=1) + "\n")
    print("wrote", len(meta), "cases;", sum(a.nbytes for a in arrays.values()) / 1e6, "MB raw")


if __name__ == "__main__":
    main()
