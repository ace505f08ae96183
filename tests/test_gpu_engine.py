"""End-to-end decision parity: replay the reference engine's per-(iteration,
layer) protocol (engine.py:118-191) on the GPU functions and compare every
cell, d* and swap decision with the reference's recorded run (sims.json)."""

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu

RANKING_OFFSET = 2 ** 48  # engine.py:115


def _replay(hm, topo, params, iterations, layers, tokens, top_k, routing, zipf_s,
            swap_frequency, gamma, base_seed, wanted):
    from paper_2508_09591_b200 import traffic
    cells, dstars, swaps = {}, {}, []
    depth = topo.num_levels
    for layer in range(layers):
        placement = hm.Placement.identity(topo.experts)
        for it in range(iterations):
            seed = hm.layer_seed(base_seed, it, layer)
            if routing == "zipf":
                mask = hm.generate_skewed(tokens, topo.experts, top_k, zipf_s, seed,
                                          RANKING_OFFSET + hm.layer_seed(base_seed, 0, layer))
            else:
                mask = hm.generate_skewed(tokens, topo.experts, top_k, 0.0, seed)
            dd, _, _ = traffic.all_times(mask, topo, params, None, dedup=True)
            raw, _, _ = traffic.all_times(mask, topo, params, None, dedup=False)
            if "std" in wanted:
                cells[(it, layer, "std")] = raw[0]
            for d in range(1, depth + 1):
                if f"h{d}" in wanted:
                    cells[(it, layer, f"h{d}")] = raw[d - 1]
                if f"hd{d}" in wanted:
                    cells[(it, layer, f"hd{d}")] = dd[d - 1]
            d_star = traffic.pick_dimension(dd)
            dstars[(it, layer)] = d_star
            if "hd" in wanted:
                cells[(it, layer, "hd")] = dd[d_star - 1]
            if "hier" in wanted:
                if swap_frequency > 0 and it % swap_frequency == 0:
                    plan = hm.select_swap(mask, topo, params, gamma, placement)
                    swaps.append({"iter": it, "layer": layer, "d_star": plan.d_star,
                                  "pair": list(plan.pair) if plan.pair else None,
                                  "predicted_saving_s": plan.predicted_saving})
                    placement = hm.apply_swap(placement, plan.pair)
                _, rep = hm.optimal_dimension(mask, topo, params, placement)
                cells[(it, layer, "hier")] = rep.best_time
    swaps.sort(key=lambda e: (e["iter"], e["layer"]))
    return cells, dstars, swaps


def _check(ref, cells, dstars, swaps):
    ref_cells = {(i, l, s): v for i, l, s, v in ref["cells"]}
    assert set(ref_cells) == set(cells)
    for k, v in ref_cells.items():
        assert cells[k] == v, k
    assert {(i, l): d for i, l, d in ref["d_star"]} == dstars
    assert swaps == ref["swap_log"]
    for s, v in ref["aggregate"].items():
        got = float(np.mean([x for (_, _, name), x in cells.items() if name == s]))
        assert got == v, s


def _cluster(hm):
    topo = hm.build_topology([4, 2, 2, 2], 128, 1024, 2)
    params = hm.LevelParams(alpha_inter=(0.497, 0.301, 0.149),
                            beta_inter=(5.29e-07, 1.17e-07, 2.06e-08),
                            alpha_intra=(0.722, 0.571, 0.114, 0.204),
                            beta_intra=(5.7e-07, 1.27e-07, 2.63e-08, 1.64e-08))
    return topo, params


def test_smoke_sim_replay(hm):
    """pkg/configs/smoke_sim.json on topology_4x8 / params_4x8 (test_output.txt:77-87)."""
    topo, params = _cluster(hm)
    wanted = ["std", "h1", "h2", "h3", "h4", "hd1", "hd2", "hd3", "hd4", "hd", "hier"]
    cells, dstars, swaps = _replay(hm, topo, params, 3, 2, 512, 8, "uniform", 0.0, 1, 10.0, 0,
                                   wanted)
    _check(G.sims()["smoke_sim"], cells, dstars, swaps)


def test_criterion6_replay(hm):
    """Acceptance criterion 6 run (test_acceptance.py:231-250, test_output.txt:38)."""
    topo, params = _cluster(hm)
    cells, dstars, swaps = _replay(hm, topo, params, 6, 2, 8192, 8, "uniform", 0.0, 1, 10.0, 7,
                                   ["std", "h2", "hd2", "hd", "hier"])
    _check(G.sims()["criterion6"], cells, dstars, swaps)


def test_zipf_qwen3_replay(hm):
    topo = hm.build_topology([8], 128, 2048, 2)
    params = hm.LevelParams((), (), (2.0e-5,), (1.3e-12,))
    cells, dstars, swaps = _replay(hm, topo, params, 4, 1, 4096, 8, "zipf", 1.2, 2, 10.0, 11,
                                   ["std", "h1", "hd1", "hd", "hier"])
    _check(G.sims()["zipf_qwen3"], cells, dstars, swaps)
