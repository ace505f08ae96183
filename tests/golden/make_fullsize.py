"""Golden vectors at the bench's FULL sizes, made by running the REFERENCE.

Run in the build container only (reads /root/reference, absent on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fullsize.py

The masks are the ones ``bench.py`` plans on (32,768 tokens = 8 ranks x 4,096):
  * B  -- ``generate_uniform(32768, 128, 8, 7)`` on topology [8]   (Qwen3, configs[1])
  * C  -- ``generate_uniform(32768, 256, 8, 7)`` on topology [2,4] (DSv3, configs[2])
  * C42-- the same DSv3 mask on the virtual 4x2 grouping
  * D  -- ``generate_skewed(32768, 128, 8, 1.2, layer_seed(0,0,0), ranking_seed=2**48+layer_seed(0,0,0))``
          on [8] (the config-D Zipf stress; engine.py:115,130 seeding)
with the B200 alpha/beta the bench uses (tools/calibrate.py fits).

Large arrays are stored as SHA-256 digests of their canonical bytes (masks as
``np.packbits`` rows, Z tensors as little-endian int64, Q as float64), so the
fixture stays a few KB while the GPU tests still compare bit for bit.  Counts,
times, d*, dup rates and the swap decision are stored as values.
Reference functions: routing.py:136-215, traffic.py:58-221, swap.py:81-252.
"""

from __future__ import annotations

import hashlib
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import hiera2a as H  # noqa: E402
from hiera2a import routing as HR  # noqa: E402
from hiera2a import traffic as HT  # noqa: E402
from hiera2a import swap as HS  # noqa: E402

OUT = Path(__file__).resolve().parent
T = 32768

# (alpha_inter, beta_inter, alpha_intra, beta_intra) -- bench.py PLANNER_CASES
P8 = ((), (), (3.36e-5,), (2.84e-13,))
P24 = ((3.14e-5,), (1.80e-13,), (3.36e-5, 3.15e-5), (2.84e-13, 3.59e-13))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def mask_sha(bits: np.ndarray) -> str:
    return sha(np.packbits(bits, axis=1))


def zsha(z: np.ndarray) -> str:
    return sha(np.asarray(z).astype("<i8"))


def qsha(q: np.ndarray) -> str:
    return sha(np.asarray(q, dtype="<f8"))


def case(name, fan, experts, embed, bits, p, gen, gamma=10.0):
    topo = H.build_topology(list(fan), experts, embed, 2)
    params = H.LevelParams(*p)
    u = topo.level_group_counts
    rec = {"name": name, "fanouts": list(fan), "experts": experts, "tokens": int(bits.shape[0]),
           "embed_dim": embed, "bytes_per_elem": 2, "params": [list(x) for x in p],
           "gamma": gamma, "generator": gen, "mask_sha256": mask_sha(bits),
           "mask_head_packed": np.packbits(bits[:64], axis=1).tolist()}
    t0 = time.perf_counter()
    for g in sorted(set(list(u[1:]) + [topo.num_gpus])):
        rec[f"dedup_g{g}"] = HT.dedup_counts(bits, g, topo).counts.tolist()
        rec[f"raw_g{g}"] = HT.raw_counts(bits, g, topo).counts.tolist()
        rec[f"duprate_g{g}"] = HT.duplication_rate(bits, g, topo)
    rec["hitG_sha256"] = mask_sha(HT.group_reduce(bits, topo.num_gpus, topo))
    cur = bits
    for level in range(1, topo.num_levels):
        cur = HR.propagate_level(cur, topo)
        rec[f"prop{level}_rows"] = int(cur.num_rows)
        rec[f"prop{level}_bits_sha256"] = mask_sha(cur.bits)
        rec[f"prop{level}_origin_sha256"] = zsha(cur.origin_token)
        rec[f"prop{level}_parent_sha256"] = zsha(cur.parent_group)
    for dedup in (True, False):
        times, ib, ab = HT.all_times(bits, topo, params, None, dedup=dedup)
        tag = "dedup" if dedup else "raw"
        rec[f"times_{tag}"] = list(times)
        rec[f"inter_bytes_{tag}"] = list(ib)
        rec[f"intra_bytes_{tag}"] = list(ab)
    d_star, rep = HT.optimal_dimension(bits, topo, params, None)
    rec["d_star"] = d_star
    rec["dup_rate_per_level"] = list(rep.dup_rate_per_level)
    rec["time_without_dedup"] = [HT.time_without_dedup(d, bits, topo, params)
                                 for d in range(1, topo.num_levels + 1)]
    st = HS.swap_tensors_incremental(bits, topo, None)
    rec["zintra_sha256"] = zsha(st.intra)
    rec["zinter_sha256"] = [zsha(z) for z in st.inter]
    rec["adjust_ops"] = st.adjust_ops
    for dim in range(1, topo.num_levels + 1):
        for gname, gm in (("g", gamma), ("inf", math.inf)):
            rec[f"q_d{dim}_{gname}_sha256"] = qsha(HS.cost_matrix(st, topo, params, dim, gm))
    plan = HS.select_swap(bits, topo, params, gamma, None)
    rec["plan_pair"] = list(plan.pair) if plan.pair else None
    rec["plan_saving"] = plan.predicted_saving
    rec["plan_d_star"] = plan.d_star
    rec["plan_no_swap"] = plan.no_swap_time
    rec["plan_q_sha256"] = qsha(plan.cost_matrix)
    print(f"{name}: {time.perf_counter() - t0:.1f} s, d*={d_star}, pair={rec['plan_pair']}",
          flush=True)
    return rec


def main():
    b = H.generate_uniform(T, 128, 8, 7).bits
    c = H.generate_uniform(T, 256, 8, 7).bits
    ls = H.layer_seed(0, 0, 0)
    d = H.generate_skewed(T, 128, 8, 1.2, ls, ranking_seed=2**48 + ls).bits
    out = [
        case("B_qwen3_8", (8,), 128, 2048, b, P8, "generate_uniform(32768,128,8,7)"),
        case("C_dsv3_2x4", (2, 4), 256, 7168, c, P24, "generate_uniform(32768,256,8,7)"),
        case("C_dsv3_4x2", (4, 2), 256, 7168, c, P24, "generate_uniform(32768,256,8,7)"),
        case("D_qwen3_zipf12", (8,), 128, 2048, d, P8,
             "generate_skewed(32768,128,8,1.2,layer_seed(0,0,0),ranking_seed=2**48+layer_seed(0,0,0))"),
    ]
    (OUT / "fullsize.json").write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", len(out), "full-size cases")


if __name__ == "__main__":
    main()
