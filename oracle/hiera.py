"""numpy restatement of the reference decision path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference ``/root/reference/pkg/src/hiera2a`` lines
it restates.  Inputs are plain values so the oracle has no dependency on
either the reference package or the product package:

* ``fanouts``  -- tuple of level fan-outs (``Topology.level_fanouts``)
* ``bits``     -- T x E numpy bool matrix in *slot* space
* ``params``   -- ``(alpha_inter, beta_inter, alpha_intra, beta_intra)`` tuples
                  (``LevelParams`` fields, ``topology.py:134-179``)
* ``token_bytes`` -- ``embed_dim * bytes_per_elem`` (``topology.py:102-103``)

Integer work (hits, counts, copy lists, swap tensors) is restated with integer
arithmetic -- the reference uses float BLAS on 0/1 data, which is exact, so
the two must agree bit for bit.  The floating-point cost model is restated
with the same numpy operations in the same order, because those operations
*define* the rounding the GPU has to reproduce.
"""

from __future__ import annotations

import math

import numpy as np


# --------------------------------------------------------------------------
# topology (topology.py:79-100)

def level_group_counts(fanouts) -> tuple[int, ...]:
    """U vector: U[0] = 1, U[i] = prod(fanouts[:i]) (topology.py:79-89)."""
    u = [1]
    for f in tuple(fanouts)[:-1]:
        u.append(u[-1] * int(f))
    return tuple(u)


def num_gpus(fanouts) -> int:
    return int(math.prod(fanouts))


def group_of_slot(slot, groups: int, experts: int):
    """Group index of a slot when E slots are cut into `groups` (topology.py:95-97)."""
    return np.asarray(slot) * groups // experts


# --------------------------------------------------------------------------
# counting (traffic.py:58-90)

def group_hits(bits: np.ndarray, groups: int) -> np.ndarray:
    """T x g bool: row t selects something in group k (traffic.py:58-64)."""
    t, e = bits.shape
    if groups < 1 or e % groups:
        raise ValueError(f"group count {groups} does not divide {e} experts")
    col_group = np.arange(e) // (e // groups)
    hit = np.zeros((t, groups), dtype=bool)
    rows, cols = np.nonzero(bits)
    hit[rows, col_group[cols]] = True
    return hit


def dedup_counts(bits: np.ndarray, groups: int) -> np.ndarray:
    """Rows per group, one per row hitting it (traffic.py:67-71)."""
    return group_hits(bits, groups).sum(axis=0, dtype=np.int64)


def raw_counts(bits: np.ndarray, groups: int) -> np.ndarray:
    """Selections per group, multiplicity kept (traffic.py:74-82)."""
    t, e = bits.shape
    if groups < 1 or e % groups:
        raise ValueError(f"group count {groups} does not divide {e} experts")
    per_col = bits.sum(axis=0, dtype=np.int64)
    return per_col.reshape(groups, e // groups).sum(axis=1)


def duplication_rate(bits: np.ndarray, groups: int) -> float:
    """1 - dedup/raw over totals (traffic.py:85-90)."""
    raw = int(raw_counts(bits, groups).sum())
    if raw == 0:
        return 0.0
    return 1.0 - int(dedup_counts(bits, groups).sum()) / raw


# --------------------------------------------------------------------------
# hierarchical propagation (routing.py:189-215)

def propagate(bits: np.ndarray, groups: int, origin: np.ndarray | None = None):
    """One copy per (row, group hit), row-major order, restricted selections.

    Returns ``(copy_bits, origin_token, parent_group)``; ``groups`` is the
    level-l group count U[l] of the mask's level l (routing.py:196-215).
    """
    t, e = bits.shape
    hit = group_hits(bits, groups)
    rows, grp = np.nonzero(hit)                      # row-major (row, group)
    size = e // groups
    col_group = np.arange(e) // size
    out = bits[rows] & (col_group[None, :] == grp[:, None])
    org = rows if origin is None else np.asarray(origin)[rows]
    return out, org.astype(np.int64), grp.astype(np.int64)


# --------------------------------------------------------------------------
# volume + time model (traffic.py:93-199)

def _time_for_dim(dim, inter_max, intra_max, fanouts, params, token_bytes) -> float:
    """Eq.1/3/6 phase sum, same op order as traffic.py:144-152."""
    a_inter, b_inter, a_intra, b_intra = params
    u = level_group_counts(fanouts)
    g = num_gpus(fanouts)
    total = 0.0
    for level in range(1, dim):
        vol = (u[level] // u[level - 1]) * inter_max[level - 1] * token_bytes
        total += vol * b_inter[level - 1] + a_inter[level - 1]
    vol = (g // u[dim - 1]) * intra_max[dim - 1] * token_bytes
    total += vol * b_intra[dim - 1] + a_intra[dim - 1]
    return total


def phase_counts(bits, fanouts, dedup=True, upto=None):
    """inter[i-1] at U[i] of the level-i copy mask; intra[d-1] per GPU of the
    level-d copy mask (traffic.py:123-141), computed by explicit propagation."""
    counter = dedup_counts if dedup else raw_counts
    u = level_group_counts(fanouts)
    g = num_gpus(fanouts)
    depth = len(fanouts) if upto is None else upto
    cur, origin = bits, None
    inter, intra = [], [counter(cur, g)]
    for level in range(1, depth):
        inter.append(counter(cur, u[level]))
        cur, origin, _ = propagate(cur, u[level], origin)
        intra.append(counter(cur, g))
    return inter, intra


def all_times(bits, fanouts, params, token_bytes, dedup=True):
    """(times, inter_bytes, intra_bytes) for d = 1..D (traffic.py:173-185)."""
    depth = len(fanouts)
    u = level_group_counts(fanouts)
    g = num_gpus(fanouts)
    inter, intra = phase_counts(bits, fanouts, dedup, depth)
    imax = [int(c.max()) if c.size else 0 for c in inter]
    amax = [int(c.max()) if c.size else 0 for c in intra]
    times = tuple(_time_for_dim(d, imax, amax, fanouts, params, token_bytes)
                  for d in range(1, depth + 1))
    inter_bytes = tuple((u[i] // u[i - 1]) * imax[i - 1] * token_bytes
                        for i in range(1, depth))
    intra_bytes = tuple((g // u[d - 1]) * amax[d - 1] * token_bytes
                        for d in range(1, depth + 1))
    return times, inter_bytes, intra_bytes


def time_with_dedup(dim, bits, fanouts, params, token_bytes) -> float:
    inter, intra = phase_counts(bits, fanouts, True, dim)
    imax = [int(c.max()) if c.size else 0 for c in inter]
    amax = [int(c.max()) if c.size else 0 for c in intra]
    return _time_for_dim(dim, imax, amax, fanouts, params, token_bytes)


def pick_dimension(times) -> int:
    """Flat wins only when strictly faster; deep ties -> smallest d
    (traffic.py:188-199)."""
    times = list(times)
    if len(times) == 1:
        return 1
    deep = min(range(2, len(times) + 1), key=lambda d: (times[d - 1], d))
    return 1 if times[0] < times[deep - 1] else deep


def optimal_dimension(bits, fanouts, params, token_bytes):
    """(d*, times, inter_bytes, intra_bytes, dup_rates) (traffic.py:202-221)."""
    times, ib, ab = all_times(bits, fanouts, params, token_bytes, True)
    u = level_group_counts(fanouts)
    rates, cur, origin = [], bits, None
    for level in range(1, len(fanouts)):
        rates.append(duplication_rate(cur, u[level]))
        cur, origin, _ = propagate(cur, u[level], origin)
    rates.append(duplication_rate(cur, num_gpus(fanouts)))
    return pick_dimension(times), times, ib, ab, tuple(rates)


# --------------------------------------------------------------------------
# swap tensors (swap.py:81-177)

def swap_tensor(bits: np.ndarray, groups: int) -> np.ndarray:
    """E x E x g per-pair dedup counts via the four-case analysis (swap.py:81-118),
    restated with integer counts:

    Z[a,b,k] = base[k] + d[a,b,k] + d[b,a,k],
    d[a,b,k] = raises[a,k]*[grp(b)=k] - drops[a,b]*[grp(a)=k]*[grp(a)!=grp(b)],
    raises[a,k] = #t: sel(t,a) & !hit(t,k);  drops[a,b] = #t: lone(t,a) & !sel(t,b).
    """
    t, e = bits.shape
    size = e // groups
    hit = group_hits(bits, groups)
    base = hit.sum(axis=0, dtype=np.int64)
    b64 = bits.astype(np.int64)
    per_group = b64.reshape(t, groups, size).sum(axis=2)
    lone = bits & np.repeat(per_group == 1, size, axis=1)
    raises = b64.T @ (~hit).astype(np.int64)              # E x g
    drops = lone.astype(np.int64).T @ (~bits).astype(np.int64)   # E x E
    grp = np.arange(e) // size
    other = grp[:, None] != grp[None, :]
    d = np.zeros((e, e, groups), dtype=np.int64)
    onehot_b = (grp[None, :, None] == np.arange(groups)[None, None, :])   # [1,E,g]
    d += raises[:, None, :] * onehot_b
    onehot_a = (grp[:, None, None] == np.arange(groups)[None, None, :])   # [E,1,g]
    d -= (drops * other)[:, :, None] * onehot_a
    return base[None, None, :] + d + d.transpose(1, 0, 2)


def swap_tensors(bits, fanouts, dim=None):
    """(inter tuple, intra) for levels 1..dim-1 and per GPU (swap.py:121-138)."""
    u = level_group_counts(fanouts)
    upto = len(fanouts) if dim is None else dim
    inter = tuple(swap_tensor(bits, u[level]) for level in range(1, upto))
    return inter, swap_tensor(bits, num_gpus(fanouts))


def swap_tensors_bruteforce(bits, fanouts):
    """Materialise every swap and recount (swap.py:141-177)."""
    t, e = bits.shape
    u = level_group_counts(fanouts)
    g = num_gpus(fanouts)
    depth = len(fanouts)
    inter = [np.zeros((e, e, u[i]), dtype=np.int64) for i in range(1, depth)]
    intra = np.zeros((e, e, g), dtype=np.int64)
    for r in range(e):
        for c in range(r, e):
            sw = bits.copy()
            sw[:, [r, c]] = sw[:, [c, r]]
            per_gpu = dedup_counts(sw, g)
            cur, origin = sw, None
            for level in range(1, depth):
                inter[level - 1][r, c] = inter[level - 1][c, r] = dedup_counts(cur, u[level])
                cur, origin, _ = propagate(cur, u[level], origin)
                assert np.array_equal(dedup_counts(cur, g), per_gpu)
            intra[r, c] = intra[c, r] = per_gpu
    return tuple(inter), intra


# --------------------------------------------------------------------------
# smooth max, cost matrix, selection (swap.py:35-57, 180-259)

def smooth_max_lastaxis(z: np.ndarray, gamma: float) -> np.ndarray:
    """m * (sum((z/m)^gamma))^(1/gamma); 0 for all-zero slices (swap.py:51-57).

    The numpy ops (true_divide, power, add.reduce over the last axis, power,
    multiply) and their order are the rounding specification the GPU kernel
    reproduces; keep them exactly as written.
    """
    m = z.max(axis=-1)
    safe = np.where(m > 0, m, 1.0)
    total = np.power(z / safe[..., None], gamma).sum(axis=-1)
    return np.where(m > 0, safe * np.power(total, 1.0 / gamma), 0.0)


def cost_matrix(inter, intra, fanouts, params, token_bytes, dim, gamma):
    """Q[r,c] = predicted seconds of the dim-D dispatch after swap (r,c)
    (swap.py:180-206)."""
    a_inter, b_inter, a_intra, b_intra = params
    u = level_group_counts(fanouts)
    g = num_gpus(fanouts)
    n = intra.shape[0]
    q = np.zeros((n, n))
    for level in range(1, dim):
        vol = (u[level] // u[level - 1]) * smooth_max_lastaxis(inter[level - 1], gamma)
        q += vol * token_bytes * b_inter[level - 1] + a_inter[level - 1]
    vol = (g // u[dim - 1]) * smooth_max_lastaxis(intra, gamma)
    q += vol * token_bytes * b_intra[dim - 1] + a_intra[dim - 1]
    return q


def select_swap(bits, fanouts, params, token_bytes, gamma=10.0):
    """(pair|None, saving, d*, no_swap_time, Q) (swap.py:226-252)."""
    d_star = optimal_dimension(bits, fanouts, params, token_bytes)[0]
    inter, intra = swap_tensors(bits, fanouts, d_star)
    q = cost_matrix(inter, intra, fanouts, params, token_bytes, d_star, gamma)
    r, c = divmod(int(np.argmin(q)), q.shape[1])
    q_exact = cost_matrix(inter, intra, fanouts, params, token_bytes, d_star, math.inf)
    no_swap = float(q_exact[0, 0])
    if r == c:
        return None, 0.0, d_star, no_swap, q
    saving = no_swap - float(q_exact[r, c])
    if saving < 0:
        return None, 0.0, d_star, no_swap, q
    return (r, c), saving, d_star, no_swap, q


def slot_view(bits: np.ndarray, slot_to_expert) -> np.ndarray:
    """bits[:, slot_to_expert] (routing.py:98-106)."""
    if slot_to_expert is None:
        return bits
    return bits[:, np.asarray(slot_to_expert)]
