"""Per-step choice of the dispatch transport by the reference's time model.

HierMoE picks the AlltoAll dimension of every step from its alpha/beta model
(``pick_dimension`` / ``optimal_dimension``, traffic.py:188-221; Algorithm 1
at PAPER.md:364-366) and compares against the non-deduplicated AlltoAll
(``time_without_dedup``, the engine's "std" strategy, engine.py:159-163).
The layer's transports are exactly those variants on the runtime hierarchy
``[P GPUs, L ranks per GPU]``:

* "none"   -- one row per selection (``time_without_dedup(1)``);
* "remote" -- d = 1: one row per (token, remote EP rank) (``time_with_dedup(1)``);
* "gpu"    -- d = 2: one row per (token, remote GPU), re-expanded into the
  GPU's ranks on arrival (inter phase over the U[1] = P GPUs, intra phase
  inside the GPU) (``time_with_dedup(2)``).

With one rank per GPU (L = 1) or one GPU (P = 1) the hierarchy is flat
([G]) and "remote" and "gpu" coincide.  The alpha/beta of each phase come
from ``tools/calibrate.py --runtime`` on the box (params JSON in the
reference schema, topology.py:156-193), shipped in ``params/``.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

from .topology import LevelParams, Topology, build_topology, load_params
from .traffic import _Model, pick_dimension

PARAMS_DIR = Path(__file__).resolve().parent / "params"
_DIM_MODE = {1: "remote", 2: "gpu"}


def runtime_topology(ranks: int, gpus: int, experts: int, hidden: int,
                     bytes_per_elem: int = 2) -> Topology:
    """The hierarchy the layer runs on: [P, L] with L = ranks / P EP ranks per
    GPU, or flat [G] when P = 1 or L = 1."""
    if ranks % gpus:
        raise ValueError(f"ranks ({ranks}) must be a multiple of gpus ({gpus})")
    local = ranks // gpus
    fan = [gpus, local] if gpus > 1 and local > 1 else [ranks]
    return build_topology(fan, experts, hidden, bytes_per_elem)


def default_params(gpus: int, levels: int) -> LevelParams:
    """B200 fits for a ``gpus``-GPU run (params/b200_runtime_n{P}.json); the
    nearest calibrated GPU count when this one was not measured.  A flat
    topology uses only the 'std' entry."""
    files = sorted(PARAMS_DIR.glob("b200_runtime_n*.json"),
                   key=lambda p: abs(int(p.stem.rsplit("n", 1)[1]) - gpus))
    if not files:
        raise FileNotFoundError(f"no runtime alpha/beta fits under {PARAMS_DIR}")
    p = load_params(files[0])
    if levels == 1:
        return LevelParams((), (), (p.alpha_std,), (p.beta_std,))
    if p.num_levels != levels:
        raise ValueError(f"{files[0].name} covers {p.num_levels} levels, need {levels}")
    return p


@dataclass(frozen=True)
class TransportChoice:
    mode: str                       # "none" | "remote" | "gpu"
    d_star: int                     # pick_dimension over the dedup times
    times: tuple                    # time_with_dedup(d), d = 1..D (seconds)
    time_without_dedup: float       # time_without_dedup(1) (seconds)


def choose_transport(mask, topology: Topology, params: LevelParams, placement=None,
                     reduce=None, allow_deep: bool = True) -> TransportChoice:
    """The reference's rule on this step's mask: d* = pick_dimension(dedup
    times); the non-deduplicated AlltoAll wins only when strictly faster than
    the d* variant.  ``reduce`` all-reduces the counts of a token-sharded mask
    (every rank then takes the same decision).  ``allow_deep=False`` limits
    the choice to d = 1 (the training layer's backward needs a per-rank
    transport)."""
    m = _Model(mask, topology, params, placement, True, reduce).fetch()
    times = m.times
    m._args = (topology, params, False)        # same counts, raw volumes
    t_std = m.finish().fetch().times[0]
    d_star = pick_dimension(times) if allow_deep else 1
    if t_std < times[d_star - 1]:
        mode = "none"
    else:
        mode = _DIM_MODE[d_star] if topology.num_levels > 1 else "gpu"
    return TransportChoice(mode, d_star, tuple(times), t_std)
