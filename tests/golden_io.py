"""Loader for the committed golden vectors (tests/golden/, made by make_golden.py)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=1)
def _arrays():
    with np.load(GOLDEN / "cases.npz") as z:
        return {k: z[k] for k in z.files}


@lru_cache(maxsize=1)
def cases() -> list[dict]:
    return json.loads((GOLDEN / "cases.json").read_text())


@lru_cache(maxsize=1)
def sims() -> dict:
    return json.loads((GOLDEN / "sims.json").read_text())


def arr(case: dict, name: str):
    return _arrays().get(f"{case['key']}_{name}")


def bits(case: dict) -> np.ndarray:
    packed = arr(case, "bits")
    return np.unpackbits(packed, axis=1, count=case["experts"]).astype(bool)


def perm(case: dict):
    return arr(case, "perm") if case["has_perm"] else None


def unpack(case: dict, name: str, width: int) -> np.ndarray:
    return np.unpackbits(arr(case, name), axis=1, count=width).astype(bool)


def params(case: dict):
    return tuple(tuple(x) for x in case["params"])


def token_bytes(case: dict) -> int:
    return case["embed_dim"] * case["bytes_per_elem"]


def level_groups(case: dict) -> tuple[int, ...]:
    u = [1]
    for f in case["fanouts"][:-1]:
        u.append(u[-1] * f)
    return tuple(u)


def gpus(case: dict) -> int:
    return int(np.prod(case["fanouts"]))
