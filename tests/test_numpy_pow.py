"""CPU checks of the product's floating-point restatement (csrc/numpy_pow.cuh,
csrc/ddmath.cuh) built for the host: numpy's pow and smooth-max rounding.

The GPU cost kernel compiles the same header; these tests pin the algorithm
without a GPU.  np.power is the oracle here (numpy *is* the reference's
arithmetic dependency, pyproject.toml:10-12).  They apply only where numpy
takes its AVX512_SKX SVML path, as on the hosts the fixtures were made on.
"""

import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

import golden_io as G
from oracle import hiera as O

NATIVE = Path(__file__).resolve().parent / "native"


def _svml_numpy() -> bool:
    try:
        from numpy._core._multiarray_umath import __cpu_features__ as f
        return bool(f.get("AVX512_SKX"))
    except Exception:
        return False


pytestmark = pytest.mark.skipif(not _svml_numpy(),
                                reason="numpy on this host does not use SVML pow")


@pytest.fixture(scope="module")
def host():
    so = NATIVE / "ddhost.so"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-frounding-math", "-fPIC", "-shared",
                    "-o", str(so), str(NATIVE / "ddhost.cpp")], check=True)
    lib = ctypes.CDLL(str(so))
    lib.hm_host_pow_cr.restype = ctypes.c_double
    lib.hm_host_pow_cr.argtypes = [ctypes.c_double, ctypes.c_double]
    return lib


def _np_pow(lib, x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(np.broadcast_to(y, x.shape), dtype=np.float64)
    out = np.empty_like(x)
    lib.hm_host_np_pow(x.ctypes.data_as(ctypes.c_void_p), y.ctypes.data_as(ctypes.c_void_p),
                       out.ctypes.data_as(ctypes.c_void_p), ctypes.c_long(x.size))
    return out


def test_np_pow_bitwise_on_smooth_max_domain(host):
    rng = np.random.default_rng(11)
    z = rng.integers(0, 1 << 20, 200000)
    m = z + rng.integers(0, 1 << 20, 200000) + 1
    for gamma in (10.0, 3.0, 17.5, 1e4, 1.5):
        r = z / m
        assert np.array_equal(_np_pow(host, r, gamma), np.power(r, gamma)), gamma
        tot = rng.uniform(1.0, 64.0, 200000)
        assert np.array_equal(_np_pow(host, tot, 1.0 / gamma), np.power(tot, 1.0 / gamma))


def test_np_pow_bitwise_wide_range(host):
    rng = np.random.default_rng(12)
    x = np.exp(rng.uniform(-60, 60, 200000))
    y = rng.uniform(0.02, 30, 200000)
    with np.errstate(over="ignore", under="ignore"):
        ref = np.power(x, y)
    got = _np_pow(host, x, y)
    assert np.array_equal(got, ref)
    assert np.array_equal(_np_pow(host, np.array([0.0, 1.0, 1e-310]), 10.0),
                          np.power(np.array([0.0, 1.0, 1e-310]), 10.0))


def test_pow_cr_is_correctly_rounded(host):
    from fractions import Fraction
    rng = np.random.default_rng(13)
    for _ in range(3000):
        m = int(rng.integers(1, 50000))
        z = int(rng.integers(0, m + 1))
        r = z / m
        assert host.hm_host_pow_cr(r, 10.0) == float(Fraction(r) ** 10)


def test_smooth_max_rows_match_numpy_on_golden_cases(host):
    f = host.hm_host_smooth_max_rows
    f.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_int, ctypes.c_double, ctypes.c_void_p]

    def smax(z, gamma):
        z = np.ascontiguousarray(z, dtype=np.int64)
        out = np.empty(z.shape[:-1])
        f(z.ctypes.data, out.size, z.shape[-1], gamma, out.ctypes.data)
        return out

    checked = 0
    for case in G.cases():
        if G.arr(case, "zintra") is None:
            continue
        sv = O.slot_view(G.bits(case), G.perm(case))
        inter, intra = O.swap_tensors(sv, tuple(case["fanouts"]))
        for z in list(inter) + [intra]:
            assert np.array_equal(smax(z, case["gamma"]),
                                  O.smooth_max_lastaxis(z, case["gamma"]))
        checked += 1
    assert checked > 100


def test_pairwise_sum_matches_numpy(host):
    host.hm_host_pairwise.restype = ctypes.c_double
    host.hm_host_pairwise.argtypes = [ctypes.c_void_p, ctypes.c_int]
    rng = np.random.default_rng(14)
    for n in list(range(1, 40)) + [64, 100, 127, 128, 129, 200, 256]:
        a = rng.random((50, n)) * rng.choice([1e-3, 1.0, 1e3], size=(50, n))
        ref = a.sum(axis=-1)
        for i in range(50):
            row = np.ascontiguousarray(a[i])
            assert host.hm_host_pairwise(row.ctypes.data, n) == ref[i], n
