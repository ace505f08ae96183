"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/hiermoe.h declares, and the Python binding covers them."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "hiermoe.h"
LIB = ROOT / "paper_2508_09591_b200" / "libhiermoe.so"


def declared() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hm_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        from paper_2508_09591_b200 import _build
        _build.build()
    return ctypes.CDLL(str(LIB))


def test_header_declares_entry_points():
    names = declared()
    assert "hm_dispatch" in names and "hm_swap_cost" in names and len(names) >= 25


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_2508_09591_b200 import _lib
    assert sorted(_lib.exported_symbols()) == declared()


def test_version_and_error_string_without_gpu(lib):
    lib.hm_version.restype = ctypes.c_int
    assert lib.hm_version() >= 10000
    lib.hm_last_error.restype = ctypes.c_char_p
    # invalid argument path runs on the host and needs no device
    lib.hm_level_counts.restype = ctypes.c_int
    st = lib.hm_level_counts(None, ctypes.c_int64(0), ctypes.c_int32(8),
                             (ctypes.c_int32 * 1)(3), ctypes.c_int32(1), None, None, None,
                             ctypes.c_int32(-1), None)
    assert st < 0
    assert b"does not divide" in lib.hm_last_error()


def test_product_fails_loudly_without_cuda(monkeypatch):
    import torch
    from paper_2508_09591_b200 import _lib
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load()


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2508_09591_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f
