"""CPU checks of the C-ABI library: it loads and exports every symbol that
include/*.h declares, and the Python binding types all of them."""

import glob
import os
import re

import pytest

from conftest import ROOT


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(bsnp_[a-z0-9_]+)\s*\(", src))
    return names


def test_header_declares_functions():
    names = _declared()
    assert {"bsnp_delta_encode", "bsnp_delta_decode", "bsnp_abi_version"} <= names


def test_library_exports_every_declared_symbol():
    from paper_2511_12376_b200 import _build, _lib
    _build.build()
    lib = _lib.load()
    for name in sorted(_declared()):
        assert hasattr(lib, name), name
    assert set(_lib.SIGNATURES) == _declared()
    assert lib.bsnp_abi_version() == 1


def test_ws_sizes_without_gpu():
    from paper_2511_12376_b200 import _lib
    lib = _lib.load()
    for n in (0, 1, 8192, 8193, 1 << 30):
        nt = -(-n // 8192)
        # header + tile status (256-aligned) + 16 KiB payload staging per tile
        assert lib.bsnp_delta_encode_ws_bytes(n) == -(-(256 + 8 * nt) // 256) * 256 + 16384 * nt
        assert lib.bsnp_delta_decode_ws_bytes(n) == 256 + 8 * -(-nt // 32) + 8 * (nt + 1)


def test_argument_errors_without_gpu():
    """Host-side argument validation runs before any CUDA call."""
    from paper_2511_12376_b200 import _lib
    lib = _lib.load()
    assert lib.bsnp_delta_encode(None, None, 10, None, None, 0, None, None, 0, None) \
        == _lib.BSNP_E_INVALID
    assert lib.bsnp_delta_encode(2, 4, 10, 8, 1, 10, 16, 32, 10**6, None) == _lib.BSNP_E_ALIGN
    assert lib.bsnp_delta_decode(2, 4, 8, 10, 11, 8, 16, 32, 10**6, None) == _lib.BSNP_E_INVALID


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2511_12376_b200")
    for py in glob.glob(os.path.join(pkg, "**", "*.py"), recursive=True):
        src = open(py).read()
        assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), py
        assert "bitsnap_oracle" not in src, py
