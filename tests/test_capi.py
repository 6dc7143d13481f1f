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
        # header + tile status (256-aligned) + 16 KiB staging slots for tiles
        # too dense for the shared-memory arena: one per tile, or a ring of 16
        # per resident CTA, whichever is fewer (the CTA count needs a GPU; one
        # CTA is assumed without one) + one granule of read-past slack
        head = -(-(256 + 8 * nt) // 256) * 256
        slots = min(nt, 16) if nt > 16 else nt
        assert lib.bsnp_delta_encode_ws_bytes(n) == head + 16384 * slots + 256
        nch = -(-nt // 32)
        assert lib.bsnp_delta_decode_ws_bytes(n) == (256 + 8 * (nch + 1) + 4 * (nt + 1) + 4 * nch
                                                     + 8 + 8 * (nt + 1))


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


def test_batch_layouts_and_errors_without_gpu():
    """The numpy mirrors of bsnp_segment / bsnp_dequant_item have the C
    sizes; the batched dequantize validates before any CUDA call."""
    from paper_2511_12376_b200 import _lib
    from paper_2511_12376_b200 import store as S
    assert S._SEG.itemsize == 24 and S._DQI.itemsize == 40
    lib = _lib.load()
    assert lib.bsnp_cluster_dequantize_batch(None, None, 0, 0, None, None) == _lib.BSNP_OK
    assert lib.bsnp_cluster_dequantize_batch(None, None, 1, 1, None, None) \
        == _lib.BSNP_E_INVALID
    assert lib.bsnp_copy_sm(None, None, 0, None) == _lib.BSNP_OK
    assert lib.bsnp_copy_sm(None, None, 5, None) == _lib.BSNP_E_INVALID


def test_quant_header_from_device_table_bytes():
    from paper_2511_12376_b200 import quantizer as Q
    for m in (2, 5, 16):
        t = Q.ClusterTable(m=m, mean=0.1, std=2.5, boundaries=tuple(range(1, m)),
                           scales=tuple(0.5 * i for i in range(m)),
                           offsets=tuple(-0.25 * i for i in range(m)))
        raw = t.to_device_bytes()
        assert Q.quant_header_raw("layer.0.w", (3, 7), raw) == Q.quant_header("layer.0.w", (3, 7), t)
