"""ctypes binding of the C-ABI in include/bitsnap_b200.h (`_bsnp.so`).

There is deliberately no CPU fallback: if the extension is missing the import
of any codec entry point fails loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "_bsnp.so")

BSNP_OK, BSNP_E_INVALID, BSNP_E_ALIGN, BSNP_E_WORKSPACE, BSNP_E_CUDA = 0, 1, 2, 3, 4
ERR_PADDING, ERR_POPCOUNT, ERR_PAYLOAD_CAP, ERR_LABEL, ERR_NONFINITE = 1, 2, 4, 8, 16

_c = ctypes
_vp, _u64, _sz, _i32 = _c.c_void_p, _c.c_uint64, _c.c_size_t, _c.c_int

# name -> (restype, argtypes); must cover every function in include/*.h
SIGNATURES = {
    "bsnp_abi_version": (_i32, []),
    "bsnp_last_error": (_c.c_char_p, []),
    "bsnp_device_sm_count": (_i32, []),
    "bsnp_host_register": (_i32, [_vp, _sz]),
    "bsnp_host_unregister": (_i32, [_vp]),
    "bsnp_delta_encode_ws_bytes": (_sz, [_u64]),
    "bsnp_delta_decode_ws_bytes": (_sz, [_u64]),
    "bsnp_delta_encode": (_i32, [_vp, _vp, _u64, _vp, _vp, _u64, _vp, _vp, _sz, _vp]),
    "bsnp_delta_decode": (_i32, [_vp, _vp, _vp, _u64, _u64, _vp, _vp, _vp, _sz, _vp]),
    "bsnp_delta_decode_dn": (_i32, [_vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "bsnp_cluster_ws_bytes": (_sz, [_u64, _u64]),
    "bsnp_cluster_fit": (_i32, [_vp, _u64, _u64, _i32, _vp, _vp, _sz, _vp]),
    "bsnp_cluster_quantize": (_i32, [_vp, _u64, _u64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "bsnp_cluster_encode": (_i32, [_vp, _u64, _u64, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "bsnp_cluster_dequantize": (_i32, [_vp, _vp, _u64, _u64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "bsnp_precision_ws_bytes": (_sz, []),
    "bsnp_precision_report": (_i32, [_vp, _vp, _u64, _vp, _vp, _sz, _vp]),
    "bsnp_gather_segments": (_i32, [_vp, _vp, _c.c_uint32, _c.c_uint32, _vp, _vp]),
    "bsnp_copy_sm": (_i32, [_vp, _vp, _u64, _vp]),
    "bsnp_cluster_dequantize_batch": (_i32, [_vp, _vp, _c.c_uint32, _c.c_uint32, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


class CodecLibraryError(RuntimeError):
    pass


def load():
    """Load and type the extension (idempotent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(SO_PATH):
                raise ImportError(
                    f"{SO_PATH} is missing: build it with "
                    "`python -m paper_2511_12376_b200._build` (no CPU fallback)")
            lib = ctypes.CDLL(SO_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype, fn.argtypes = res, args
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc == BSNP_OK:
        return
    lib = load()
    detail = lib.bsnp_last_error().decode(errors="replace") if rc == BSNP_E_CUDA else ""
    names = {BSNP_E_INVALID: "invalid argument", BSNP_E_ALIGN: "misaligned pointer",
             BSNP_E_WORKSPACE: "workspace too small", BSNP_E_CUDA: "CUDA error"}
    raise CodecLibraryError(f"{what}: {names.get(rc, rc)} {detail}".strip())
