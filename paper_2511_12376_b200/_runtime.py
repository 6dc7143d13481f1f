"""Device plumbing around the C-ABI: workspaces, status blocks, staging.

PyTorch is used only for device memory, pinned host memory and streams; all
codec arithmetic runs in `_bsnp.so`.
"""

from __future__ import annotations

import os
import threading

import numpy as np
import torch

from . import _lib

_tls = threading.local()


def device_of(t: torch.Tensor | None = None) -> torch.device:
    if t is not None and t.is_cuda:
        return t.device
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_12376_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _cache() -> dict:
    c = getattr(_tls, "cache", None)
    if c is None:
        c = _tls.cache = {}
    return c


def workspace(device: torch.device, nbytes: int, slot: str = "ws") -> torch.Tensor:
    """Growable per-(thread, device, stream, slot) scratch buffer.

    Work on one stream is ordered, so reuse across calls is safe; distinct
    streams get distinct buffers.
    """
    key = (slot, device.index, stream_ptr(device))
    c = _cache()
    buf = c.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty((max(int(nbytes * 1.25), 256) + 255) // 256 * 256, dtype=torch.uint8,
                          device=device)
        c[key] = buf
    keep = getattr(_tls, "keep", None)
    if keep is not None:
        keep.append(buf)
    return buf


class keep_workspaces:
    """Collect every workspace handed out inside the block (e.g. while a CUDA
    graph is captured): the graph records their addresses, so its owner must
    keep them alive for as long as it may replay — the per-thread cache may
    swap in a bigger buffer and free the captured one."""

    def __enter__(self):
        self.prev = getattr(_tls, "keep", None)
        self.bufs = []
        _tls.keep = self.bufs
        return self.bufs

    def __exit__(self, *exc):
        _tls.keep = self.prev
        if self.prev is not None:
            self.prev.extend(self.bufs)
        return False


_NVTX = os.environ.get("BSNP_NVTX", "0") != "0"


class nvtx:
    """NVTX range around a record's / a group's / a link's launches
    (per-tensor ranges in nsys / ncu timelines).  Off unless
    BSNP_NVTX=1: a range costs ~1 us of host time, and a GPT-2-sized save
    launches ~450 records."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        if _NVTX:
            torch.cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *exc):
        if _NVTX:
            torch.cuda.nvtx.range_pop()
        return False


def new_status(device: torch.device, count: int = 1) -> torch.Tensor:
    """`count` bsnp_status blocks (16 B each) as an int64 [count, 2] tensor."""
    return torch.empty((count, 2), dtype=torch.int64, device=device)


def read_status(st: torch.Tensor):
    """-> list of (count, err_flags) after a device sync on the status copy."""
    h = st.cpu().numpy()
    return [(int(r[0]) & 0xFFFFFFFFFFFFFFFF, int(r[1]) & 0xFFFFFFFF) for r in h]


def pinned(nbytes: int, slot: str = "pin") -> torch.Tensor:
    key = ("pin", slot)
    c = _cache()
    buf = c.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 4096), dtype=torch.uint8, pin_memory=True)
        c[key] = buf
    return buf[:nbytes]


def h2d_bytes(data, device: torch.device, dtype: torch.dtype = torch.uint8) -> torch.Tensor:
    """Host bytes -> new device tensor (via pinned staging)."""
    raw = np.frombuffer(data, dtype=np.uint8)
    out = torch.empty(raw.size, dtype=torch.uint8, device=device)
    if raw.size:
        stage = pinned(raw.size, "h2d")
        stage.numpy()[:] = raw
        out.copy_(stage, non_blocking=True)
        torch.cuda.current_stream(device).synchronize()  # staging buffer is reused
    return out.view(dtype)


def d2h_bytes(t: torch.Tensor) -> bytes:
    """Device tensor -> bytes (via pinned staging)."""
    flat = t.reshape(-1).view(torch.uint8)
    if flat.numel() == 0:
        return b""
    stage = pinned(flat.numel(), "d2h")
    stage.copy_(flat, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return stage.numpy().tobytes()


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def lib():
    return _lib.load()
