"""Lossless bitmask delta codec for 16-bit model states — B200 path.

Drop-in for /root/reference/pkg/src/bitsnap/bitmask.py: the same names,
argument meaning, error types/messages and byte-identical BSDL records.  The
arithmetic (change test, mask packing, stream compaction, scatter decode)
runs in the sm_100a kernels of `_bsnp.so` (csrc/bitmask.cu); this module only
validates arguments, moves bytes and builds headers.

Two layers:
  * device API  — `encode_delta_device` / `decode_delta_device` on CUDA
    tensors (fp16 / bf16 / int16 / uint16 storage), no host round trip;
  * compat API  — `encode_delta` / `decode_delta` / `chain_encode` on the
    reference's `TensorBlob` (host bytes), as the reference callers use them.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import torch

from . import _lib
from . import _runtime as rt
from .tensors import ByteCursor, ElementType, TensorBlob, pack_shape_header

DELTA_MAGIC = b"BSDL"
DELTA_VERSION = 1
# magic(4) + version(2) + n(8) + n_c(8) + name_len(2) + rank(1) + extent(8)
DELTA_FIXED_OVERHEAD = 33


class DeltaError(ValueError):
    """bitmask.py:29."""


@dataclass(frozen=True)
class DeltaRecord:
    """Packed change mask + changed 16-bit values of one tensor (bitmask.py:33-64)."""

    tensor_name: str
    shape: tuple
    total_elements: int
    changed_count: int
    packed_mask: bytes
    payload: bytes

    def __post_init__(self):
        object.__setattr__(self, "shape", tuple(int(s) for s in self.shape))
        n, n_c = self.total_elements, self.changed_count
        if len(self.packed_mask) != (n + 7) // 8:
            raise DeltaError(f"mask is {len(self.packed_mask)} bytes, expected {(n + 7) // 8}")
        if len(self.payload) != 2 * n_c:
            raise DeltaError(f"payload is {len(self.payload)} bytes, expected {2 * n_c}")

    @property
    def serialized_size(self) -> int:
        return (DELTA_FIXED_OVERHEAD + len(self.tensor_name.encode("utf-8"))
                + 8 * (len(self.shape) - 1) + len(self.packed_mask) + len(self.payload))


@dataclass(frozen=True)
class DeltaCheckpoint:
    """One iteration's model-state change set against its predecessor."""

    iteration: int
    base_iteration: int
    records: tuple

    def __post_init__(self):
        object.__setattr__(self, "records", tuple(self.records))


# ---------------------------------------------------------------------------
# device API
# ---------------------------------------------------------------------------

@dataclass
class DeviceDelta:
    """Encoder output resident in HBM: mask u8[ceil(n/8)], payload int16[n_c]."""

    mask: torch.Tensor
    payload: torch.Tensor
    n: int
    n_c: int


def _as_i16(t: torch.Tensor) -> torch.Tensor:
    if t.element_size() != 2:
        raise DeltaError("delta encoding requires F16 tensors")
    t = t.reshape(-1)
    if not t.is_contiguous():
        t = t.contiguous()
    return t.view(torch.int16)


def encode_delta_async(base: torch.Tensor, target: torch.Tensor, mask: torch.Tensor,
                       payload: torch.Tensor, status: torch.Tensor) -> None:
    """Enqueue one encode on the current stream; n_c lands in status[0]."""
    b, c = _as_i16(base), _as_i16(target)
    n = b.numel()
    dev = b.device
    ws_n = rt.lib().bsnp_delta_encode_ws_bytes(n)
    ws = rt.workspace(dev, ws_n, "enc")
    _lib.check(rt.lib().bsnp_delta_encode(
        b.data_ptr(), c.data_ptr(), n, mask.data_ptr(), payload.data_ptr(),
        payload.numel(), status.data_ptr(), ws.data_ptr(), ws.numel(),
        rt.stream_ptr(dev)), "bsnp_delta_encode")


def encode_delta_device(base: torch.Tensor, target: torch.Tensor) -> DeviceDelta:
    """bitmask.py:94-111 on device tensors.  Reads n_c back (one small sync)."""
    if base.shape != target.shape:
        raise DeltaError(f"shape mismatch: {tuple(base.shape)} vs {tuple(target.shape)}")
    b, c = _as_i16(base), _as_i16(target)
    n = b.numel()
    dev = rt.device_of(b)
    mask = torch.empty((n + 7) // 8, dtype=torch.uint8, device=dev)
    scratch = rt.workspace(dev, 2 * max(n, 1), "payload").view(torch.int16)
    st = rt.new_status(dev)
    encode_delta_async(b, c, mask, scratch, st)
    (n_c, flags), = rt.read_status(st)
    if flags & _lib.ERR_PAYLOAD_CAP:
        raise DeltaError("internal: payload capacity exceeded")
    return DeviceDelta(mask=mask, payload=scratch[:n_c].clone(), n=n, n_c=n_c)


def decode_delta_async(base: torch.Tensor, mask: torch.Tensor, payload: torch.Tensor,
                       n_c: int, out: torch.Tensor, status: torch.Tensor) -> None:
    """Enqueue one decode on the current stream (out may be base: in-place)."""
    b = _as_i16(base)
    o = out.reshape(-1).view(torch.int16)
    n = b.numel()
    dev = b.device
    ws_n = rt.lib().bsnp_delta_decode_ws_bytes(n)
    ws = rt.workspace(dev, ws_n, "dec")
    _lib.check(rt.lib().bsnp_delta_decode(
        b.data_ptr(), mask.data_ptr(), payload.data_ptr() if payload.numel() else None,
        n, n_c, o.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(),
        rt.stream_ptr(dev)), "bsnp_delta_decode")


def decode_delta_async_dn(base: torch.Tensor, mask: torch.Tensor, payload: torch.Tensor,
                          n_c_status: torch.Tensor, out: torch.Tensor,
                          status: torch.Tensor) -> None:
    """decode_delta_async out of place with n_c read on the device from
    `n_c_status` (the encode's status block: its count word), so an encode
    and the decode of its record queue back to back with no host round
    trip (bsnp_delta_decode_dn).  payload: the encode's payload buffer."""
    b = _as_i16(base)
    o = out.reshape(-1).view(torch.int16)
    n = b.numel()
    dev = b.device
    ws = rt.workspace(dev, rt.lib().bsnp_delta_decode_ws_bytes(n), "dec")
    _lib.check(rt.lib().bsnp_delta_decode_dn(
        b.data_ptr(), mask.data_ptr(), payload.data_ptr() if payload.numel() else None,
        n, n_c_status.data_ptr(), o.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(),
        rt.stream_ptr(dev)), "bsnp_delta_decode_dn")


def _raise_decode_flags(flags: int, popcount: int, n_c: int) -> None:
    if flags & _lib.ERR_PADDING:
        raise DeltaError("nonzero padding bits in mask")
    if flags & _lib.ERR_POPCOUNT:
        raise DeltaError(f"mask popcount {popcount} != recorded changed_count {n_c}")


def decode_delta_device(base: torch.Tensor, mask: torch.Tensor, payload: torch.Tensor,
                        n_c: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """bitmask.py:114-140 on device tensors.  `out=base` applies in place
    (chain replay); base is untouched if the mask fails validation."""
    n = base.numel()
    if mask.numel() != (n + 7) // 8:
        raise DeltaError(f"mask is {mask.numel()} bytes, expected {(n + 7) // 8}")
    if payload.numel() != n_c:
        raise DeltaError(f"payload is {2 * payload.numel()} bytes, expected {2 * n_c}")
    if out is None:
        out = torch.empty_like(base)
    st = rt.new_status(rt.device_of(base))
    decode_delta_async(base, mask, payload.reshape(-1).view(torch.int16), n_c, out, st)
    (pc, flags), = rt.read_status(st)
    _raise_decode_flags(flags, pc, n_c)
    return out


# ---------------------------------------------------------------------------
# compat API (reference signatures over host TensorBlob bytes)
# ---------------------------------------------------------------------------

def _check_pair(base: TensorBlob, target: TensorBlob) -> None:
    """bitmask.py:83-91 (same checks, same order, same messages)."""
    if base.name != target.name:
        raise DeltaError(f"name mismatch: {base.name!r} vs {target.name!r}")
    if base.dtype is not ElementType.F16 or target.dtype is not ElementType.F16:
        raise DeltaError("delta encoding requires F16 tensors")
    if base.shape != target.shape:
        raise DeltaError(f"shape mismatch for {base.name!r}: {base.shape} vs {target.shape}")


def encode_delta(base: TensorBlob, target: TensorBlob) -> DeltaRecord:
    """Bit i of the mask is set iff element i of target differs from base."""
    _check_pair(base, target)
    dev = rt.device_of()
    b = rt.h2d_bytes(base.data, dev, torch.int16)
    c = rt.h2d_bytes(target.data, dev, torch.int16)
    d = encode_delta_device(b, c)
    return DeltaRecord(tensor_name=target.name, shape=target.shape, total_elements=d.n,
                       changed_count=d.n_c, packed_mask=rt.d2h_bytes(d.mask),
                       payload=rt.d2h_bytes(d.payload))


def decode_delta(base: TensorBlob, rec: DeltaRecord) -> TensorBlob:
    """Inverse of encode_delta; reconstruction is bitwise exact."""
    if base.name != rec.tensor_name:
        raise DeltaError(f"name mismatch: {base.name!r} vs {rec.tensor_name!r}")
    if base.shape != rec.shape:
        raise DeltaError(f"shape mismatch for {base.name!r}: {base.shape} vs {rec.shape}")
    if base.num_elements != rec.total_elements:
        raise DeltaError("element count mismatch")
    dev = rt.device_of()
    b = rt.h2d_bytes(base.data, dev, torch.int16)
    m = rt.h2d_bytes(rec.packed_mask, dev)
    p = rt.h2d_bytes(rec.payload, dev, torch.int16)
    out = decode_delta_device(b, m, p, rec.changed_count)
    return TensorBlob(name=base.name, dtype=ElementType.F16, shape=base.shape,
                      data=rt.d2h_bytes(out))


def chain_encode(base, targets) -> list:
    """bitmask.py:147-178: delta k is taken against checkpoint k-1.

    The predecessor's model states stay resident in HBM between steps, so each
    tensor crosses PCIe once per checkpoint.
    """
    out = []
    prev = base
    dev = rt.device_of()
    resident = {t.name: rt.h2d_bytes(t.data, dev, torch.int16) for t in base.model_states}
    for tgt in targets:
        if tgt.iteration <= prev.iteration:
            raise DeltaError(f"iterations must be strictly increasing: "
                             f"{prev.iteration} then {tgt.iteration}")
        if {t.name for t in tgt.model_states} != set(resident):
            raise DeltaError(f"tensor structure mismatch at iteration {tgt.iteration}")
        prev_map = {t.name: t for t in prev.model_states}
        records, nxt = [], {}
        for t in tgt.model_states:
            _check_pair(prev_map[t.name], t)
            cur = rt.h2d_bytes(t.data, dev, torch.int16)
            d = encode_delta_device(resident[t.name], cur)
            records.append(DeltaRecord(tensor_name=t.name, shape=t.shape,
                                       total_elements=d.n, changed_count=d.n_c,
                                       packed_mask=rt.d2h_bytes(d.mask),
                                       payload=rt.d2h_bytes(d.payload)))
            nxt[t.name] = cur
        out.append(DeltaCheckpoint(iteration=tgt.iteration, base_iteration=prev.iteration,
                                   records=tuple(records)))
        resident, prev = nxt, tgt
    return out


# ---------------------------------------------------------------------------
# size laws and BSDL serialization (bitmask.py:181-238)
# ---------------------------------------------------------------------------

def delta_size_bytes(n: int, n_c: int) -> int:
    """Serialized size of a delta for an empty name and rank 1."""
    if not 0 <= n_c <= n:
        raise DeltaError(f"need 0 <= n_c <= n, got n={n}, n_c={n_c}")
    return (n + 7) // 8 + 2 * n_c + DELTA_FIXED_OVERHEAD


def naive_delta_size_bytes(n: int, n_c: int) -> int:
    """Unpacked one-byte-per-element mask variant, for comparison only."""
    if not 0 <= n_c <= n:
        raise DeltaError(f"need 0 <= n_c <= n, got n={n}, n_c={n_c}")
    return n + 2 * n_c + DELTA_FIXED_OVERHEAD


def delta_header(name: str, shape, n: int, n_c: int) -> bytes:
    return pack_shape_header(DELTA_MAGIC, struct.pack("<HQQ", DELTA_VERSION, n, n_c),
                             name, shape)


def serialize_delta(rec: DeltaRecord) -> bytes:
    return (delta_header(rec.tensor_name, rec.shape, rec.total_elements, rec.changed_count)
            + rec.packed_mask + rec.payload)


def deserialize_delta(b: bytes) -> DeltaRecord:
    cur = ByteCursor(b)
    cur.magic(DELTA_MAGIC)
    (ver,) = cur.unpack("<H")
    if ver != DELTA_VERSION:
        raise DeltaError(f"unsupported delta version {ver}")
    n, n_c = cur.unpack("<QQ")
    name, shape = cur.name_and_shape()
    mask = bytes(cur.take((n + 7) // 8))
    payload = bytes(cur.take(2 * n_c))
    return DeltaRecord(tensor_name=name, shape=shape, total_elements=n, changed_count=n_c,
                       packed_mask=mask, payload=payload)
