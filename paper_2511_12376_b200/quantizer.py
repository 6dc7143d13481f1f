"""Lossy 8-bit cluster quantization of F32 optimizer states — B200 path.

Drop-in for /root/reference/pkg/src/bitsnap/quantizer.py: the same names,
argument meaning, error types/messages and byte-identical BSQT records.  The
arithmetic — float64 mean/std with numpy's pairwise-summation tree, normal-
quantile boundaries, per-cluster min/max, labels, codes, reconstruction —
runs in the sm_100a kernels of `_bsnp.so` (csrc/quant.cu).

Two layers:
  * device API  — `cluster_fit_device` / `cluster_quantize_device` /
    `cluster_encode_device` / `cluster_dequantize_device` on CUDA float32
    tensors, per tensor (block=0, the reference's behaviour) or per block of
    `block` elements (one table per block, BASELINE configs[2]);
  * compat API  — `build_clusters` / `quantize` / `dequantize` on the
    reference's `TensorBlob` (host bytes).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import _runtime as rt
from .tensors import ByteCursor, ElementType, TensorBlob, pack_shape_header

QUANT_MAGIC = b"BSQT"
QUANT_VERSION = 1
MIN_CLUSTERS = 2
MAX_CLUSTERS = 16
# Denominator floor of the mean relative error (quantizer.py:31-33).
MRE_EPSILON = 1e-12
TABLE_BYTES = 256  # sizeof(bsnp_cluster_table)
_TABLE_FMT = "<2f15f16f16f2I"


class QuantizerError(ValueError):
    """quantizer.py:36."""


def qmap(codes) -> np.ndarray:
    """Map uint8 codes to the normalized domain [0, 1] (quantizer.py:40-42)."""
    return np.asarray(codes, dtype=np.float64) / 255.0


@dataclass(frozen=True)
class ClusterTable:
    """Per-unit clustering parameters (quantizer.py:45-65)."""

    m: int
    mean: float
    std: float
    boundaries: tuple
    scales: tuple
    offsets: tuple

    def __post_init__(self):
        if not MIN_CLUSTERS <= self.m <= MAX_CLUSTERS:
            raise QuantizerError(f"cluster count {self.m} outside [2, 16]")
        if len(self.boundaries) != self.m - 1:
            raise QuantizerError("need m-1 boundaries")
        if len(self.scales) != self.m or len(self.offsets) != self.m:
            raise QuantizerError("need m scales and m offsets")
        b = self.boundaries
        if any(b[i] > b[i + 1] for i in range(len(b) - 1)):
            raise QuantizerError("boundaries must be ascending")

    # device struct (include/bitsnap_b200.h: bsnp_cluster_table)
    def to_device_bytes(self) -> bytes:
        pad = lambda v, k: list(v) + [0.0] * (k - len(v))
        head = struct.pack(_TABLE_FMT, self.mean, self.std, *pad(self.boundaries, 15),
                           *pad(self.scales, 16), *pad(self.offsets, 16), self.m, 0)
        return head + b"\0" * (TABLE_BYTES - len(head))

    @classmethod
    def from_device_bytes(cls, raw: bytes) -> "ClusterTable":
        v = struct.unpack_from(_TABLE_FMT, raw)
        m = v[49]
        return cls(m=m, mean=v[0], std=v[1], boundaries=tuple(v[2:2 + m - 1]),
                   scales=tuple(v[17:17 + m]), offsets=tuple(v[33:33 + m]))


@dataclass(frozen=True)
class QuantizedTensor:
    """Cluster table, packed 4-bit labels and one u8 code per element."""

    name: str
    shape: tuple
    table: ClusterTable
    packed_labels: bytes
    codes: bytes

    def __post_init__(self):
        object.__setattr__(self, "shape", tuple(int(s) for s in self.shape))
        n = self.num_elements
        if len(self.packed_labels) != (n + 1) // 2:
            raise QuantizerError("packed label bytes != ceil(n/2)")
        if len(self.codes) != n:
            raise QuantizerError("need one code byte per element")

    @property
    def num_elements(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n


# ---------------------------------------------------------------------------
# device API
# ---------------------------------------------------------------------------

def _check_m(m: int) -> None:
    if not MIN_CLUSTERS <= m <= MAX_CLUSTERS:
        raise QuantizerError(f"cluster count {m} outside [2, 16]")


def _flat_f32(x: torch.Tensor) -> torch.Tensor:
    if x.dtype != torch.float32:
        raise QuantizerError("cluster quantization requires F32 tensors")
    x = x.reshape(-1)
    return x if x.is_contiguous() else x.contiguous()


def num_units(n: int, block: int) -> int:
    if block and block % 8:
        raise QuantizerError(f"block {block} must be a multiple of 8")
    return 1 if (not block or block >= n) else -(-n // block)


def unit_label_bytes(n: int, block: int) -> int:
    """Bytes of the concatenated per-unit packed label streams."""
    u = num_units(n, block)
    if u == 1:
        return (n + 1) // 2
    last = n - (u - 1) * block
    return (u - 1) * (block // 2) + (last + 1) // 2


def _ws(dev, n, block):
    return rt.workspace(dev, rt.lib().bsnp_cluster_ws_bytes(n, block), "quant")


def cluster_fit_async(x: torch.Tensor, m: int, block: int, tables: torch.Tensor) -> None:
    x = _flat_f32(x)
    ws = _ws(x.device, x.numel(), block)
    _lib.check(rt.lib().bsnp_cluster_fit(x.data_ptr(), x.numel(), block, m, tables.data_ptr(),
                                         ws.data_ptr(), ws.numel(), rt.stream_ptr(x.device)),
               "bsnp_cluster_fit")


def cluster_quantize_async(x: torch.Tensor, block: int, tables: torch.Tensor,
                           labels: torch.Tensor, codes: torch.Tensor) -> None:
    x = _flat_f32(x)
    ws = _ws(x.device, x.numel(), block)
    _lib.check(rt.lib().bsnp_cluster_quantize(
        x.data_ptr(), x.numel(), block, tables.data_ptr(), labels.data_ptr(), codes.data_ptr(),
        ws.data_ptr(), ws.numel(), rt.stream_ptr(x.device)), "bsnp_cluster_quantize")


def cluster_encode_async(x: torch.Tensor, m: int, block: int, tables: torch.Tensor,
                         labels: torch.Tensor, codes: torch.Tensor) -> None:
    x = _flat_f32(x)
    ws = _ws(x.device, x.numel(), block)
    _lib.check(rt.lib().bsnp_cluster_encode(
        x.data_ptr(), x.numel(), block, m, tables.data_ptr(), labels.data_ptr(),
        codes.data_ptr(), ws.data_ptr(), ws.numel(), rt.stream_ptr(x.device)),
        "bsnp_cluster_encode")


def cluster_dequantize_async(labels: torch.Tensor, codes: torch.Tensor, n: int, block: int,
                             tables: torch.Tensor, out: torch.Tensor,
                             status: torch.Tensor) -> None:
    ws = _ws(out.device, n, block)
    _lib.check(rt.lib().bsnp_cluster_dequantize(
        labels.data_ptr(), codes.data_ptr(), n, block, tables.data_ptr(), out.data_ptr(),
        status.data_ptr(), ws.data_ptr(), ws.numel(), rt.stream_ptr(out.device)),
        "bsnp_cluster_dequantize")


@dataclass
class DeviceQuant:
    """Quantized state resident in HBM (per-unit tables + labels + codes)."""

    tables: torch.Tensor   # u8 [units * 256]
    labels: torch.Tensor   # u8 [unit_label_bytes]
    codes: torch.Tensor    # u8 [n]
    n: int
    block: int
    m: int

    def host_tables(self) -> list:
        raw = rt.d2h_bytes(self.tables)
        return [ClusterTable.from_device_bytes(raw[i:i + TABLE_BYTES])
                for i in range(0, len(raw), TABLE_BYTES)]


def new_tables(n: int, block: int, device) -> torch.Tensor:
    return torch.empty(num_units(n, block) * TABLE_BYTES, dtype=torch.uint8, device=device)


def _raise_nonfinite(tables: torch.Tensor, name: str = "") -> None:
    flags = tables.view(torch.int32).view(-1, TABLE_BYTES // 4)[:, 50]
    if int(flags.max().item()) & _lib.ERR_NONFINITE:
        raise QuantizerError(f"tensor {name!r} has non-finite values (NaN/Inf); "
                             "cluster statistics are undefined")


def cluster_fit_device(x: torch.Tensor, m: int = MAX_CLUSTERS, block: int = 0) -> torch.Tensor:
    """build_clusters (quantizer.py:100-135) per unit; returns device tables."""
    _check_m(m)
    x = _flat_f32(x)
    if x.numel() == 0:
        raise QuantizerError("cannot cluster empty tensor")
    tables = new_tables(x.numel(), block, x.device)
    cluster_fit_async(x, m, block, tables)
    _raise_nonfinite(tables)
    return tables


def cluster_encode_device(x: torch.Tensor, m: int = MAX_CLUSTERS, block: int = 0,
                          check: bool = True) -> DeviceQuant:
    """build_clusters + quantize per unit, all in HBM."""
    _check_m(m)
    x = _flat_f32(x)
    n = x.numel()
    if n == 0:
        raise QuantizerError("cannot cluster empty tensor")
    dev = x.device
    tables = new_tables(n, block, dev)
    labels = torch.empty(unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
    codes = torch.empty(n, dtype=torch.uint8, device=dev)
    cluster_encode_async(x, m, block, tables, labels, codes)
    if check:
        _raise_nonfinite(tables)
    return DeviceQuant(tables, labels, codes, n, block, m)


def cluster_quantize_device(x: torch.Tensor, tables: torch.Tensor, block: int = 0):
    """quantize (quantizer.py:161-189) with given device tables -> (labels, codes)."""
    x = _flat_f32(x)
    n = x.numel()
    labels = torch.empty(unit_label_bytes(n, block), dtype=torch.uint8, device=x.device)
    codes = torch.empty(n, dtype=torch.uint8, device=x.device)
    cluster_quantize_async(x, block, tables, labels, codes)
    return labels, codes


def cluster_dequantize_device(q: DeviceQuant, out: torch.Tensor | None = None) -> torch.Tensor:
    """dequantize (quantizer.py:192-204) on device; raises on label >= m."""
    dev = q.codes.device
    if out is None:
        out = torch.empty(q.n, dtype=torch.float32, device=dev)
    st = rt.new_status(dev)
    cluster_dequantize_async(q.labels, q.codes, q.n, q.block, q.tables, out, st)
    (maxlab, flags), = rt.read_status(st)
    if flags & _lib.ERR_LABEL:
        m = q.m if q.m else q.host_tables()[0].m
        raise QuantizerError(f"label {maxlab} >= m={m}")
    return out


# ---------------------------------------------------------------------------
# compat API (reference signatures over host TensorBlob bytes)
# ---------------------------------------------------------------------------

def _device_f32(t: TensorBlob) -> torch.Tensor:
    if t.dtype is not ElementType.F32:
        raise QuantizerError(f"tensor {t.name!r} is not F32")
    return rt.h2d_bytes(t.data, rt.device_of(), torch.float32)


def build_clusters(t: TensorBlob, m: int = MAX_CLUSTERS) -> ClusterTable:
    """Fit a normal distribution to t and cut it into m quantile clusters."""
    _check_m(m)
    x = _device_f32(t)
    if x.numel() == 0:
        raise QuantizerError(f"cannot cluster empty tensor {t.name!r}")
    tables = new_tables(x.numel(), 0, x.device)
    cluster_fit_async(x, m, 0, tables)
    raw = rt.d2h_bytes(tables)
    if struct.unpack_from("<I", raw, 200)[0] & _lib.ERR_NONFINITE:
        raise QuantizerError(f"tensor {t.name!r} has non-finite values (NaN/Inf); "
                             "cluster statistics are undefined")
    return ClusterTable.from_device_bytes(raw)


def quantize(t: TensorBlob, table: ClusterTable) -> QuantizedTensor:
    """Assign each element its cluster label and nearest 8-bit code."""
    x = _device_f32(t)
    n = x.numel()
    dev = x.device
    tables = rt.h2d_bytes(table.to_device_bytes(), dev)
    if n == 0:
        return QuantizedTensor(t.name, t.shape, table, b"", b"")
    labels, codes = cluster_quantize_device(x, tables, 0)
    return QuantizedTensor(name=t.name, shape=t.shape, table=table,
                           packed_labels=rt.d2h_bytes(labels), codes=rt.d2h_bytes(codes))


def dequantize(q: QuantizedTensor) -> TensorBlob:
    """Reconstruct element i as qmap(code_i) * scale_label + offset_label."""
    n = q.num_elements
    if n == 0:
        return TensorBlob(name=q.name, dtype=ElementType.F32, shape=q.shape, data=b"")
    dev = rt.device_of()
    dq = DeviceQuant(tables=rt.h2d_bytes(q.table.to_device_bytes(), dev),
                     labels=rt.h2d_bytes(q.packed_labels, dev),
                     codes=rt.h2d_bytes(q.codes, dev), n=n, block=0, m=q.table.m)
    out = cluster_dequantize_device(dq)
    return TensorBlob(name=q.name, dtype=ElementType.F32, shape=q.shape,
                      data=rt.d2h_bytes(out))


# ---------------------------------------------------------------------------
# label packing, size laws and BSQT serialization (quantizer.py:146-277)
# ---------------------------------------------------------------------------

def pack_labels(labels) -> bytes:
    """Host format helper: two 4-bit labels per byte, low nibble = even index."""
    lab = np.asarray(labels, dtype=np.uint8).ravel()
    if lab.size % 2:
        lab = np.concatenate([lab, np.zeros(1, np.uint8)])
    return (lab[0::2] | (lab[1::2] << 4)).astype(np.uint8).tobytes()


def unpack_labels(packed: bytes, n: int) -> np.ndarray:
    b = np.frombuffer(packed, dtype=np.uint8)
    out = np.empty(b.size * 2, dtype=np.uint8)
    out[0::2] = b & 0x0F
    out[1::2] = b >> 4
    return out[:n]


def quantized_size_bytes(n: int, m: int) -> int:
    """Idealized storage cost; (3/2)n + 136 for m = 16 (quantizer.py:207-213)."""
    _check_m(m)
    return 8 * m + n + (n + 1) // 2 + 8


def serialized_quant_size(name: str, rank: int, n: int, m: int) -> int:
    """Exact size of serialize_quantized output (quantizer.py:216-226)."""
    return (7 + 8 + 4 * (m - 1) + 8 * m + 2 + len(name.encode("utf-8"))
            + 1 + 8 * rank + (n + 1) // 2 + n)


def quant_header(name: str, shape, table: ClusterTable) -> bytes:
    m = table.m
    fields = struct.pack(f"<HBff{m - 1}f{m}f{m}f", QUANT_VERSION, m, table.mean, table.std,
                         *table.boundaries, *table.scales, *table.offsets)
    return pack_shape_header(QUANT_MAGIC, fields, name, shape)


def quant_header_raw(name: str, shape, raw: bytes) -> bytes:
    """quant_header from a device table's bytes (bsnp_cluster_table): the
    f32 fields are copied as they are."""
    m = int.from_bytes(raw[196:200], "little")
    fields = (struct.pack("<HB", QUANT_VERSION, m) + raw[0:8 + 4 * (m - 1)]
              + raw[68:68 + 4 * m] + raw[132:132 + 4 * m])
    return pack_shape_header(QUANT_MAGIC, fields, name, shape)


def serialize_quantized(q: QuantizedTensor) -> bytes:
    return quant_header(q.name, q.shape, q.table) + q.packed_labels + q.codes


def deserialize_quantized(b: bytes) -> QuantizedTensor:
    cur = ByteCursor(b)
    cur.magic(QUANT_MAGIC)
    (ver,) = cur.unpack("<H")
    if ver != QUANT_VERSION:
        raise QuantizerError(f"unsupported quantized-tensor version {ver}")
    (m,) = cur.unpack("<B")
    mean, std = cur.unpack("<ff")
    bnd = cur.unpack(f"<{m - 1}f")
    scl = cur.unpack(f"<{m}f")
    off = cur.unpack(f"<{m}f")
    name, shape = cur.name_and_shape()
    n = 1
    for s in shape:
        n *= s
    packed = bytes(cur.take((n + 1) // 2))
    codes = bytes(cur.take(n))
    table = ClusterTable(m=m, mean=mean, std=std, boundaries=bnd, scales=scl, offsets=off)
    return QuantizedTensor(name=name, shape=shape, table=table, packed_labels=packed,
                           codes=codes)


def precision_report(original: TensorBlob, restored: TensorBlob) -> dict:
    """Mean relative error and mean squared error (quantizer.py:280-296),
    reduced on the device (float64 accumulation)."""
    if original.shape != restored.shape or original.dtype is not restored.dtype:
        raise QuantizerError("precision_report requires matching shape and dtype")
    o = _device_f32(original)
    r = _device_f32(restored)
    from .metrics import precision_device
    return precision_device(o, r)
