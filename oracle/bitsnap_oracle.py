"""CPU oracle for the BitSnap codec hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference algorithm
(`/root/reference/pkg/src/bitsnap/{bitmask,quantizer,tensors,store}.py`).
It exists so that `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU
baseline leg can CHECK the B200 path.  Nothing in `paper_2511_12376_b200/`
imports it; the product path never falls back to it.

Pinning: every function here is checked against golden vectors produced by
running the reference package itself (`tests/golden/make_golden.py`, run in
the build container where `/root/reference` exists) — see
`tests/test_oracle_golden.py`.  Numerics follow numpy 2.3.5 / scipy 1.18.1
(the versions of this image), the same versions the golden vectors were made
with.

Layout conventions (all little-endian, reference tensors.py:1-6):
  * F16 tensors are handled as raw uint16 bit patterns (bf16 bits travel the
    same way — the codec never interprets values, bitmask.py:79-80, 97-99).
  * F32 tensors are float32.
"""

from __future__ import annotations

import struct

import numpy as np

# Reference constants (bitmask.py:21-26, quantizer.py:263-271, tensors.py:15-17)
DELTA_MAGIC = b"BSDL"
QUANT_MAGIC = b"BSQT"
TENSOR_MAGIC = b"BSNP"
VERSION = 1
DELTA_FIXED_OVERHEAD = 33
MIN_CLUSTERS, MAX_CLUSTERS = 2, 16
MRE_EPSILON = 1e-12


class OracleDeltaError(ValueError):
    """Mirrors bitmask.DeltaError (bitmask.py:29)."""


class OracleQuantError(ValueError):
    """Mirrors quantizer.QuantizerError (quantizer.py:36)."""


# --------------------------------------------------------------------------
# Bitmask delta codec (reference bitmask.py:94-140)
# --------------------------------------------------------------------------

def delta_encode(base: np.ndarray, cur: np.ndarray):
    """bitmask.py:94-111.  Returns (mask u8[ceil(n/8)], payload u16[n_c], n_c).

    changed[i] = raw bit patterns differ; mask is LSB-first packed
    (element e -> byte e>>3, bit e&7); payload = cur[changed] in index order.
    """
    b = np.ascontiguousarray(base).view(np.uint16).ravel()
    c = np.ascontiguousarray(cur).view(np.uint16).ravel()
    if b.shape != c.shape:
        raise OracleDeltaError("shape mismatch")
    diff = b != c
    mask = np.packbits(diff, bitorder="little")
    payload = c[diff]
    return mask, payload, int(payload.size)


def delta_decode(base: np.ndarray, mask: np.ndarray, payload: np.ndarray,
                 n: int, n_c: int) -> np.ndarray:
    """bitmask.py:114-140 (validation order :128-135, then scatter :136-137)."""
    b = np.ascontiguousarray(base).view(np.uint16).ravel()
    if b.size != n:
        raise OracleDeltaError("element count mismatch")
    bits = np.unpackbits(np.asarray(mask, dtype=np.uint8), bitorder="little")
    if np.any(bits[n:]):
        raise OracleDeltaError("nonzero padding bits in mask")
    sel = bits[:n].astype(bool)
    pc = int(np.count_nonzero(sel))
    if pc != n_c:
        raise OracleDeltaError(
            f"mask popcount {pc} != recorded changed_count {n_c}")
    out = b.copy()
    out[sel] = np.asarray(payload).view(np.uint16)
    return out


def ref_encode_bytes(base: bytes, cur: bytes):
    """bitmask.py:94-111 step for step on the TensorBlob byte strings the
    reference works on (frombuffer views, count_nonzero, packbits, the
    boolean gather, both tobytes copies and the record's length checks,
    :44-54): the reference CPU cost of one encode, for the bench's CPU arm.
    Returns (mask bytes, payload bytes, n_c)."""
    b = np.frombuffer(base, dtype="<u2")
    t = np.frombuffer(cur, dtype="<u2")
    changed = b != t
    n = int(changed.size)
    n_c = int(np.count_nonzero(changed))
    mask = np.packbits(changed, bitorder="little").tobytes()
    payload = t[changed].tobytes()
    if len(mask) != (n + 7) // 8 or len(payload) != 2 * n_c:
        raise OracleDeltaError("record lengths")
    return mask, payload, n_c


def ref_decode_bytes(base: bytes, mask: bytes, payload: bytes, n: int, n_c: int) -> bytes:
    """bitmask.py:114-140 step for step on bytes (unpackbits, padding check,
    bool cast, popcount check, copy, scatter, the output tobytes copy)."""
    bits = np.unpackbits(np.frombuffer(mask, dtype=np.uint8), bitorder="little")
    if np.any(bits[n:]):
        raise OracleDeltaError("nonzero padding bits in mask")
    changed = bits[:n].astype(bool)
    if int(np.count_nonzero(changed)) != n_c:
        raise OracleDeltaError("mask popcount mismatch")
    out = np.frombuffer(base, dtype="<u2").copy()
    out[changed] = np.frombuffer(payload, dtype="<u2")
    return out.tobytes()


def delta_size(n: int, n_c: int) -> int:
    """bitmask.py:181-191 — serialized BSDL size for an empty name, rank 1."""
    if not 0 <= n_c <= n:
        raise OracleDeltaError(f"need 0 <= n_c <= n, got n={n}, n_c={n_c}")
    return (n + 7) // 8 + 2 * n_c + DELTA_FIXED_OVERHEAD


def delta_record(name: str, shape, n: int, n_c: int, mask, payload) -> bytes:
    """BSDL layout, bitmask.py:201-215."""
    nb = name.encode("utf-8")
    head = DELTA_MAGIC + struct.pack("<HQQH", VERSION, n, n_c, len(nb)) + nb
    head += struct.pack("<B", len(shape)) + b"".join(
        struct.pack("<Q", int(s)) for s in shape)
    return head + np.asarray(mask, np.uint8).tobytes() + \
        np.asarray(payload).view(np.uint16).astype("<u2").tobytes()


def raw_record(name: str, dtype_code: int, shape, data: bytes) -> bytes:
    """BSNP layout, tensors.py:110-130 (dtype_code 0 = F16, 1 = F32)."""
    nb = name.encode("utf-8")
    head = TENSOR_MAGIC + struct.pack("<HBH", VERSION, dtype_code, len(nb)) + nb
    head += struct.pack("<B", len(shape)) + b"".join(
        struct.pack("<Q", int(s)) for s in shape)
    return head + bytes(data)


# --------------------------------------------------------------------------
# numpy's pairwise summation, restated (what np.sum / np.mean / np.std do on a
# contiguous float64 vector; numpy/_core/src/umath/loops_utils.h.src).  The
# GPU fit kernels reproduce exactly this tree.  Pinned by
# tests/test_oracle_golden.py::test_pairwise_matches_numpy.
# --------------------------------------------------------------------------

PW_BLOCK = 128


def pairwise_sum(a: np.ndarray) -> float:
    a = np.asarray(a, dtype=np.float64)
    n = a.size
    if n < 8:
        res = 0.0
        for v in a:
            res = res + float(v)
        return res
    if n <= PW_BLOCK:
        body = n - (n % 8)
        r = a[:body].reshape(-1, 8)
        acc = r[0].copy()
        for row in r[1:]:
            acc = acc + row                     # 8 independent f64 chains
        res = float(((acc[0] + acc[1]) + (acc[2] + acc[3]))
                    + ((acc[4] + acc[5]) + (acc[6] + acc[7])))
        for v in a[body:]:
            res = res + float(v)
        return res
    half = (n // 2) - ((n // 2) % 8)
    return pairwise_sum(a[:half]) + pairwise_sum(a[half:])


# --------------------------------------------------------------------------
# Cluster quantizer (reference quantizer.py:100-204)
# --------------------------------------------------------------------------

def ndtri_z(m: int) -> np.ndarray:
    """Normal quantiles z_k = Phi^-1(k/m), k = 1..m-1 (quantizer.py:352-353)."""
    from scipy.special import ndtri
    return ndtri(np.arange(1, m) / m)


def cluster_fit(x: np.ndarray, m: int = 16) -> dict:
    """quantizer.py:100-135.  Returns the f32-rounded ClusterTable fields."""
    if not MIN_CLUSTERS <= m <= MAX_CLUSTERS:
        raise OracleQuantError(f"cluster count {m} outside [2, 16]")
    v = np.asarray(x, dtype=np.float32).astype(np.float64).ravel()
    if v.size == 0:
        raise OracleQuantError("cannot cluster empty tensor")
    mu = float(np.mean(v))
    sigma = float(np.std(v))
    b64 = mu + sigma * ndtri_z(m)
    lab = np.searchsorted(b64, v, side="left")
    lo = np.zeros(m)
    span = np.zeros(m)
    for c in range(m):
        sel = v[lab == c]
        if sel.size:
            lo[c] = float(sel.min())
            span[c] = float(sel.max()) - lo[c]
    return {
        "m": m,
        "mean": np.float32(mu),
        "std": np.float32(sigma),
        "boundaries": b64.astype(np.float32),
        "scales": span.astype(np.float32),
        "offsets": lo.astype(np.float32),
    }


def pack_nibbles(labels: np.ndarray) -> np.ndarray:
    """quantizer.py:146-150: low nibble = even index, odd tail padded with 0."""
    lab = np.asarray(labels, dtype=np.uint8).ravel()
    if lab.size % 2:
        lab = np.concatenate([lab, np.zeros(1, np.uint8)])
    return (lab[0::2] | (lab[1::2] << 4)).astype(np.uint8)


def unpack_nibbles(packed: np.ndarray, n: int) -> np.ndarray:
    """quantizer.py:153-158."""
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty(p.size * 2, np.uint8)
    out[0::2] = p & 0xF
    out[1::2] = p >> 4
    return out[:n]


def cluster_quantize(x: np.ndarray, table: dict):
    """quantizer.py:161-189.  Returns (packed labels u8, codes u8, labels u8)."""
    v = np.asarray(x, dtype=np.float32).astype(np.float64).ravel()
    bnd = np.asarray(table["boundaries"], dtype=np.float32).astype(np.float64)
    lab = np.searchsorted(bnd, v, side="left").astype(np.uint8)
    if int(lab.max(initial=0)) >= table["m"]:
        raise OracleQuantError("internal: label overflow")
    s = np.asarray(table["scales"], np.float32).astype(np.float64)[lab]
    b = np.asarray(table["offsets"], np.float32).astype(np.float64)[lab]
    xn = np.zeros_like(v)
    occ = s > 0
    xn[occ] = (v[occ] - b[occ]) / s[occ]
    np.clip(xn, 0.0, 1.0, out=xn)
    codes = np.clip(np.ceil(xn * 255.0 - 0.5).astype(np.int64), 0, 255)
    return pack_nibbles(lab), codes.astype(np.uint8), lab


def cluster_dequantize(packed: np.ndarray, codes: np.ndarray, n: int,
                       table: dict) -> np.ndarray:
    """quantizer.py:192-204."""
    lab = unpack_nibbles(packed, n)
    if n and int(lab.max()) >= table["m"]:
        raise OracleQuantError(f"label {int(lab.max())} >= m={table['m']}")
    s = np.asarray(table["scales"], np.float32).astype(np.float64)[lab]
    b = np.asarray(table["offsets"], np.float32).astype(np.float64)[lab]
    q = np.asarray(codes, dtype=np.uint8).astype(np.float64) / 255.0
    return (q * s + b).astype(np.float32)


def quant_record(name: str, shape, table: dict, packed, codes) -> bytes:
    """BSQT layout, quantizer.py:229-248."""
    m = table["m"]
    nb = name.encode("utf-8")
    f = lambda a: np.asarray(a, np.float32).astype("<f4").tobytes()
    head = QUANT_MAGIC + struct.pack("<HB", VERSION, m)
    head += f([table["mean"], table["std"]]) + f(table["boundaries"])
    head += f(table["scales"]) + f(table["offsets"])
    head += struct.pack("<H", len(nb)) + nb + struct.pack("<B", len(shape))
    head += b"".join(struct.pack("<Q", int(s)) for s in shape)
    return head + np.asarray(packed, np.uint8).tobytes() + \
        np.asarray(codes, np.uint8).tobytes()


def quant_record_size(name: str, rank: int, n: int, m: int) -> int:
    """quantizer.py:216-226."""
    return (7 + 8 + 4 * (m - 1) + 8 * m + 2 + len(name.encode("utf-8"))
            + 1 + 8 * rank + (n + 1) // 2 + n)


def precision(orig: np.ndarray, rest: np.ndarray) -> dict:
    """quantizer.py:280-296."""
    o = np.asarray(orig, np.float32).astype(np.float64).ravel()
    r = np.asarray(rest, np.float32).astype(np.float64).ravel()
    err = o - r
    mse = float(np.mean(err ** 2)) if o.size else 0.0
    sig = np.abs(o) > MRE_EPSILON
    mre = float(np.mean(np.abs(err[sig]) / np.abs(o[sig]))) if np.any(sig) else 0.0
    return {"mre": mre, "mse": mse}


def blockwise(x: np.ndarray, block: int):
    """Per-block mode: the reference applied to each slice."""
    x = np.asarray(x).ravel()
    return [x[i:i + block] for i in range(0, x.size, block)] if block else [x]


# --------------------------------------------------------------------------
# Checkpoint driver (reference store.py:214-272): per-tensor codec choice and
# sequential offsets.  Tensors are (name, shape, dtype_code, ndarray).
# --------------------------------------------------------------------------

def encode_checkpoint(model, optimizer, prev_model, kind: str, clusters: int = 16):
    entries, chunks, off = [], [], 0

    def add(name, group, codec, blob):
        nonlocal off
        entries.append({"name": name, "group": group, "codec": codec,
                        "offset": off, "length": len(blob)})
        chunks.append(blob)
        off += len(blob)

    prev = {t[0]: t for t in (prev_model or [])}
    for name, shape, _, arr in model:
        raw = raw_record(name, 0, shape, np.asarray(arr).view(np.uint16).tobytes())
        if kind == "base":
            add(name, "model", "RAW", raw)
            continue
        mask, payload, n_c = delta_encode(prev[name][3], arr)
        enc = delta_record(name, shape, int(np.prod(shape, dtype=np.int64)), n_c,
                           mask, payload)
        if len(enc) < len(raw):
            add(name, "model", "DELTA", enc)
        else:
            add(name, "model", "RAW", raw)
    for name, shape, _, arr in optimizer:
        tab = cluster_fit(arr, clusters)
        packed, codes, _ = cluster_quantize(arr, tab)
        add(name, "optimizer", "QUANT", quant_record(name, shape, tab, packed, codes))
    return entries, b"".join(chunks)
