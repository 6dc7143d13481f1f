"""The CPU oracle fanned out over the host's cores, for parity checks at the
BASELINE configs' full sizes (test infrastructure only).

Every function here returns exactly what the single-process oracle returns:
  * delta_encode over 8-aligned element ranges: the mask bytes and payloads of
    consecutive ranges concatenate to the whole tensor's (bitmask.py:97-103:
    packbits is per byte, the payload keeps ascending element order);
  * cluster_fit: mean / std are numpy's pairwise reductions of the WHOLE unit
    (computed once, in the parent), the labels against the float64 boundaries
    are elementwise and the per-cluster min / max are order-independent, so
    they are taken per range and folded (quantizer.py:110-125);
  * cluster_quantize is elementwise given the table (quantizer.py:161-189);
  * per-block units are independent: one task per block.
Workers are forked after the arrays are set as module globals, so nothing is
pickled but indices.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import warnings

import numpy as np

from oracle import bitsnap_oracle as O

_G: dict = {}
_CHUNK = 1 << 24


def cores() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def _pool():
    # the workers only run numpy on the parent's arrays (no CUDA, no locks)
    warnings.filterwarnings("ignore", "This process .* is multi-threaded", DeprecationWarning)
    return mp.get_context("fork").Pool(cores())


def _ranges(n: int, chunk: int = _CHUNK):
    return [(s, min(n, s + chunk)) for s in range(0, n, chunk)]


# ------------------------------------------------------------------ bitmask
def _delta_part(r):
    s, e = r
    mask, payload, n_c = O.delta_encode(_G["base"][s:e], _G["cur"][s:e])
    return mask, payload, n_c


def delta_encode(base: np.ndarray, cur: np.ndarray, chunk: int = _CHUNK):
    """== O.delta_encode(base, cur) -> (mask, payload, n_c)."""
    assert chunk % 8 == 0
    _G["base"], _G["cur"] = base, cur
    with _pool() as p:
        parts = p.map(_delta_part, _ranges(base.size, chunk))
    return (np.concatenate([m for m, _, _ in parts]),
            np.concatenate([q for _, q, _ in parts]),
            sum(k for _, _, k in parts))


# ---------------------------------------------------------------- quantizer
def _fit_part(r):
    s, e = r
    v = _G["x"][s:e].astype(np.float64)
    lab = np.searchsorted(_G["b64"], v, side="left")
    m = _G["m"]
    lo = np.full(m, np.inf)
    hi = np.full(m, -np.inf)
    cnt = np.bincount(lab, minlength=m)
    for c in range(m):
        if cnt[c]:
            sel = v[lab == c]
            lo[c] = sel.min()
            hi[c] = sel.max()
    return lo, hi, cnt


def cluster_fit(x: np.ndarray, m: int = 16, chunk: int = _CHUNK) -> dict:
    """== O.cluster_fit(x, m) for one (large) unit."""
    v = np.asarray(x, np.float32).astype(np.float64).ravel()
    mu = float(np.mean(v))
    sigma = float(np.std(v))
    del v
    b64 = mu + sigma * O.ndtri_z(m)
    _G["x"], _G["b64"], _G["m"] = np.asarray(x, np.float32).ravel(), b64, m
    with _pool() as p:
        parts = p.map(_fit_part, _ranges(x.size, chunk))
    lo = np.min([a for a, _, _ in parts], axis=0)
    hi = np.max([b for _, b, _ in parts], axis=0)
    cnt = np.sum([c for _, _, c in parts], axis=0)
    offs = np.where(cnt > 0, lo, 0.0)
    span = np.where(cnt > 0, hi - np.where(cnt > 0, lo, 0.0), 0.0)
    return {"m": m, "mean": np.float32(mu), "std": np.float32(sigma),
            "boundaries": b64.astype(np.float32), "scales": span.astype(np.float32),
            "offsets": offs.astype(np.float32)}


def _quant_part(r):
    s, e = r
    _, codes, lab = O.cluster_quantize(_G["x"][s:e], _G["table"])
    return codes, lab


def cluster_quantize(x: np.ndarray, table: dict, chunk: int = 1 << 22):
    """== O.cluster_quantize(x, table) -> (packed labels, codes, labels)."""
    _G["x"], _G["table"] = np.asarray(x, np.float32).ravel(), table
    with _pool() as p:
        parts = p.map(_quant_part, _ranges(x.size, chunk))
    codes = np.concatenate([c for c, _ in parts])
    lab = np.concatenate([l for _, l in parts])
    return O.pack_nibbles(lab), codes, lab


def _block_part(u):
    block, m = _G["block"], _G["m"]
    xs = _G["x"][u * block:(u + 1) * block]
    t = O.cluster_fit(xs, m)
    out = {"table": t}
    if u in _G["full"]:
        packed, codes, _ = O.cluster_quantize(xs, t)
        out["packed"], out["codes"] = packed, codes
        if u in _G["deq"]:
            out["deq"] = O.cluster_dequantize(packed, codes, xs.size, t)
    return out


def blockwise(x: np.ndarray, block: int, m: int, full=(), deq=()):
    """O.cluster_fit of every block; labels / codes of the blocks in `full`
    and the dequantized values of those in `deq` (== the single-process
    oracle applied per block)."""
    x = np.asarray(x, np.float32).ravel()
    _G.update(x=x, block=block, m=m, full=set(full), deq=set(deq))
    units = (x.size + block - 1) // block
    with _pool() as p:
        return p.map(_block_part, range(units), chunksize=4)
