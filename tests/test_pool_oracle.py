"""The fanned-out oracle (tests/pool_oracle.py) returns exactly what the
single-process oracle returns (it is the checker of the full-size GPU parity
tests, tests/test_fullsize_gpu.py)."""

import numpy as np
import pytest

from oracle import bitsnap_oracle as O
import pool_oracle as PO


def _same_table(a, b):
    for k in ("mean", "std", "boundaries", "scales", "offsets"):
        assert np.asarray(a[k], np.float32).tobytes() == np.asarray(b[k], np.float32).tobytes(), k


def test_delta_encode_chunks_concatenate():
    rng = np.random.default_rng(3)
    n = 100003
    base = rng.integers(0, 1 << 16, n, dtype=np.uint16)
    cur = base.copy()
    idx = rng.choice(n, 2000, replace=False)
    cur[idx] ^= 1
    want = O.delta_encode(base, cur)
    got = PO.delta_encode(base, cur, chunk=8 * 1001)
    assert got[2] == want[2]
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


@pytest.mark.parametrize("dist", ["m", "v", "spiky"])
def test_cluster_fit_and_quantize_chunks(dist):
    rng = np.random.default_rng(len(dist))
    n = 300007
    x = rng.standard_normal(n) * 1e-3
    if dist == "v":
        x = x * x
    if dist == "spiky":
        x[rng.choice(n, 50, replace=False)] = 7.0
    x = x.astype(np.float32)
    for m in (16, 5):
        want = O.cluster_fit(x, m)
        got = PO.cluster_fit(x, m, chunk=65536)
        _same_table(got, want)
        wp, wc, wl = O.cluster_quantize(x, want)
        gp, gc, gl = PO.cluster_quantize(x, got, chunk=40000)
        assert np.array_equal(gp, wp) and np.array_equal(gc, wc)


def test_blockwise_matches_per_block_oracle():
    rng = np.random.default_rng(9)
    block = 4096
    x = (rng.standard_normal(5 * block + 77) * 1e-3).astype(np.float32)
    res = PO.blockwise(x, block, 16, full=(0, 5), deq=(5,))
    assert len(res) == 6
    for u, r in enumerate(res):
        xs = x[u * block:(u + 1) * block]
        _same_table(r["table"], O.cluster_fit(xs, 16))
    p, c, _ = O.cluster_quantize(x[5 * block:], res[5]["table"])
    assert np.array_equal(res[5]["codes"], c) and np.array_equal(res[5]["packed"], p)
    assert np.array_equal(res[5]["deq"], O.cluster_dequantize(p, c, x.size - 5 * block,
                                                               res[5]["table"]))
