"""The reference's own hot-path tests, restated against this package's
reference-named API (INTEGRATION.md option A: `from paper_2511_12376_b200
import bitmask, quantizer` in place of `bitsnap.bitmask / quantizer`):

  * pkg/tests/test_bitmask.py — KATs, round trips, errors, chain_encode
    (:128-185), size laws (:195-260);
  * pkg/tests/test_quantizer.py — boundaries, degenerate tensors, balance,
    endpoints, the 256-way argmin oracle, error bounds, sizes, packing,
    precision report;
  * pkg/tests/test_acceptance.py::test_01..07 — the SPEC's codec criteria.

Same seeds and shapes as the reference (its `rng` fixture is
default_rng(1234), pkg/tests/conftest.py:7-9); the synthetic generators of
pkg/src/bitsnap/synth.py:10-78 are restated below.  Every call runs the
sm_100a kernels through the C-ABI.
"""

import math
import time

import numpy as np
import pytest

from paper_2511_12376_b200 import bitmask as B
from paper_2511_12376_b200 import quantizer as Q
from paper_2511_12376_b200.tensors import Checkpoint, ElementType, TensorBlob

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------- synth (restated)
def random_f16_blob(rng, name, shape):
    n = int(np.prod(shape, dtype=np.int64)) if len(shape) else 1
    bits = rng.integers(0, 1 << 16, size=n, dtype=np.uint16)
    return TensorBlob(name, ElementType.F16, tuple(shape), bits.astype("<u2").tobytes())


def random_f32_blob(rng, name, shape, scale=1.0):
    n = int(np.prod(shape, dtype=np.int64)) if len(shape) else 1
    return TensorBlob(name, ElementType.F32, tuple(shape),
                      rng.normal(0.0, scale, size=n).astype("<f4").tobytes())


def random_checkpoint(rng, iteration):
    model = {"layer0.weight": (64, 32), "layer1.weight": (128,)}
    opt = {"adam.exp_avg": (64, 32), "adam.exp_avg_sq": (128,)}
    return Checkpoint(iteration=iteration,
                      model_states=tuple(random_f16_blob(rng, k, s) for k, s in model.items()),
                      optimizer_states=tuple(random_f32_blob(rng, k, s) for k, s in opt.items()))


def perturb_checkpoint(rng, ckpt, iteration, frac):
    model = []
    for t in ckpt.model_states:
        v = np.frombuffer(t.data, dtype="<u2").copy()
        k = int(round(v.size * frac))
        if k:
            idx = rng.choice(v.size, size=k, replace=False)
            v[idx] ^= rng.integers(1, 1 << 16, size=k, dtype=np.uint16)
        model.append(TensorBlob(t.name, t.dtype, t.shape, v.tobytes()))
    return Checkpoint(iteration=iteration, model_states=tuple(model),
                      optimizer_states=ckpt.optimizer_states)


def f16_blob(values_u16, name="t", shape=None):
    arr = np.asarray(values_u16, dtype="<u2")
    return TensorBlob(name, ElementType.F16, tuple(shape or (arr.size,)), arr.tobytes())


def f32_blob(values, name="t"):
    arr = np.asarray(values, dtype="<f4")
    return TensorBlob(name, ElementType.F32, (arr.size,), arr.tobytes())


# ------------------------------------------------------- test_bitmask.py
def test_identical_tensors_give_empty_delta(rng):
    t = random_f16_blob(rng, "w", (100,))
    rec = B.encode_delta(t, t)
    assert (rec.changed_count, rec.payload, rec.packed_mask) == (0, b"", b"\x00" * 13)


def test_hand_packed_mask_byte():
    vals = list(range(8))
    vals[1], vals[6] = 1000, 2000
    rec = B.encode_delta(f16_blob(range(8)), f16_blob(vals))
    assert rec.packed_mask == b"\x42" and rec.changed_count == 2
    assert np.frombuffer(rec.payload, dtype="<u2").tolist() == [1000, 2000]


def test_padding_bits_are_zero(rng):
    rec = B.encode_delta(random_f16_blob(rng, "w", (13,)), random_f16_blob(rng, "w", (13,)))
    assert rec.packed_mask[-1] >> 5 == 0


def test_all_zero_mask_and_random_round_trips(rng):
    base = random_f16_blob(rng, "w", (64,))
    assert B.decode_delta(base, B.encode_delta(base, base)).data == base.data
    for _ in range(300):
        n = int(rng.integers(1, 500))
        a, b = random_f16_blob(rng, "w", (n,)), random_f16_blob(rng, "w", (n,))
        assert B.decode_delta(a, B.encode_delta(a, b)).data == b.data


def test_nan_and_signed_zero_payloads_roundtrip():
    base, target = f16_blob([0x0000, 0x3C00, 0x0000]), f16_blob([0x8000, 0x7E00, 0x0000])
    rec = B.encode_delta(base, target)
    assert rec.changed_count == 2 and B.decode_delta(base, rec).data == target.data


def test_mismatch_and_corruption_errors(rng):
    a, b = random_f16_blob(rng, "a", (4,)), random_f16_blob(rng, "b", (4,))
    c = random_f16_blob(rng, "a", (5,))
    f32 = TensorBlob("a", ElementType.F32, (4,), b"\x00" * 16)
    for x, y, key in ((a, b, "name"), (a, c, "shape"), (f32, f32, "F16")):
        with pytest.raises(B.DeltaError, match=key):
            B.encode_delta(x, y)
    base, target = random_f16_blob(rng, "w", (32,)), random_f16_blob(rng, "w", (32,))
    rec = B.encode_delta(base, target)
    with pytest.raises(B.DeltaError):
        B.DeltaRecord(rec.tensor_name, rec.shape, rec.total_elements, rec.changed_count,
                      rec.packed_mask, rec.payload + b"\x00\x00")
    base, target = random_f16_blob(rng, "w", (16,)), random_f16_blob(rng, "w", (16,))
    rec = B.encode_delta(base, target)
    assert rec.changed_count > 0
    bad = B.DeltaRecord(rec.tensor_name, rec.shape, rec.total_elements, rec.changed_count,
                        b"\x00" * len(rec.packed_mask), rec.payload)
    with pytest.raises(B.DeltaError, match="popcount"):
        B.decode_delta(base, bad)


def test_chain_encode_identity_base():
    base = random_checkpoint(np.random.default_rng(7), 0)
    same = random_checkpoint(np.random.default_rng(7), 1)
    deltas = B.chain_encode(base, [same])
    assert len(deltas) == 1 and deltas[0].base_iteration == 0 and deltas[0].iteration == 1
    assert all(r.changed_count == 0 for r in deltas[0].records)


def test_chain_disjoint_changes_are_independent(rng):
    base = random_f16_blob(rng, "w", (90,))
    prev = np.frombuffer(base.data, dtype="<u2")
    targets = []
    for lo, hi in [(0, 10), (30, 45), (60, 80)]:
        nxt = prev.copy()
        nxt[lo:hi] ^= 0x1111
        targets.append(nxt)
        prev = nxt
    ckpts = [Checkpoint(iteration=i + 1, model_states=(f16_blob(t, name="w"),))
             for i, t in enumerate(targets)]
    deltas = B.chain_encode(Checkpoint(iteration=0, model_states=(base,)), ckpts)
    # each step's count is that step's span: every delta is against its predecessor
    assert [d.records[0].changed_count for d in deltas] == [10, 15, 20]
    assert [d.base_iteration for d in deltas] == [0, 1, 2]


def test_chain_apply_reconstructs_final(rng):
    chain = [random_checkpoint(rng, 0)]
    for i in range(5):
        chain.append(perturb_checkpoint(rng, chain[-1], i + 1, 0.1))
    deltas = B.chain_encode(chain[0], chain[1:])
    cur = {t.name: t for t in chain[0].model_states}
    for dc in deltas:
        cur = {r.tensor_name: B.decode_delta(cur[r.tensor_name], r) for r in dc.records}
    for t in chain[-1].model_states:
        assert cur[t.name].data == t.data
    # and each record equals a direct encode against the predecessor
    for prev, tgt, dc in zip(chain, chain[1:], deltas):
        pm = {t.name: t for t in prev.model_states}
        for t, r in zip(tgt.model_states, dc.records):
            assert B.serialize_delta(r) == B.serialize_delta(B.encode_delta(pm[t.name], t))


def test_chain_rejects_non_increasing_iterations_and_structure(rng):
    base = random_checkpoint(rng, 5)
    with pytest.raises(B.DeltaError, match="increasing"):
        B.chain_encode(base, [random_checkpoint(rng, 5)])
    other = Checkpoint(iteration=6, model_states=(random_f16_blob(rng, "x", (3,)),))
    with pytest.raises(B.DeltaError, match="structure"):
        B.chain_encode(base, [other])


def test_size_laws(rng):
    assert B.delta_size_bytes(16, 0) == 2 + B.DELTA_FIXED_OVERHEAD
    for _ in range(50):
        n = int(rng.integers(1, 300))
        rec = B.encode_delta(random_f16_blob(rng, "weight", (n,)),
                             random_f16_blob(rng, "weight", (n,)))
        b = B.serialize_delta(rec)
        assert len(b) == B.delta_size_bytes(n, rec.changed_count) + len("weight") \
            == rec.serialized_size
        assert B.deserialize_delta(b) == rec
    base = random_f16_blob(rng, "w", (256,))
    arr = np.frombuffer(base.data, dtype="<u2")
    sizes = set()
    for _ in range(10):
        t = arr.copy()
        t[rng.choice(256, size=40, replace=False)] ^= 0x0101
        rec = B.encode_delta(base, f16_blob(t, name="w"))
        assert rec.changed_count == 40
        sizes.add(rec.serialized_size)
    assert len(sizes) == 1
    n = 1 << 16
    for n_c in range(0, n + 1, 997):
        assert (B.delta_size_bytes(n, n_c) < 2 * n) == \
            (n_c < (15 / 16) * n - B.DELTA_FIXED_OVERHEAD / 2)
    assert B.naive_delta_size_bytes(n, n // 2 - B.DELTA_FIXED_OVERHEAD) < 2 * n
    assert B.naive_delta_size_bytes(n, n // 2 + 1) >= 2 * n
    n = 1 << 20
    r = [2 * n / B.delta_size_bytes(n, int(f * n)) for f in np.linspace(0, 1, 33)]
    assert all(a > b for a, b in zip(r, r[1:]))
    with pytest.raises(B.DeltaError):
        B.delta_size_bytes(10, 11)


# ----------------------------------------------------- test_quantizer.py
def _inverse_normal_cdf(p):
    lo, hi = -20.0, 20.0
    for _ in range(200):
        mid = (lo + hi) / 2
        if 0.5 * (1 + math.erf(mid / math.sqrt(2))) < p:
            lo = mid
        else:
            hi = mid
    return (lo + hi) / 2


def test_boundaries(rng):
    t = random_f32_blob(rng, "t", (1000,))
    v = np.frombuffer(t.data, dtype="<f4").astype(np.float64)
    assert Q.build_clusters(t, 2).boundaries[0] == pytest.approx(np.mean(v), abs=1e-5)
    t = random_f32_blob(rng, "t", (10_000,))
    table = Q.build_clusters(t, 4)
    v = np.frombuffer(t.data, dtype="<f4").astype(np.float64)
    for k, b in enumerate(table.boundaries, start=1):
        assert b == pytest.approx(np.mean(v) + np.std(v) * _inverse_normal_cdf(k / 4),
                                  rel=1e-5, abs=1e-7)


def test_constant_tensor_and_validation(rng):
    t = f32_blob([3.25] * 100)
    table = Q.build_clusters(t, 8)
    assert all(b == pytest.approx(3.25) for b in table.boundaries)
    q = Q.quantize(t, table)
    assert set(Q.unpack_labels(q.packed_labels, 100).tolist()) == {0}
    assert set(q.codes) == {0}
    assert np.all(np.frombuffer(Q.dequantize(q).data, dtype="<f4") == np.float32(3.25))
    t = f32_blob([-7.5] * 33)
    assert Q.dequantize(Q.quantize(t, Q.build_clusters(t, 16))).data == t.data
    for m in (0, 1, 17):
        with pytest.raises(Q.QuantizerError):
            Q.build_clusters(random_f32_blob(rng, "t", (10,)), m)
    with pytest.raises(Q.QuantizerError):
        Q.build_clusters(f32_blob([]), 4)


def test_balance_and_endpoints(rng):
    n, m = 200_000, 16
    t = random_f32_blob(rng, "t", (n,))
    table = Q.build_clusters(t, m)
    v = np.frombuffer(t.data, dtype="<f4").astype(np.float64)
    counts = np.bincount(np.searchsorted(np.asarray(table.boundaries), v, side="left"),
                         minlength=m)
    assert np.all(np.abs(counts - n / m) <= 5 * math.sqrt(n))
    t = random_f32_blob(rng, "t", (5000,))
    q = Q.quantize(t, Q.build_clusters(t, 4))
    v = np.frombuffer(t.data, dtype="<f4")
    lab = Q.unpack_labels(q.packed_labels, v.size)
    codes = np.frombuffer(q.codes, dtype=np.uint8)
    for c in range(4):
        sel = lab == c
        if sel.any():
            assert codes[sel][np.argmin(v[sel])] == 0
            assert codes[sel][np.argmax(v[sel])] == 255


def _argmin_codes(values, labels, table):
    s = np.asarray(table.scales)[labels]
    b = np.asarray(table.offsets)[labels]
    x = np.clip(np.where(s > 0, (values - b) / np.where(s > 0, s, 1.0), 0.0), 0.0, 1.0)
    grid = Q.qmap(np.arange(256))
    out = np.empty(values.size, np.uint8)
    for lo in range(0, values.size, 1 << 16):
        c = x[lo:lo + (1 << 16)]
        out[lo:lo + c.size] = np.abs(grid[None, :] - c[:, None]).argmin(axis=1)
    return out


def test_codes_match_exhaustive_argmin_oracle(rng):
    t = random_f32_blob(rng, "t", (10_000,))
    table = Q.build_clusters(t, 16)
    q = Q.quantize(t, table)
    v = np.frombuffer(t.data, dtype="<f4").astype(np.float64)
    assert np.array_equal(np.frombuffer(q.codes, np.uint8),
                          _argmin_codes(v, Q.unpack_labels(q.packed_labels, v.size), table))


def test_error_bound_per_element(rng):
    for _ in range(100):
        n = int(rng.integers(10, 2000))
        t = random_f32_blob(rng, "t", (n,), scale=float(rng.uniform(0.01, 10)))
        q = Q.quantize(t, Q.build_clusters(t, int(rng.integers(2, 17))))
        r = np.frombuffer(Q.dequantize(q).data, dtype="<f4").astype(np.float64)
        v = np.frombuffer(t.data, dtype="<f4").astype(np.float64)
        s = np.asarray(q.table.scales)[Q.unpack_labels(q.packed_labels, n)]
        assert np.all(np.abs(r - v) <= s / 510 + np.abs(v) * 1e-6 + 1e-12)


def test_label_overflow_sizes_packing(rng):
    t = random_f32_blob(rng, "t", (8,))
    q = Q.quantize(t, Q.build_clusters(t, 2))
    bad = type(q)(name=q.name, shape=q.shape, table=q.table,
                  packed_labels=Q.pack_labels(np.full(8, 9, dtype=np.uint8)), codes=q.codes)
    with pytest.raises(Q.QuantizerError, match="label"):
        Q.dequantize(bad)
    assert Q.quantized_size_bytes(1_000_000, 16) == 1_500_136
    assert Q.quantized_size_bytes(0, 16) == 8 * 16 + 8
    with pytest.raises(Q.QuantizerError):
        Q.quantized_size_bytes(100, 1)
    for n in (1, 2, 101, 5000):
        t = random_f32_blob(rng, "moments", (n,))
        q = Q.quantize(t, Q.build_clusters(t, 16))
        b = Q.serialize_quantized(q)
        assert len(b) == Q.serialized_quant_size("moments", 1, n, 16)
        assert len(b) == Q.quantized_size_bytes(n, 16) - (8 * 16 + 8) + \
            Q.serialized_quant_size("moments", 1, 0, 16)
        assert Q.deserialize_quantized(b) == q
    for n in (0, 1, 2, 7, 8, 33):
        lab = rng.integers(0, 16, size=n).astype(np.uint8)
        packed = Q.pack_labels(lab)
        assert len(packed) == (n + 1) // 2 and np.array_equal(Q.unpack_labels(packed, n), lab)


def test_precision_report(rng):
    t = random_f32_blob(rng, "t", (100,))
    assert Q.precision_report(t, t) == {"mre": 0.0, "mse": 0.0}
    o = np.array([1.0, -2.0, 4.0, 0.0], dtype="<f4")
    r = np.array([1.1, -2.2, 3.6, 0.5], dtype="<f4")
    rep = Q.precision_report(f32_blob(o), f32_blob(r))
    err = o.astype(np.float64) - r.astype(np.float64)
    assert rep["mse"] == pytest.approx(np.mean(err ** 2), rel=1e-12)
    assert rep["mre"] == pytest.approx(np.mean(np.abs(err[:3]) / np.abs(o[:3].astype(np.float64))),
                                       rel=1e-12)
    o = rng.normal(0, 1, size=10_000).astype("<f4")
    r = (o.astype(np.float64) + 1e-7).astype("<f4")
    assert Q.precision_report(f32_blob(o), f32_blob(r))["mse"] < 1e-13
    with pytest.raises(Q.QuantizerError):
        Q.precision_report(random_f32_blob(rng, "a", (4,)), random_f32_blob(rng, "a", (5,)))


# ----------------------------------------------- test_acceptance.py 01..07
def test_01_bitmask_losslessness_10k_pairs():
    rng = np.random.default_rng(0)
    specials = np.array([0x0000, 0x8000, 0x7E00, 0xFE00, 0x7C00, 0xFC00], dtype=np.uint16)
    start = time.monotonic()
    for i in range(10_000):
        n = int(rng.integers(1, 257))
        bv = rng.integers(0, 1 << 16, size=n, dtype=np.uint16)
        tv = bv.copy()
        k = int(rng.integers(0, n + 1))
        if k:
            idx = rng.choice(n, size=k, replace=False)
            tv[idx] = rng.choice(specials, size=k) if i % 3 else \
                rng.integers(0, 1 << 16, size=k, dtype=np.uint16)
        shape = (n,) if i % 2 else (1, n)
        base, target = f16_blob(bv, "w", shape), f16_blob(tv, "w", shape)
        assert B.decode_delta(base, B.encode_delta(base, target)).data == target.data
    assert time.monotonic() - start < 60.0


def test_02_sixteen_x_ceiling():
    n = 1 << 20
    t = f16_blob(np.random.default_rng(1).integers(0, 1 << 16, size=n, dtype=np.uint16), "w")
    rec = B.encode_delta(t, t)
    size = len(B.serialize_delta(rec))
    assert rec.changed_count == 0 and size == (n + 7) // 8 + B.DELTA_FIXED_OVERHEAD + 1
    assert 15.5 <= 2 * n / size <= 16.0


def test_03_five_x_at_fifteen_percent():
    n = 1 << 20
    n_c = int(0.15 * n)
    rng = np.random.default_rng(2)
    bv = rng.integers(0, 1 << 16, size=n, dtype=np.uint16)
    tv = bv.copy()
    tv[rng.choice(n, size=n_c, replace=False)] ^= 0x0001
    rec = B.encode_delta(f16_blob(bv, "w"), f16_blob(tv, "w"))
    assert rec.changed_count == n_c
    ratio, expected = 2 * n / len(B.serialize_delta(rec)), 2 / (0.125 + 0.30)
    assert abs(ratio - expected) / expected <= 0.02


def test_04_benefit_threshold_crossing():
    n = 1 << 20
    adj = lambda f: 2 * n / (B.delta_size_bytes(n, int(f * n)) - B.DELTA_FIXED_OVERHEAD)
    assert adj(0.90) > 1.0 and adj(0.9375) == 1.0 and adj(0.95) < 1.0


def test_05_quantizer_exhaustive_oracle_equivalence():
    n = 1_000_000
    t = random_f32_blob(np.random.default_rng(3), "t", (n,))
    table = Q.build_clusters(t, 16)
    q = Q.quantize(t, table)
    v = np.frombuffer(t.data, dtype="<f4").astype(np.float64)
    want = _argmin_codes(v, Q.unpack_labels(q.packed_labels, n), table)
    assert int(np.count_nonzero(np.frombuffer(q.codes, np.uint8) != want)) == 0


def test_06_quantizer_ratio():
    n, m = 1_000_000, 16
    t = random_f32_blob(np.random.default_rng(4), "t", (n,))
    size = len(Q.serialize_quantized(Q.quantize(t, Q.build_clusters(t, m))))
    assert size == Q.serialized_quant_size("t", 1, n, m)
    ideal = (3 * n) // 2 + 136
    assert abs(size - ideal) / ideal <= 0.001 and 4 * n / size >= 2.5


def test_07_quantizer_error_bound_and_mse():
    rng = np.random.default_rng(5)
    for _ in range(100):
        n = int(rng.integers(64, 5000))
        t = random_f32_blob(rng, "t", (n,), scale=float(rng.uniform(1e-3, 100.0)))
        q = Q.quantize(t, Q.build_clusters(t, 16))
        v = np.frombuffer(t.data, dtype="<f4").astype(np.float64)
        r = np.frombuffer(Q.dequantize(q).data, dtype="<f4").astype(np.float64)
        s = np.asarray(q.table.scales)[Q.unpack_labels(q.packed_labels, n)]
        ulp = np.spacing(np.abs(v).astype(np.float32)).astype(np.float64)
        assert np.all(np.abs(r - v) <= s / 510 + ulp)
    t = random_f32_blob(np.random.default_rng(6), "t", (1_000_000,), scale=1.0)
    r = Q.dequantize(Q.quantize(t, Q.build_clusters(t, 16)))
    err = (np.frombuffer(t.data, dtype="<f4").astype(np.float64)
           - np.frombuffer(r.data, dtype="<f4").astype(np.float64))
    assert float(np.mean(err ** 2)) <= 1e-5


# ------------------------------------------------------ empty tensors (edge)
# BSDL bytes of the reference's encode_delta on an empty F16 tensor named "e"
# (run here: bitmask.py:94-111 + serialize_delta :201-215): n = n_c = 0, no
# mask, no payload
_EMPTY_BSDL = {
    (0,): "4253444c010000000000000000000000000000000000010065010000000000000000",
    (3, 0): "4253444c0100000000000000000000000000000000000100650203000000000000000000000000000000",
}


@pytest.mark.parametrize("shape", [(0,), (3, 0)])
def test_empty_tensor_delta(shape):
    """An empty tensor encodes to the reference's header-only record and
    decodes back to itself (no kernel needs to touch a byte)."""
    a = TensorBlob("e", ElementType.F16, shape, b"")
    rec = B.encode_delta(a, a)
    assert rec.total_elements == 0 and rec.changed_count == 0
    assert B.serialize_delta(rec).hex() == _EMPTY_BSDL[shape]
    assert B.deserialize_delta(bytes.fromhex(_EMPTY_BSDL[shape])) == rec
    out = B.decode_delta(a, rec)
    assert out.shape == shape and out.data == b""
    assert B.delta_size_bytes(0, 0) + 8 * (len(shape) - 1) + 1 == len(B.serialize_delta(rec))
