"""Pin the CPU oracle against the reference's own outputs (golden vectors
made by tests/golden/make_golden.py from /root/reference).  CPU only."""

import hashlib
import json
import os
import struct
import sys

import numpy as np
import pytest

from oracle import bitsnap_oracle as O


def _bsdl_fields(b: bytes):
    assert b[:4] == b"BSDL"
    ver, n, n_c, nl = struct.unpack_from("<HQQH", b, 4)
    p = 4 + 2 + 8 + 8 + 2
    name = b[p:p + nl].decode("utf-8"); p += nl
    rank = b[p]; p += 1
    shape = struct.unpack_from(f"<{rank}Q", b, p); p += 8 * rank
    return name, tuple(shape), n, n_c, p


def test_bitmask_oracle_matches_reference_bytes(bitmask_golden, golden_index):
    for case in golden_index["bitmask"]:
        i = case["i"]
        base, cur = bitmask_golden[f"c{i}_base"], bitmask_golden[f"c{i}_cur"]
        want = bitmask_golden[f"c{i}_bsdl"].tobytes()
        mask, payload, n_c = O.delta_encode(base, cur)
        got = O.delta_record(case["name"], case["shape"], base.size, n_c, mask, payload)
        assert got == want, case["name"]
        assert n_c == case["n_c"]
        dec = O.delta_decode(base, mask, payload, base.size, n_c)
        assert np.array_equal(dec, cur)
        assert O.delta_size(base.size, n_c) + len(case["name"].encode()) + \
            8 * (len(case["shape"]) - 1) == len(want)


def test_bitmask_byte_level_port_matches_reference(bitmask_golden, golden_index):
    """The bench's CPU arm (oracle.ref_encode_bytes / ref_decode_bytes, the
    reference's byte-level sequence) gives the reference's records."""
    for case in golden_index["bitmask"]:
        i = case["i"]
        base, cur = bitmask_golden[f"c{i}_base"], bitmask_golden[f"c{i}_cur"]
        bb = base.astype("<u2").tobytes()
        cb = cur.astype("<u2").tobytes()
        mask, payload, n_c = O.ref_encode_bytes(bb, cb)
        got = O.delta_record(case["name"], case["shape"], base.size, n_c,
                             np.frombuffer(mask, np.uint8), np.frombuffer(payload, "<u2"))
        assert got == bitmask_golden[f"c{i}_bsdl"].tobytes(), case["name"]
        assert O.ref_decode_bytes(bb, mask, payload, base.size, n_c) == cb


def test_bitmask_kat_0x42(bitmask_golden, golden_index):
    case = next(c for c in golden_index["bitmask"] if c["name"] == "kat_0x42")
    blob = bitmask_golden[f"c{case['i']}_bsdl"].tobytes()
    _, _, n, n_c, p = _bsdl_fields(blob)
    assert blob[p:p + 1] == b"\x42" and n_c == 2
    assert np.frombuffer(blob[p + 1:], "<u2").tolist() == [1000, 2000]


def test_bitmask_oracle_errors():
    base = np.arange(16, dtype=np.uint16)
    cur = base.copy(); cur[3] = 77
    mask, payload, n_c = O.delta_encode(base, cur)
    with pytest.raises(O.OracleDeltaError, match="popcount"):
        O.delta_decode(base, np.zeros_like(mask), payload, 16, n_c)
    m13 = np.zeros(2, np.uint8); m13[1] = 0x80
    with pytest.raises(O.OracleDeltaError, match="padding"):
        O.delta_decode(base[:13], m13, payload[:0], 13, 0)


def test_quant_oracle_matches_reference_bytes(quant_golden, golden_index):
    for case in golden_index["quant"]:
        i = case["i"]
        x = quant_golden[f"q{i}_x"]
        want = quant_golden[f"q{i}_bsqt"].tobytes()
        tab = O.cluster_fit(x, case["m"])
        packed, codes, _ = O.cluster_quantize(x, tab)
        got = O.quant_record(case["name"], (x.size,), tab, packed, codes)
        assert got == want, case["name"]
        assert len(got) == O.quant_record_size(case["name"], 1, x.size, case["m"])
        deq = O.cluster_dequantize(packed, codes, x.size, tab)
        assert np.array_equal(deq.view(np.uint32),
                              quant_golden[f"q{i}_deq"].view(np.uint32)), case["name"]


def test_pairwise_matches_numpy():
    rng = np.random.default_rng(5)
    for n in list(range(1, 140)) + [255, 256, 257, 1000, 4097, 8192, 8193, 65541]:
        a = (rng.standard_normal(n) * 1e-3).astype(np.float32).astype(np.float64)
        assert O.pairwise_sum(a) + 0.0 == float(np.sum(a)), n
        mu = (0.0 + O.pairwise_sum(a)) / n
        assert mu == float(np.mean(a))
        d = a - mu
        assert np.sqrt((0.0 + O.pairwise_sum(d * d)) / n) == float(np.std(a))


def test_ndtri_table_matches_scipy(golden_index):
    from paper_2511_12376_b200 import _ndtri
    for m in range(2, 17):
        z = O.ndtri_z(m)
        assert [float(v).hex() for v in z] == golden_index["ndtri"][str(m)]
        assert list(_ndtri.Z[m]) == [float(v) for v in z]


def test_checkpoint_oracle_matches_reference(checkpoint_golden, golden_index):
    meta = golden_index["checkpoint"]
    g = checkpoint_golden
    model0, model1, opt = [], [], []
    for name, shape in meta["shapes"].items():
        shape = tuple(shape)
        model0.append((name, shape, 0, g[f"w0:{name}"]))
        model1.append((name, shape, 0, g[f"w1:{name}"]))
    for name, shape in meta["shapes"].items():
        for kind in ("m", "v"):
            opt.append((f"adam.{kind}.{name}", tuple(shape), 1, g[f"{kind}:{name}"]))
    # the reference interleaves m and v per tensor (make_golden.make_checkpoint)
    e0, blob0 = O.encode_checkpoint(model0, opt, None, "base")
    e1, blob1 = O.encode_checkpoint(model1, opt, model0, "delta")
    assert hashlib.sha256(blob0).hexdigest() == meta["blob0_sha256"]
    assert hashlib.sha256(blob1).hexdigest() == meta["blob1_sha256"]
    man1 = json.loads(g["manifest1"].tobytes())
    assert [(t["name"], t["codec"], t["offset"], t["length"]) for t in man1["tensors"]] \
        == [(t["name"], t["codec"], t["offset"], t["length"]) for t in e1]
    assert any(t["codec"] == "RAW" for t in e1 if t["group"] == "model")


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"),
                    reason="live reference only in the build container")
def test_oracle_vs_live_reference_random():
    sys.path.insert(0, "/root/reference/pkg/src")
    from bitsnap import quantizer, tensors
    rng = np.random.default_rng(99)
    for _ in range(30):
        n = int(rng.integers(1, 20000))
        m = int(rng.integers(2, 17))
        x = (rng.standard_normal(n) * rng.uniform(1e-4, 10)).astype(np.float32)
        t = tensors.TensorBlob("x", tensors.ElementType.F32, (n,), x.tobytes())
        q = quantizer.quantize(t, quantizer.build_clusters(t, m))
        tab = O.cluster_fit(x, m)
        packed, codes, _ = O.cluster_quantize(x, tab)
        assert O.quant_record("x", (n,), tab, packed, codes) == \
            quantizer.serialize_quantized(q)


def _c0_records(names):
    """Worker: the oracle's encode_checkpoint records of some C0 tensors
    (model DELTA/RAW, then the two QUANT states) — concatenated in
    checkpoint order they are the whole blob (store.py:240-247 offsets are
    sequential)."""
    import bench_checkpoint as BC
    data = _C0["data"]
    out = {}
    for n in names:
        w0, w1, m, v = data[n]
        shp = w0.shape
        _, blob_w = O.encode_checkpoint([(n, shp, 0, w1)], [], [(n, shp, 0, w0)], "delta", 16)
        _, blob_o = O.encode_checkpoint([], [(BC.M_PREFIX + n, shp, 1, m),
                                             (BC.V_PREFIX + n, shp, 1, v)], None, "delta", 16)
        out[n] = (blob_w, blob_o)
    return out


_C0: dict = {}


def test_c0_published_blob():
    """BASELINE.md §2 / SURVEY §6: the reference's whole-checkpoint encode of
    the C0 pair (SURVEY §8(d) CPU-generator recipe) is 1,244,398,080 ->
    438,174,150 B.  The oracle reproduces that size and the reference's
    blob digest (tests/golden/c0_ratio.json, made by make_c0_ratio.py from
    the reference store); the GPU bench checks its blob against the same
    digest (bench.py run_c0)."""
    import multiprocessing as mp
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
    import bench_checkpoint as BC
    _C0["data"] = data = BC.generate_cpu_recipe_host("C0")
    names = list(data)
    ncpu = max(1, min(16, len(os.sched_getaffinity(0))))
    groups = [names[i::ncpu] for i in range(ncpu)]
    with mp.get_context("fork").Pool(ncpu) as p:
        parts = {}
        for d in p.map(_c0_records, groups):
            parts.update(d)
    blob = b"".join(parts[n][0] for n in names) + b"".join(parts[n][1] for n in names)
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c0_ratio.json")))
    raw = sum(w.nbytes + m.nbytes + v.nbytes for w, _, m, v in data.values())
    assert raw == 1_244_398_080 == ref["raw_bytes"]
    assert len(blob) == 438_174_150 == ref["delta_blob_bytes"]
    assert hashlib.sha256(blob).hexdigest() == ref["blob_sha256"]
