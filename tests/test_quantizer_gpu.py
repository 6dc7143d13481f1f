"""Parity of the sm_100a cluster quantizer against the oracle and the
reference's golden vectors.  Tables, labels and codes are compared bit for
bit (the north-star tolerance — <= 1e-4 label mismatches at ties, 1e-6
relative dequantization error — is not needed: the kernels reproduce numpy's
float64 arithmetic exactly).  Ports pkg/tests/test_quantizer.py and
test_acceptance.py::test_05..07."""

import math
import struct

import numpy as np
import pytest

from oracle import bitsnap_oracle as O

pytestmark = pytest.mark.gpu


def _f32(t_np, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(t_np, dtype=np.float32)).to(dev)


def _tables_equal(host_table, ora):
    f = lambda v: np.asarray(v, np.float32).view(np.uint32).tolist()
    assert host_table.m == ora["m"]
    assert f([host_table.mean, host_table.std]) == f([ora["mean"], ora["std"]])
    assert f(host_table.boundaries) == f(ora["boundaries"])
    assert f(host_table.scales) == f(ora["scales"])
    assert f(host_table.offsets) == f(ora["offsets"])


def _check_units(x, m, block, dq):
    """Every unit of a device encode equals the oracle on that slice."""
    n = x.size
    tabs = dq.host_tables()
    labels = dq.labels.cpu().numpy()
    codes = dq.codes.cpu().numpy()
    units = O.blockwise(x, block if block and block < n else 0)
    assert len(tabs) == len(units)
    lpos = 0
    for u, xs in enumerate(units):
        ora = O.cluster_fit(xs, m)
        _tables_equal(tabs[u], ora)
        packed, c, _ = O.cluster_quantize(xs, ora)
        start = u * (block if block and block < n else 0)
        assert np.array_equal(codes[start:start + xs.size], c), f"codes unit {u}"
        assert np.array_equal(labels[lpos:lpos + packed.size], packed), f"labels unit {u}"
        lpos += packed.size


def test_golden_records_byte_identical(dev, quant_golden, golden_index):
    from paper_2511_12376_b200 import quantizer as Q
    from paper_2511_12376_b200.tensors import ElementType, TensorBlob
    for case in golden_index["quant"]:
        i = case["i"]
        x = quant_golden[f"q{i}_x"]
        t = TensorBlob(case["name"], ElementType.F32, (x.size,), x.astype("<f4").tobytes())
        table = Q.build_clusters(t, case["m"])
        q = Q.quantize(t, table)
        assert Q.serialize_quantized(q) == quant_golden[f"q{i}_bsqt"].tobytes(), case["name"]
        deq = Q.dequantize(q)
        assert deq.data == quant_golden[f"q{i}_deq"].tobytes(), case["name"]
        assert Q.deserialize_quantized(Q.serialize_quantized(q)) == q


@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 127, 128, 129, 136, 1000, 8191, 8192, 8193,
                               16385, 100003, 1000003, (1 << 20) + 5])
@pytest.mark.parametrize("dist", ["unit", "adam_m", "adam_v"])
def test_per_tensor_vs_oracle(dev, n, dist):
    from paper_2511_12376_b200 import quantizer as Q
    rng = np.random.default_rng(n + len(dist))
    x = {"unit": lambda: rng.standard_normal(n),
         "adam_m": lambda: rng.standard_normal(n) * 1e-3,
         "adam_v": lambda: (rng.standard_normal(n) * 1e-3) ** 2}[dist]().astype(np.float32)
    m = int(rng.integers(2, 17)) if n % 2 else 16
    dq = Q.cluster_encode_device(_f32(x, dev), m, 0)
    _check_units(x, m, 0, dq)
    # dequantize: bit-exact against the oracle's float64 reconstruction
    out = Q.cluster_dequantize_device(dq).cpu().numpy()
    ora = O.cluster_fit(x, m)
    packed, codes, _ = O.cluster_quantize(x, ora)
    ref = O.cluster_dequantize(packed, codes, n, ora)
    assert np.array_equal(out.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("n,block", [(1 << 20, 1 << 17), ((1 << 20) + 24, 1 << 16),
                                     (300000, 4096), (50000, 8), (65536, 65536),
                                     (1000, 1 << 20)])
def test_per_block_vs_oracle(dev, n, block):
    from paper_2511_12376_b200 import quantizer as Q
    rng = np.random.default_rng(block)
    x = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    dq = Q.cluster_encode_device(_f32(x, dev), 16, block)
    _check_units(x, 16, block, dq)
    out = Q.cluster_dequantize_device(dq).cpu().numpy()
    for u, xs in enumerate(O.blockwise(x, block if block < n else 0)):
        ora = O.cluster_fit(xs, 16)
        p, c, _ = O.cluster_quantize(xs, ora)
        s = u * block
        assert np.array_equal(out[s:s + xs.size].view(np.uint32),
                              O.cluster_dequantize(p, c, xs.size, ora).view(np.uint32))


def test_fit_then_quantize_separately(dev):
    from paper_2511_12376_b200 import quantizer as Q
    x = (np.random.default_rng(4).standard_normal(70001) * 3 + 1).astype(np.float32)
    xt = _f32(x, dev)
    tables = Q.cluster_fit_device(xt, 11, 8192)
    labels, codes = Q.cluster_quantize_device(xt, tables, 8192)
    dq = Q.DeviceQuant(tables, labels, codes, x.size, 8192, 11)
    _check_units(x, 11, 8192, dq)


def test_constant_and_degenerate(dev):
    """test_quantizer.py:65-74, 165-168: constant tensors round-trip exactly."""
    from paper_2511_12376_b200 import quantizer as Q
    from paper_2511_12376_b200.tensors import ElementType, TensorBlob
    for val, n, m in ((3.25, 100, 8), (-7.5, 33, 16), (0.0, 5000, 16)):
        t = TensorBlob("t", ElementType.F32, (n,), np.full(n, val, "<f4").tobytes())
        table = Q.build_clusters(t, m)
        assert all(b == pytest.approx(val) for b in table.boundaries)
        q = Q.quantize(t, table)
        assert set(Q.unpack_labels(q.packed_labels, n).tolist()) == {0}
        assert set(q.codes) == {0}
        assert Q.dequantize(q).data == t.data


def test_validation_errors(dev):
    from paper_2511_12376_b200 import quantizer as Q
    from paper_2511_12376_b200.tensors import ElementType, TensorBlob
    t = TensorBlob("t", ElementType.F32, (10,), np.ones(10, "<f4").tobytes())
    for m in (0, 1, 17):
        with pytest.raises(Q.QuantizerError, match="outside"):
            Q.build_clusters(t, m)
    with pytest.raises(Q.QuantizerError, match="empty"):
        Q.build_clusters(TensorBlob("e", ElementType.F32, (0,), b""), 4)
    with pytest.raises(Q.QuantizerError, match="not F32"):
        Q.build_clusters(TensorBlob("h", ElementType.F16, (4,), b"\0" * 8), 4)
    bad = np.ones(10, "<f4"); bad[3] = np.nan
    with pytest.raises(Q.QuantizerError, match="non-finite"):
        Q.build_clusters(TensorBlob("n", ElementType.F32, (10,), bad.tobytes()), 4)
    # label overflow on dequantize (test_quantizer.py:171-180)
    x = TensorBlob("t", ElementType.F32, (8,),
                   np.random.default_rng(1).standard_normal(8).astype("<f4").tobytes())
    q = Q.quantize(x, Q.build_clusters(x, 2))
    broken = Q.QuantizedTensor(q.name, q.shape, q.table,
                               Q.pack_labels(np.full(8, 9, np.uint8)), q.codes)
    with pytest.raises(Q.QuantizerError, match="label 9 >= m=2"):
        Q.dequantize(broken)


def test_exhaustive_argmin_oracle_1e6(dev):
    """test_acceptance.py:116-138: codes == 256-way argmin (first index on ties)."""
    from paper_2511_12376_b200 import quantizer as Q
    x = np.random.default_rng(3).standard_normal(1_000_000).astype(np.float32)
    dq = Q.cluster_encode_device(_f32(x, dev), 16, 0)
    tab = dq.host_tables()[0]
    codes = dq.codes.cpu().numpy()
    labels = Q.unpack_labels(dq.labels.cpu().numpy().tobytes(), x.size)
    s = np.asarray(tab.scales)[labels]
    b = np.asarray(tab.offsets)[labels]
    v = x.astype(np.float64)
    xn = np.clip(np.where(s > 0, (v - b) / np.where(s > 0, s, 1.0), 0.0), 0.0, 1.0)
    grid = Q.qmap(np.arange(256))
    for lo in range(0, x.size, 1 << 16):
        want = np.abs(grid[None, :] - xn[lo:lo + (1 << 16), None]).argmin(axis=1)
        assert np.array_equal(codes[lo:lo + (1 << 16)], want)


def test_error_bound_and_mse(dev):
    """test_acceptance.py:154-175 and test_quantizer.py:151-162."""
    from paper_2511_12376_b200 import quantizer as Q
    rng = np.random.default_rng(5)
    for _ in range(40):
        n = int(rng.integers(64, 5000))
        x = (rng.standard_normal(n) * rng.uniform(1e-3, 100.0)).astype(np.float32)
        dq = Q.cluster_encode_device(_f32(x, dev), 16, 0)
        r = Q.cluster_dequantize_device(dq).cpu().numpy().astype(np.float64)
        tab = dq.host_tables()[0]
        lab = Q.unpack_labels(dq.labels.cpu().numpy().tobytes(), n)
        s = np.asarray(tab.scales)[lab]
        ulp = np.spacing(np.abs(x)).astype(np.float64)
        assert np.all(np.abs(r - x) <= s / 510 + ulp)
    x = np.random.default_rng(6).standard_normal(1_000_000).astype(np.float32)
    dq = Q.cluster_encode_device(_f32(x, dev), 16, 0)
    r = Q.cluster_dequantize_device(dq).cpu().numpy().astype(np.float64)
    assert float(np.mean((x - r) ** 2)) <= 1e-5


def test_tie_values_take_smaller_code(dev):
    """Values engineered onto exact half-steps of a [0, 1] cluster: the code
    must be the smaller neighbour (ceil(x*255 - 0.5), quantizer.py:180-181)."""
    from paper_2511_12376_b200 import quantizer as Q
    from paper_2511_12376_b200.tensors import ElementType, TensorBlob
    j = np.arange(255)
    ties = ((j + 0.5) / 255.0).astype(np.float32)
    x = np.concatenate([[0.0, 1.0], ties, np.nextafter(ties, 2), np.nextafter(ties, -2)])
    x = x.astype(np.float32)
    t = TensorBlob("t", ElementType.F32, (x.size,), x.tobytes())
    table = Q.ClusterTable(m=2, mean=0.5, std=1.0, boundaries=(2.0,), scales=(1.0, 0.0),
                           offsets=(0.0, 0.0))
    q = Q.quantize(t, table)
    tab = {"m": 2, "boundaries": [2.0], "scales": [1.0, 0.0], "offsets": [0.0, 0.0]}
    _, codes, _ = O.cluster_quantize(x, tab)
    assert q.codes == codes.tobytes()


def test_precision_report(dev):
    from paper_2511_12376_b200 import quantizer as Q
    from paper_2511_12376_b200.tensors import ElementType, TensorBlob
    f = lambda a: TensorBlob("t", ElementType.F32, (len(a),), np.asarray(a, "<f4").tobytes())
    rep = Q.precision_report(f([1.0, -2.0, 4.0, 0.0]), f([1.1, -2.2, 3.6, 0.5]))
    want = O.precision(np.array([1.0, -2.0, 4.0, 0.0], np.float32),
                       np.array([1.1, -2.2, 3.6, 0.5], np.float32))
    assert rep["mse"] == pytest.approx(want["mse"], rel=1e-12)
    assert rep["mre"] == pytest.approx(want["mre"], rel=1e-12)
    x = np.random.default_rng(8).standard_normal(100_000).astype(np.float32)
    y = (x.astype(np.float64) + 1e-7).astype(np.float32)
    rep = Q.precision_report(f(x), f(y))
    want = O.precision(x, y)
    assert rep["mse"] == pytest.approx(want["mse"], rel=1e-9)
    assert rep["mre"] == pytest.approx(want["mre"], rel=1e-9)


def test_size_laws_and_serialization(dev):
    from paper_2511_12376_b200 import quantizer as Q
    from paper_2511_12376_b200.tensors import ElementType, TensorBlob
    assert Q.quantized_size_bytes(1_000_000, 16) == 1_500_136
    rng = np.random.default_rng(9)
    for n in (1, 2, 101, 5000):
        x = rng.standard_normal(n).astype("<f4")
        t = TensorBlob("moments", ElementType.F32, (n,), x.tobytes())
        b = Q.serialize_quantized(Q.quantize(t, Q.build_clusters(t, 16)))
        assert len(b) == Q.serialized_quant_size("moments", 1, n, 16)


@pytest.mark.slow
@pytest.mark.parametrize("dist", ["adam_m", "adam_v"])
def test_c2_shape_per_block_sampled(dev, dist):
    """2^26-element tensor, block 2^20: sampled blocks bit-exact vs the oracle,
    every block's table well-formed, round trip within the error bound."""
    import torch
    from paper_2511_12376_b200 import quantizer as Q
    n, block = 1 << 26, 1 << 20
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.randn(n, device=dev, generator=g) * 1e-3
    if dist == "adam_v":
        x = x * x
    dq = Q.cluster_encode_device(x, 16, block)
    tabs = dq.host_tables()
    assert len(tabs) == 64
    xh = x.cpu().numpy()
    codes = dq.codes.cpu().numpy()
    labels = dq.labels.cpu().numpy()
    for u in (0, 17, 63):
        xs = xh[u * block:(u + 1) * block]
        ora = O.cluster_fit(xs, 16)
        _tables_equal(tabs[u], ora)
        p, c, _ = O.cluster_quantize(xs, ora)
        assert np.array_equal(codes[u * block:(u + 1) * block], c)
        assert np.array_equal(labels[u * block // 2:(u + 1) * block // 2], p)
    out = Q.cluster_dequantize_device(dq)
    err = (out - x).abs()
    scale = torch.tensor([max(t.scales) for t in tabs], device=dev).repeat_interleave(block)
    assert bool((err <= scale / 510 + x.abs() * 1.2e-7).all())


def _dist(name, n, rng):
    if name == "adam_m":
        return rng.standard_normal(n) * 1e-3
    if name == "adam_v":
        return (rng.standard_normal(n) * 1e-3) ** 2
    if name == "discrete":      # few distinct values: threshold bins are empty
        return rng.integers(-3, 4, n) * 0.25
    if name == "sparse":        # mostly zeros, a few large spikes
        x = np.zeros(n)
        k = max(1, n // 1000)
        x[rng.choice(n, k, replace=False)] = rng.standard_normal(k) * 50
        return x
    if name == "offset":        # large mean, tiny spread (cancellation)
        return 3.0 + rng.standard_normal(n) * 1e-5
    if name == "uniform":
        return rng.uniform(-1, 1, n)
    raise ValueError(name)


_DISTS = ["adam_m", "adam_v", "discrete", "sparse", "offset", "uniform"]


def _cases(shapes, keep):
    """shape x distribution x m, minus the large combinations the CPU
    oracle's time budget leaves out (`keep` says which large ones stay)."""
    return [(lb, u, t, d, m) for lb, u, t in shapes for d in _DISTS for m in (16, 7, 2)
            if keep(lb, d, m)]


@pytest.mark.parametrize("log2b,units,tail,dist,m", _cases(
    [(13, 5, 0), (16, 3, 1000), (20, 2, 8), (21, 1, 0)],
    lambda lb, d, m: not ((lb >= 20 and m != 16) or (lb == 21 and d not in ("adam_m",
                                                                            "discrete")))))
def test_power_of_two_blocks_vs_oracle(dev, log2b, units, tail, dist, m):
    """Power-of-two blocks of 2^13..2^21 (perfect tree tiles) plus a ragged
    tail unit; sparse/discrete data force the exact min/max round.  Every
    unit is bit-exact vs the oracle, and the fit-only path gives the same
    tables."""
    from paper_2511_12376_b200 import quantizer as Q
    block = 1 << log2b
    n = units * block + tail
    rng = np.random.default_rng(log2b * 100 + m)
    x = _dist(dist, n, rng).astype(np.float32)
    if dist == "offset" and units > 1:
        x[block:2 * block] = 1.5          # a constant block (sd = 0)
    dq = Q.cluster_encode_device(_f32(x, dev), m, block)
    _check_units(x, m, block, dq)
    tables = Q.cluster_fit_device(_f32(x, dev), m, block)   # fit-only path
    assert bytes(tables.cpu().numpy()) == bytes(dq.tables.cpu().numpy())


def test_repeatable_and_nonfinite(dev):
    import torch
    from paper_2511_12376_b200 import quantizer as Q
    n, block = 1 << 22, 1 << 18
    g = torch.Generator(device=dev).manual_seed(9)
    x = torch.randn(n, device=dev, generator=g) * 1e-3
    a = Q.cluster_encode_device(x, 16, block)
    for _ in range(3):
        b = Q.cluster_encode_device(x, 16, block)
        assert torch.equal(a.codes, b.codes) and torch.equal(a.labels, b.labels)
        assert torch.equal(a.tables, b.tables)
    x[block * 3 + 5] = float("nan")
    with pytest.raises(Q.QuantizerError, match="non-finite"):
        Q.cluster_encode_device(x, 16, block)


@pytest.mark.parametrize("log2b,units,tail,dist,m", _cases(
    [(13, 9, 0), (13, 8, 100), (16, 8, 1000), (17, 10, 8), (20, 8, 0)],
    lambda lb, d, m: not (lb == 20 and (m != 16 or d not in ("adam_m", "discrete")))))
def test_many_units_vs_oracle(dev, log2b, units, tail, dist, m):
    """Encodes of 8-10 units plus a ragged tail: one-sided data (adam_v: the
    lower fit thresholds lie below every element, so those clusters are
    empty and decided from the unit extremes), constant blocks (decided
    directly), discrete / sparse data (the exact min/max round).  Bit-exact
    vs the oracle."""
    from paper_2511_12376_b200 import quantizer as Q
    block = 1 << log2b
    n = units * block + tail
    rng = np.random.default_rng(log2b * 1000 + m + units)
    x = _dist(dist, n, rng).astype(np.float32)
    if dist == "offset":
        x[2 * block:3 * block] = -0.75    # a constant block (sd = 0)
    dq = Q.cluster_encode_device(_f32(x, dev), m, block)
    _check_units(x, m, block, dq)


@pytest.mark.parametrize("n,block", [((1 << 24) + 12345, 0), (2 * (1 << 23) + 5000, 1 << 23)])
def test_large_units_pre_reduced_combine(dev, n, block):
    """Units of more than 1024 tree tiles (2^23+ elements) fold their tile
    partials in groups of 1024 before the per-unit combine (the same perfect
    tree); a ragged last unit of few tiles takes the direct combine.  Tables,
    labels and codes bit-exact vs the oracle."""
    from paper_2511_12376_b200 import quantizer as Q
    rng = np.random.default_rng(n)
    x = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    dq = Q.cluster_encode_device(_f32(x, dev), 16, block)
    _check_units(x, 16, block, dq)


@pytest.mark.parametrize("n,block,dist,m", [
    ((1 << 20) + 5, 0, "adam_m", 16), (100003, 8192, "adam_v", 7), (5 * 8192 + 100, 8192,
                                                                     "offset", 16),
    (3 * (1 << 16) + 1000, 1 << 16, "uniform", 2), ((1 << 24) + 12345, 0, "adam_v", 16),
    (9 * 8192, 8192, "discrete", 16)])
def test_exact_variance_fallback_vs_oracle(dev, monkeypatch, n, block, dist, m):
    """The default fit reads x once: sigma comes from a rigorous interval
    around numpy's variance (quant_stats.cuh), and only units whose f32
    outputs the interval leaves undecided take numpy's variance tree.
    BSNP_VAR_EXACT=1 sends every unit down that fallback: both paths must be
    bit-exact vs the oracle and give identical bytes."""
    from paper_2511_12376_b200 import quantizer as Q
    rng = np.random.default_rng(n + m)
    x = _dist(dist, n, rng).astype(np.float32)
    xt = _f32(x, dev)
    a = Q.cluster_encode_device(xt, m, block)
    monkeypatch.setenv("BSNP_VAR_EXACT", "1")
    b = Q.cluster_encode_device(xt, m, block)
    _check_units(x, m, block, b)
    for f in ("tables", "labels", "codes"):
        assert bytes(getattr(a, f).cpu().numpy()) == bytes(getattr(b, f).cpu().numpy()), f


def test_precision_report_deterministic(dev):
    """The float64 reduction has a fixed order (no atomics): the same bits on
    every run (quantizer.py:280-296 semantics, rel 1e-9 of numpy's order)."""
    import torch
    from paper_2511_12376_b200.metrics import precision_device
    g = torch.Generator(device=dev).manual_seed(4)
    x = torch.randn((1 << 24) + 77, device=dev, generator=g)
    y = x + torch.randn(x.numel(), device=dev, generator=g) * 1e-4
    x[::1000] = 0.0
    reps = [precision_device(x, y) for _ in range(5)]
    assert all(r == reps[0] for r in reps)
    want = O.precision(x.cpu().numpy(), y.cpu().numpy())
    assert reps[0]["mse"] == pytest.approx(want["mse"], rel=1e-9)
    assert reps[0]["mre"] == pytest.approx(want["mre"], rel=1e-9)


@pytest.mark.parametrize("n,block,dist,m", [
    ((1 << 20) + 5, 0, "adam_m", 16), (100003, 8192, "adam_v", 7),
    (3 * (1 << 16) + 1000, 1 << 16, "uniform", 2), (9 * 8192, 8192, "discrete", 16),
    (5000, 0, "adam_v", 16)])
def test_four_pass_path_matches_window_path(dev, monkeypatch, n, block, dist, m):
    """BSNP_WINDOW=0 runs the four-pass kernels (numpy's mean tree, variance
    tree, per-element min/max with fit labels, then quantize): a second exact
    implementation of quantizer.py:100-189.  Both are bit-exact vs the
    oracle and give identical bytes."""
    from paper_2511_12376_b200 import quantizer as Q
    rng = np.random.default_rng(n * 3 + m)
    x = _dist(dist, n, rng).astype(np.float32)
    xt = _f32(x, dev)
    a = Q.cluster_encode_device(xt, m, block)
    monkeypatch.setenv("BSNP_WINDOW", "0")
    b = Q.cluster_encode_device(xt, m, block)
    _check_units(x, m, block, b)
    for f in ("tables", "labels", "codes"):
        assert bytes(getattr(a, f).cpu().numpy()) == bytes(getattr(b, f).cpu().numpy()), f


@pytest.mark.parametrize("n,block,dist,m,env", [
    (15 * 32768 + 32749, 32768, "offset_big", 5, None),         # the stress-test case
    (2 * (1 << 20) + (1 << 20) - 7, 1 << 20, "adam_m", 16, "BSNP_VAR_EXACT"),
    (2 * (1 << 20) + (1 << 20) - 9, 1 << 20, "adam_v", 16, "BSNP_WINDOW"),
    ((1 << 23) + (1 << 23) - 19, 1 << 23, "adam_m", 16, None),  # last unit > kPreGroup tiles
    ((1 << 23) + (1 << 23) - 19, 1 << 23, "offset", 16, "BSNP_VAR_EXACT"),
])
def test_last_unit_deeper_than_full_units(dev, monkeypatch, n, block, dist, m, env):
    """numpy's split of a slightly shorter last unit can leave a piece above
    one tree tile and so need one more level: the last unit then has MORE
    tiles than a full unit (e.g. 32749 elements: 8 tiles vs 4 for 32768).
    The variance fallback, the pre-reduction of > 1024-tile units and the
    four-pass path enumerate T_max tile slots per unit; every unit equals
    the oracle (regression: the stress run's 'offset' case, whose units all
    take the exact variance tree, had a wrong sigma in its last unit)."""
    from paper_2511_12376_b200 import quantizer as Q
    if env == "BSNP_VAR_EXACT":
        monkeypatch.setenv("BSNP_VAR_EXACT", "1")
    elif env == "BSNP_WINDOW":
        monkeypatch.setenv("BSNP_WINDOW", "0")
    rng = np.random.default_rng(n % 100003)
    if dist == "offset_big":    # |mean| / sd ~ 1e7: sigma's interval is too wide, exact tree
        x = (1e4 + rng.standard_normal(n) * 1e-3).astype(np.float32)
    else:
        x = _dist(dist, n, rng).astype(np.float32)
    dq = Q.cluster_encode_device(_f32(x, dev), m, block)
    _check_units(x, m, block, dq)


def test_concurrent_quantizer_callers_from_threads(dev):
    """build_clusters / quantize / dequantize from three host threads at once
    (per-thread workspaces): each thread's records equal the oracle's."""
    import threading
    from paper_2511_12376_b200 import quantizer as Q
    from paper_2511_12376_b200.tensors import ElementType, TensorBlob
    errors = []

    def work(seed):
        try:
            rng = np.random.default_rng(seed)
            for _ in range(4):
                n = int(rng.integers(1, 200_000))
                m = int(rng.integers(2, 17))
                x = (rng.standard_normal(n) * 1e-3).astype(np.float32)
                t = TensorBlob("t", ElementType.F32, (n,), x.tobytes())
                table = Q.build_clusters(t, m)
                ora = O.cluster_fit(x, m)
                _tables_equal(table, ora)
                q = Q.quantize(t, table)
                packed, codes, _ = O.cluster_quantize(x, ora)
                assert q.codes == codes.tobytes() and q.packed_labels == packed.tobytes()
                assert Q.dequantize(q).data == O.cluster_dequantize(packed, codes, n, ora).tobytes()
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=work, args=(s,)) for s in range(3)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
