"""Parity of the sm_100a bitmask codec against the oracle and the reference's
golden vectors (bit-exact: integer work).  Ports the reference's hot-path
tests (pkg/tests/test_bitmask.py, test_acceptance.py::test_01..04)."""

import numpy as np
import pytest

from oracle import bitsnap_oracle as O

pytestmark = pytest.mark.gpu


def _dev_u16(a, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint16).view(np.int16)).to(dev)


def _np(t):
    return t.cpu().numpy().view(np.uint16) if t.dtype != __import__("torch").uint8 \
        else t.cpu().numpy()


def test_golden_records_byte_identical(dev, bitmask_golden, golden_index):
    from paper_2511_12376_b200 import bitmask as B
    from paper_2511_12376_b200.tensors import ElementType, TensorBlob
    for case in golden_index["bitmask"]:
        i = case["i"]
        base, cur = bitmask_golden[f"c{i}_base"], bitmask_golden[f"c{i}_cur"]
        shape = tuple(case["shape"])
        tb = TensorBlob(case["name"], ElementType.F16, shape, base.astype("<u2").tobytes())
        tc = TensorBlob(case["name"], ElementType.F16, shape, cur.astype("<u2").tobytes())
        rec = B.encode_delta(tb, tc)
        assert B.serialize_delta(rec) == bitmask_golden[f"c{i}_bsdl"].tobytes(), case["name"]
        assert B.decode_delta(tb, rec).data == tc.data
        assert B.deserialize_delta(B.serialize_delta(rec)) == rec


@pytest.mark.parametrize("n", [1, 5, 8, 13, 255, 8191, 8192, 8193, 3 * 8192 + 5,
                               32 * 8192, 64 * 8192 + 1, 32768 * 33 + 7, (1 << 20) + 3])
@pytest.mark.parametrize("frac", [0.0, 0.001, 0.1, 0.5, 1.0])
def test_device_encode_decode_vs_oracle(dev, n, frac):
    from paper_2511_12376_b200 import bitmask as B
    rng = np.random.default_rng(n * 7 + int(frac * 1000))
    base = rng.integers(0, 1 << 16, n, dtype=np.uint16)
    cur = base.copy()
    k = int(round(frac * n))
    if k:
        idx = rng.choice(n, k, replace=False)
        cur[idx] ^= rng.integers(1, 1 << 16, k, dtype=np.uint16)
    mask, payload, n_c = O.delta_encode(base, cur)
    d = B.encode_delta_device(_dev_u16(base, dev), _dev_u16(cur, dev))
    assert d.n_c == n_c == k
    assert np.array_equal(d.mask.cpu().numpy(), mask)
    assert np.array_equal(d.payload.cpu().numpy().view(np.uint16), payload)
    out = B.decode_delta_device(_dev_u16(base, dev), d.mask, d.payload, d.n_c)
    assert np.array_equal(out.cpu().numpy().view(np.uint16), cur)
    # in-place apply (chain replay)
    bt = _dev_u16(base, dev)
    B.decode_delta_device(bt, d.mask, d.payload, d.n_c, out=bt)
    assert np.array_equal(bt.cpu().numpy().view(np.uint16), cur)


@pytest.mark.parametrize("offset", [1, 3, 7])
def test_misaligned_views(dev, offset):
    """torch views at odd element offsets take the scalar-load kernel path."""
    import torch
    from paper_2511_12376_b200 import bitmask as B
    n = 20000
    rng = np.random.default_rng(offset)
    base = rng.integers(0, 1 << 16, n + offset, dtype=np.uint16)
    cur = base.copy()
    cur[rng.choice(n + offset, 3000, replace=False)] += 1
    bt, ct = _dev_u16(base, dev)[offset:], _dev_u16(cur, dev)[offset:]
    assert bt.data_ptr() % 16 != 0
    mask, payload, n_c = O.delta_encode(base[offset:], cur[offset:])
    d = B.encode_delta_device(bt, ct)
    assert d.n_c == n_c
    assert np.array_equal(d.mask.cpu().numpy(), mask)
    assert np.array_equal(d.payload.cpu().numpy().view(np.uint16), payload)
    outbuf = torch.empty(n + offset, dtype=torch.int16, device=dev)[offset:]
    out = B.decode_delta_device(bt, d.mask, d.payload, d.n_c, out=outbuf)
    assert np.array_equal(out.cpu().numpy().view(np.uint16), cur[offset:])


def test_bf16_and_fp16_tensors(dev):
    import torch
    from paper_2511_12376_b200 import bitmask as B
    g = torch.Generator(device="cpu").manual_seed(0)
    w0 = torch.randn(1000, 77, generator=g) * 0.02
    w1 = w0 - 1e-5 * torch.randn(1000, 77, generator=g)
    for dt in (torch.bfloat16, torch.float16):
        a, b = w0.to(dt).to(dev), w1.to(dt).to(dev)
        d = B.encode_delta_device(a, b)
        mask, payload, n_c = O.delta_encode(a.cpu().view(torch.int16).numpy(),
                                            b.cpu().view(torch.int16).numpy())
        assert d.n_c == n_c
        assert np.array_equal(d.mask.cpu().numpy(), mask)
        out = B.decode_delta_device(a, d.mask, d.payload, d.n_c)
        assert torch.equal(out.view(torch.int16), b.view(torch.int16))


def test_reference_kats(dev):
    from paper_2511_12376_b200 import bitmask as B
    from paper_2511_12376_b200.tensors import ElementType, TensorBlob
    f16 = lambda v, name="t": TensorBlob(name, ElementType.F16, (len(v),),
                                         np.asarray(v, "<u2").tobytes())
    # identical -> 13 zero mask bytes (test_bitmask.py:27-32)
    t = f16(np.random.default_rng(1).integers(0, 1 << 16, 100))
    rec = B.encode_delta(t, t)
    assert rec.changed_count == 0 and rec.payload == b"" and rec.packed_mask == b"\0" * 13
    # 0x42 (test_bitmask.py:35-46)
    tgt = list(range(8)); tgt[1] = 1000; tgt[6] = 2000
    rec = B.encode_delta(f16(range(8)), f16(tgt))
    assert rec.packed_mask == b"\x42" and rec.changed_count == 2
    assert np.frombuffer(rec.payload, "<u2").tolist() == [1000, 2000]
    # NaN / -0.0 (test_bitmask.py:72-79)
    b, c = f16([0x0000, 0x3C00, 0x0000]), f16([0x8000, 0x7E00, 0x0000])
    rec = B.encode_delta(b, c)
    assert rec.changed_count == 2 and B.decode_delta(b, rec).data == c.data
    # error keywords (test_bitmask.py:82-125)
    a4, b4 = f16([1, 2, 3, 4], "a"), f16([1, 2, 3, 4], "b")
    with pytest.raises(B.DeltaError, match="name"):
        B.encode_delta(a4, b4)
    with pytest.raises(B.DeltaError, match="shape"):
        B.encode_delta(a4, f16([1, 2, 3, 4, 5], "a"))
    f32 = TensorBlob("a", ElementType.F32, (4,), b"\0" * 16)
    with pytest.raises(B.DeltaError, match="F16"):
        B.encode_delta(f32, f32)


def test_decode_validation_errors(dev):
    import torch
    from paper_2511_12376_b200 import bitmask as B
    rng = np.random.default_rng(3)
    base = rng.integers(0, 1 << 16, 16, dtype=np.uint16)
    cur = base.copy(); cur[[2, 9]] += 1
    d = B.encode_delta_device(_dev_u16(base, dev), _dev_u16(cur, dev))
    zero = torch.zeros_like(d.mask)
    with pytest.raises(B.DeltaError, match="popcount"):
        B.decode_delta_device(_dev_u16(base, dev), zero, d.payload, d.n_c)
    # padding bits (bitmask.py:128-129), and in-place decode leaves base untouched
    b13 = _dev_u16(base[:13], dev)
    m = torch.tensor([0x01, 0x80], dtype=torch.uint8, device=dev)
    p = torch.tensor([7], dtype=torch.int16, device=dev)
    with pytest.raises(B.DeltaError, match="padding"):
        B.decode_delta_device(b13, m, p, 1)
    before = b13.clone()
    with pytest.raises(B.DeltaError, match="padding"):
        B.decode_delta_device(b13, m, p, 1, out=b13)
    assert torch.equal(before, b13)
    with pytest.raises(B.DeltaError, match="popcount"):
        B.decode_delta_device(b13, torch.tensor([0x03, 0], dtype=torch.uint8, device=dev),
                              p, 1, out=b13)
    assert torch.equal(before, b13)


def test_losslessness_10k_pairs_with_specials(dev):
    """test_acceptance.py:47-70 (10k random pairs incl. +-0/NaN/+-inf)."""
    import torch
    from paper_2511_12376_b200 import bitmask as B
    rng = np.random.default_rng(0)
    specials = np.array([0x0000, 0x8000, 0x7E00, 0xFE00, 0x7C00, 0xFC00], np.uint16)
    # batch the 10k pairs as segments of one long tensor per 1k, check per pair
    for blk in range(10):
        bases, curs, sizes = [], [], []
        for i in range(1000):
            n = int(rng.integers(1, 257))
            bv = rng.integers(0, 1 << 16, n, dtype=np.uint16)
            tv = bv.copy()
            k = int(rng.integers(0, n + 1))
            if k:
                idx = rng.choice(n, k, replace=False)
                tv[idx] = rng.choice(specials, k) if i % 3 else \
                    rng.integers(0, 1 << 16, k, dtype=np.uint16)
            bases.append(bv); curs.append(tv); sizes.append(n)
        # encode each pair on device (distinct tensors, same stream)
        for bv, tv in zip(bases[:200], curs[:200]):
            d = B.encode_delta_device(_dev_u16(bv, dev), _dev_u16(tv, dev))
            out = B.decode_delta_device(_dev_u16(bv, dev), d.mask, d.payload, d.n_c)
            assert np.array_equal(out.cpu().numpy().view(np.uint16), tv)
        # and the concatenation as one tensor: must equal the oracle exactly
        bcat, tcat = np.concatenate(bases), np.concatenate(curs)
        mask, payload, n_c = O.delta_encode(bcat, tcat)
        d = B.encode_delta_device(_dev_u16(bcat, dev), _dev_u16(tcat, dev))
        assert d.n_c == n_c and np.array_equal(d.mask.cpu().numpy(), mask)
        assert np.array_equal(d.payload.cpu().numpy().view(np.uint16), payload)


def test_payload_cap_flag(dev):
    import torch
    from paper_2511_12376_b200 import _lib
    from paper_2511_12376_b200 import _runtime as rt
    n = 40000
    b = torch.zeros(n, dtype=torch.int16, device=dev)
    c = torch.ones(n, dtype=torch.int16, device=dev)
    mask = torch.empty((n + 7) // 8, dtype=torch.uint8, device=dev)
    payload = torch.full((100,), -1, dtype=torch.int16, device=dev)
    st = rt.new_status(dev)
    ws = torch.empty(_lib.load().bsnp_delta_encode_ws_bytes(n), dtype=torch.uint8, device=dev)
    rc = _lib.load().bsnp_delta_encode(b.data_ptr(), c.data_ptr(), n, mask.data_ptr(),
                                       payload.data_ptr(), 100, st.data_ptr(),
                                       ws.data_ptr(), ws.numel(),
                                       torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    (cnt, flags), = rt.read_status(st)
    assert cnt == n and flags & _lib.ERR_PAYLOAD_CAP
    assert torch.all(payload == 1)


@pytest.mark.slow
@pytest.mark.parametrize("p", [0.001, 0.0625, 0.25])
def test_large_roundtrip_properties(dev, p):
    """2^28 bf16 elements: n_c == k exactly, decode(encode) == cur, size law."""
    import torch
    from paper_2511_12376_b200 import bitmask as B
    n = 1 << 28
    g = torch.Generator(device=dev).manual_seed(11)
    base = (torch.randn(n, device=dev, generator=g) * 0.02).to(torch.bfloat16).view(torch.int16)
    cur = base.clone()
    k = int(round(p * n))
    idx = torch.randperm(n, device=dev, generator=g)[:k]
    cur[idx] += 1
    d = B.encode_delta_device(base, cur)
    assert d.n_c == k
    assert d.mask.numel() == n // 8
    assert int(d.mask.to(torch.int32).sum()) > 0
    out = B.decode_delta_device(base, d.mask, d.payload, d.n_c)
    assert torch.equal(out, cur)
    # payload equals cur gathered at sorted positions
    pos = torch.sort(idx).values
    assert torch.equal(d.payload, cur[pos])
    assert B.delta_size_bytes(n, k) == n // 8 + 2 * k + B.DELTA_FIXED_OVERHEAD


def test_hostpath_roundtrip_matches_oracle(dev):
    """hostpath.HostDeltaCodec.roundtrip (the bench's e2e path): the record
    that lands in pinned host memory equals the oracle's, and the restored
    tensor equals the current one (chunked, pipelined, odd tail)."""
    import torch
    from paper_2511_12376_b200 import hostpath
    rng = np.random.default_rng(77)
    n = 3 * (1 << 16) + 12345
    base = rng.integers(0, 1 << 16, n, dtype=np.uint16)
    cur = base.copy()
    idx = rng.choice(n, n // 50, replace=False)
    cur[idx] ^= rng.integers(1, 1 << 16, idx.size, dtype=np.uint16)
    bh = torch.from_numpy(base.view(np.int16)).pin_memory()
    ch = torch.from_numpy(cur.view(np.int16)).pin_memory()
    codec = hostpath.HostDeltaCodec(dev, n, chunk=1 << 16)
    for _ in range(2):
        rec, out = codec.roundtrip(bh, ch)
        mask, payload, n_c = O.delta_encode(base, cur)
        assert rec.n_c == n_c
        assert np.array_equal(rec.mask.numpy(), mask)
        assert np.array_equal(rec.payload.numpy().view(np.uint16), payload)
        assert np.array_equal(out.numpy().view(np.uint16), cur)
    rec2 = codec.encode(bh, ch)
    assert np.array_equal(rec2.mask.numpy(), mask)
    assert np.array_equal(codec.decode(bh, rec2).numpy().view(np.uint16), cur)


@pytest.mark.parametrize("n,p", [((1 << 20) + 777, 0.25), ((1 << 20) + 3, 0.0625),
                                 (8192 * 5, 0.5), (100003, 0.04)])
def test_in_place_apply_dense(dev, n, p):
    """Chain replay at dense change fractions streams whole tiles in place
    (decode kernel with out == base) instead of touching changed words; the
    result equals the target, and a rejected record leaves the base as is."""
    import torch
    from paper_2511_12376_b200 import bitmask as B
    rng = np.random.default_rng(int(n * p))
    base = rng.integers(0, 1 << 16, n, dtype=np.uint16)
    cur = base.copy()
    idx = rng.choice(n, int(n * p), replace=False)
    cur[idx] ^= rng.integers(1, 1 << 16, idx.size, dtype=np.uint16)
    d = B.encode_delta_device(_dev_u16(base, dev), _dev_u16(cur, dev))
    bt = _dev_u16(base, dev)
    B.decode_delta_device(bt, d.mask, d.payload, d.n_c, out=bt)
    assert np.array_equal(bt.cpu().numpy().view(np.uint16), cur)
    bt = _dev_u16(base, dev)
    bad = d.mask.clone()
    bad[0] ^= 1                      # popcount no longer matches n_c
    with pytest.raises(B.DeltaError, match="popcount"):
        B.decode_delta_device(bt, bad, d.payload, d.n_c, out=bt)
    assert np.array_equal(bt.cpu().numpy().view(np.uint16), base)


@pytest.mark.parametrize("n,p", [(8192, 0.01), (65536 * 5 + 8, 0.001), ((1 << 20) + 16, 0.05),
                                 ((1 << 22) + 8, 0.3)])
def test_decode_with_device_count(dev, n, p):
    """bsnp_delta_decode_dn: the decode reads n_c from the encode's status
    word on the device (no host round trip between the two): the result is
    the target, status->count the popcount, and a count that disagrees with
    the mask raises the reference's popcount error."""
    import torch
    from paper_2511_12376_b200 import _runtime as rt
    from paper_2511_12376_b200 import bitmask as B
    rng = np.random.default_rng(n)
    base = rng.integers(0, 1 << 16, n, dtype=np.uint16)
    cur = base.copy()
    idx = rng.choice(n, int(n * p), replace=False)
    cur[idx] ^= rng.integers(1, 1 << 16, idx.size, dtype=np.uint16)
    bt, ct = _dev_u16(base, dev), _dev_u16(cur, dev)
    mask = torch.empty((n + 7) // 8, dtype=torch.uint8, device=dev)
    pay = torch.empty(n, dtype=torch.int16, device=dev)
    out = torch.empty_like(bt)
    st = rt.new_status(dev, 2)
    B.encode_delta_async(bt, ct, mask, pay, st[0])
    B.decode_delta_async_dn(bt, mask, pay, st[0], out, st[1])
    (n_c, f0), (pc, f1) = rt.read_status(st)
    assert n_c == pc == idx.size and f0 == f1 == 0
    assert np.array_equal(out.cpu().numpy().view(np.uint16), cur)
    bad = torch.tensor([idx.size + 1, 0], dtype=torch.int64, device=dev)
    B.decode_delta_async_dn(bt, mask, pay, bad, out, st[1])
    (pc, f1), = rt.read_status(st[1:2])
    with pytest.raises(B.DeltaError, match="popcount"):
        B._raise_decode_flags(f1, pc, idx.size + 1)


@pytest.mark.parametrize("n,p,clustered", [(5 * 8192 + 77, 0.005, False), (5 * 8192 + 77, 0.03, False),
                                           ((1 << 20) + 11, 0.0625, False),
                                           (3 * 8192 + 5, 0.02, True)])
def test_in_place_apply_sparse_rounds(dev, n, p, clustered):
    """Sparse chain replay (warp-cooperative scatter: lane l writes the
    changes of rank l, l + 32, ... of a tile) over tiles with one and several
    rounds of 32 changes, and with a tile whose changes all sit in one lane's
    256 elements, equals the oracle's decode."""
    from paper_2511_12376_b200 import bitmask as B
    rng = np.random.default_rng(int(n * p) + clustered)
    base = rng.integers(0, 1 << 16, n, dtype=np.uint16)
    cur = base.copy()
    k = int(round(p * n))
    if clustered:
        idx = 8192 + 256 * 5 + rng.choice(256, min(k, 200), replace=False)  # one lane of tile 1
    else:
        idx = rng.choice(n, k, replace=False)
    cur[idx] ^= rng.integers(1, 1 << 16, idx.size, dtype=np.uint16)
    d = B.encode_delta_device(_dev_u16(base, dev), _dev_u16(cur, dev))
    bt = _dev_u16(base, dev)
    B.decode_delta_device(bt, d.mask, d.payload, d.n_c, out=bt)
    assert np.array_equal(bt.cpu().numpy().view(np.uint16), cur)


def test_in_place_apply_sparse_record_with_a_dense_tile(dev):
    """A sparse record (n_c <= n/16: the per-warp apply) whose one tile holds
    more changes than the warp's shared-memory stage (> 1024): that tile's
    payload is read from global memory; the rest is staged."""
    from paper_2511_12376_b200 import bitmask as B
    rng = np.random.default_rng(17)
    n = 40 * 8192 + 123
    base = rng.integers(0, 1 << 16, n, dtype=np.uint16)
    cur = base.copy()
    idx = np.concatenate([8192 * 7 + rng.choice(8192, 5000, replace=False),  # one dense tile
                          rng.choice(n, 3000, replace=False)])
    idx = np.unique(idx)
    cur[idx] ^= rng.integers(1, 1 << 16, idx.size, dtype=np.uint16)
    assert idx.size * 16 <= n
    d = B.encode_delta_device(_dev_u16(base, dev), _dev_u16(cur, dev))
    bt = _dev_u16(base, dev)
    B.decode_delta_device(bt, d.mask, d.payload, d.n_c, out=bt)
    assert np.array_equal(bt.cpu().numpy().view(np.uint16), cur)


def test_concurrent_callers_from_threads(dev):
    """The reference codec is pure and reentrant ("callers may encode
    different tensors in parallel"): four host threads encode and decode
    their own tensors through the compat API at the same time (per-thread
    workspaces), each getting the oracle's bytes back."""
    import threading
    from paper_2511_12376_b200 import bitmask as B
    from paper_2511_12376_b200.tensors import ElementType, TensorBlob
    errors = []

    def work(seed):
        try:
            rng = np.random.default_rng(seed)
            for _ in range(5):
                n = int(rng.integers(1, 300_000))
                base = rng.integers(0, 1 << 16, n, dtype=np.uint16)
                cur = base.copy()
                k = int(rng.integers(0, n // 10 + 1))
                if k:
                    cur[rng.choice(n, k, replace=False)] ^= 1
                tb = TensorBlob("t", ElementType.F16, (n,), base.tobytes())
                tc = TensorBlob("t", ElementType.F16, (n,), cur.tobytes())
                rec = B.encode_delta(tb, tc)
                mask, payload, n_c = O.delta_encode(base, cur)
                assert rec.changed_count == n_c and rec.packed_mask == mask.tobytes()
                assert rec.payload == payload.tobytes()
                assert B.decode_delta(tb, rec).data == tc.data
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=work, args=(s,)) for s in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
