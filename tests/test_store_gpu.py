"""Checkpoint driver on the GPU: encode_checkpoint (store.py:214-272) and the
load-side chain replay (store.py:418-474) against the reference's own
outputs (tests/golden/checkpoint_golden.npz, made by running the reference
store) and the CPU oracle."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from oracle import bitsnap_oracle as O
from paper_2511_12376_b200 import planner as P
from paper_2511_12376_b200 import store as S
from paper_2511_12376_b200.tensors import Checkpoint, ElementType, TensorBlob

pytestmark = pytest.mark.gpu


def _golden_ckpts(g, meta):
    model0, model1, opt = [], [], []
    for name, shape in meta["shapes"].items():
        shape = tuple(shape)
        model0.append(TensorBlob(name, ElementType.F16, shape, g[f"w0:{name}"].astype("<u2").tobytes()))
        model1.append(TensorBlob(name, ElementType.F16, shape, g[f"w1:{name}"].astype("<u2").tobytes()))
        for kind in ("m", "v"):
            opt.append(TensorBlob(f"adam.{kind}.{name}", ElementType.F32, shape,
                                  g[f"{kind}:{name}"].astype("<f4").tobytes()))
    return (Checkpoint(iteration=100, model_states=model0, optimizer_states=opt),
            Checkpoint(iteration=110, model_states=model1, optimizer_states=opt))


def test_encode_checkpoint_matches_reference_golden(dev, checkpoint_golden, golden_index):
    g, meta = checkpoint_golden, golden_index["checkpoint"]
    c0, c1 = _golden_ckpts(g, meta)
    man0, blob0 = S.encode_checkpoint(c0, None, S.KIND_BASE, 16)
    man1, blob1 = S.encode_checkpoint(c1, c0, S.KIND_DELTA, 16)
    assert blob0 == g["blob0"].tobytes()
    assert blob1 == g["blob1"].tobytes()
    assert man0.to_bytes() == g["manifest0"].tobytes()
    assert man1.to_bytes() == g["manifest1"].tobytes()


def test_resident_encoder_device_tensors(dev, checkpoint_golden, golden_index):
    """Device-resident save path: DeviceTensors in, previous model states kept
    in HBM between saves (no prev argument), same bytes as the reference."""
    g, meta = checkpoint_golden, golden_index["checkpoint"]
    c0, c1 = _golden_ckpts(g, meta)

    def on_device(c, bf16):
        wrap = []
        for t in c.model_states:
            a = torch.from_numpy(np.frombuffer(t.data, np.int16).copy()).to(dev)
            wrap.append(S.DeviceTensor(t.name, t.dtype, t.shape,
                                       a.view(torch.bfloat16) if bf16 else a))
        opt = [S.DeviceTensor(t.name, t.dtype, t.shape,
                              torch.from_numpy(np.frombuffer(t.data, np.float32).copy())
                              .to(dev).reshape(t.shape)) for t in c.optimizer_states]
        return Checkpoint(iteration=c.iteration, model_states=wrap, optimizer_states=opt)

    enc = S.CheckpointEncoder(dev, clusters=16)
    d0 = on_device(c0, bf16=True)
    man0, out0 = enc.encode(d0, None, S.KIND_BASE)
    man1, out1 = enc.encode(on_device(c1, bf16=True), None, S.KIND_DELTA)
    assert out0.numpy().tobytes() == g["blob0"].tobytes()
    assert out1.numpy().tobytes() == g["blob1"].tobytes()
    assert man1.to_bytes() == g["manifest1"].tobytes()
    assert man1.base_iteration == 100


@pytest.mark.parametrize("graphs", ["1", "0"])
def test_in_place_updates_between_saves(dev, checkpoint_golden, golden_index, monkeypatch,
                                        graphs):
    """A training loop saves its LIVE parameter buffers, which the optimizer
    changes in place between saves: the resident delta base
    must be the encoder's own copy, or every later delta would compare each
    buffer with itself (n_c = 0) and a restore would give back the base."""
    monkeypatch.setenv("BSNP_GRAPHS", graphs)
    g, meta = checkpoint_golden, golden_index["checkpoint"]
    c0, c1 = _golden_ckpts(g, meta)
    live = [torch.from_numpy(np.frombuffer(t.data, np.int16).copy()).to(dev)
            for t in c0.model_states]
    opt = [S.DeviceTensor(t.name, t.dtype, t.shape,
                          torch.from_numpy(np.frombuffer(t.data, np.float32).copy()).to(dev))
           for t in c0.optimizer_states]

    def snap(it):
        return Checkpoint(iteration=it, optimizer_states=opt, model_states=[
            S.DeviceTensor(t.name, t.dtype, t.shape, a) for t, a in zip(c0.model_states, live)])

    enc = S.CheckpointEncoder(dev, clusters=16)
    chain, states = [], []
    rng = np.random.default_rng(3)
    for it in range(4):
        man, out = enc.encode(snap(100 + it), None, S.KIND_BASE if it == 0 else S.KIND_DELTA)
        chain.append((man, out.numpy().tobytes()))
        states.append([a.cpu().numpy().copy() for a in live])
        for a in live:          # the optimizer step: in place
            k = max(1, a.numel() // 50)
            idx = torch.from_numpy(rng.choice(a.numel(), k, replace=False)).to(dev)
            a.view(-1)[idx] += 1
    for it in range(1, 4):
        rec = S.decode_chain(chain[:it + 1])
        for t, want in zip(rec.model_states, states[it]):
            assert t.data == want.tobytes()
        assert any(e.codec == S.CODEC_DELTA for e in chain[it][0].tensors)
    # borrow mode refuses a base that is the same memory as the new state
    enc_b = S.CheckpointEncoder(dev, clusters=16, keep_prev="borrow")
    enc_b.encode(snap(200), None, S.KIND_BASE)
    with pytest.raises(S.StoreError, match="mutated in place"):
        enc_b.encode(snap(201), None, S.KIND_DELTA)


def test_decode_chain_round_trip(dev, checkpoint_golden, golden_index):
    g, meta = checkpoint_golden, golden_index["checkpoint"]
    c0, c1 = _golden_ckpts(g, meta)
    chain = [(S.CheckpointManifest.from_bytes(g["manifest0"].tobytes()), g["blob0"].tobytes()),
             (S.CheckpointManifest.from_bytes(g["manifest1"].tobytes()), g["blob1"].tobytes())]
    out = S.decode_chain(chain)
    assert out.iteration == 110
    assert [t.name for t in out.model_states] == [t.name for t in c1.model_states]
    for a, b in zip(out.model_states, c1.model_states):
        assert a.data == b.data and a.shape == b.shape and a.dtype is ElementType.F16
    for a, b in zip(out.optimizer_states, c1.optimizer_states):
        x = np.frombuffer(b.data, np.float32)
        tab = O.cluster_fit(x, 16)
        p, c, _ = O.cluster_quantize(x, tab)
        want = O.cluster_dequantize(p, c, x.size, tab)
        assert a.data == want.astype("<f4").tobytes()
    # base alone
    out0 = S.decode_chain(chain[:1])
    for a, b in zip(out0.model_states, c0.model_states):
        assert a.data == b.data


def _random_ckpt(rng, iteration, prev=None):
    shapes = [(1000, 3), (8191,), (5,), (64, 64), (1,), (0,), (3, 3, 3)]
    model = []
    for i, shp in enumerate(shapes):
        n = int(np.prod(shp))
        if prev is None:
            a = rng.integers(0, 1 << 16, n, dtype=np.uint16)
        else:
            a = np.frombuffer(prev.model_states[i].data, np.uint16).copy()
            k = int(n * [0.01, 0.3, 1.0, 0.0, 1.0, 0, 0.5][i])
            idx = rng.choice(n, k, replace=False) if k else np.zeros(0, np.int64)
            a[idx] ^= rng.integers(1, 1 << 16, k, dtype=np.uint16)
        model.append(TensorBlob(f"p{i}", ElementType.F16, shp, a.tobytes()))
    opt = [TensorBlob(f"o{i}", ElementType.F32, (n,),
                      (rng.standard_normal(n) * s).astype(np.float32).tobytes())
           for i, (n, s) in enumerate([(3000, 1e-3), (1, 1.0), (129, 5.0), (70000, 1e-6)])]
    return Checkpoint(iteration=iteration, model_states=model, optimizer_states=opt)


def _oracle(ck, prev, kind, clusters=16):
    conv = lambda ts, code: [(t.name, t.shape, code,
                              np.frombuffer(t.data, np.uint16 if code == 0 else np.float32))
                             for t in ts]
    return O.encode_checkpoint(conv(ck.model_states, 0), conv(ck.optimizer_states, 1),
                               conv(prev.model_states, 0) if prev else None, kind, clusters)


@pytest.mark.parametrize("clusters", [16, 5, 2])
def test_random_chain_vs_oracle(dev, clusters):
    rng = np.random.default_rng(clusters)
    c0 = _random_ckpt(rng, 1)
    c1 = _random_ckpt(rng, 2, c0)
    c2 = _random_ckpt(rng, 3, c1)
    enc = S.CheckpointEncoder(dev, clusters=clusters)
    chain = []
    for ck, prev, kind in ((c0, None, "base"), (c1, c0, "delta"), (c2, c1, "delta")):
        man, out = enc.encode(ck, None, kind)      # prev resident on the device
        entries, want = _oracle(ck, prev, kind, clusters)
        assert out.numpy().tobytes() == want
        assert [vars(e) for e in man.tensors] == entries
        chain.append((man, out.numpy().tobytes()))
    rec = S.decode_chain(chain)
    for a, b in zip(rec.model_states, c2.model_states):
        assert a.data == b.data
    # the batched dequantize (one launch per upload chunk) vs the oracle
    assert [t.name for t in rec.optimizer_states] == [t.name for t in c2.optimizer_states]
    for a, b in zip(rec.optimizer_states, c2.optimizer_states):
        x = np.frombuffer(b.data, np.float32)
        tab = O.cluster_fit(x, clusters)
        p, c, _ = O.cluster_quantize(x, tab)
        assert a.data == O.cluster_dequantize(p, c, x.size, tab).astype("<f4").tobytes()


def test_store_errors(dev):
    rng = np.random.default_rng(5)
    c0 = _random_ckpt(rng, 1)
    c1 = _random_ckpt(rng, 2, c0)
    with pytest.raises(S.MissingPreviousError):
        S.encode_checkpoint(c1, None, S.KIND_DELTA)
    other = Checkpoint(iteration=1, model_states=c0.model_states[:-1],
                       optimizer_states=c0.optimizer_states)
    with pytest.raises(S.StoreError, match="structure"):
        S.encode_checkpoint(c1, other, S.KIND_DELTA)
    with pytest.raises(S.StoreError, match="kind"):
        S.encode_checkpoint(c0, None, "full")
    # a corrupt delta record (padding bits) is rejected on replay
    man0, b0 = S.encode_checkpoint(c0, None, S.KIND_BASE)
    man1, b1 = S.encode_checkpoint(c1, c0, S.KIND_DELTA)
    e = [x for x in man1.tensors if x.codec == "DELTA" and x.name == "p6"][0]
    bad = bytearray(b1)
    hdr = 4 + 2 + 8 + 8 + 2 + len("p6") + 1 + 8 * 3
    n = 27
    bad[e.offset + hdr + (n + 7) // 8 - 1] |= 0x80
    from paper_2511_12376_b200.bitmask import DeltaError
    with pytest.raises(DeltaError, match="padding"):
        S.decode_chain([(man0, b0), (man1, bytes(bad))])
    # a label >= m in a quantized record (quantizer.py:196-197) is rejected
    man5, b5 = S.encode_checkpoint(c1, c0, S.KIND_DELTA, clusters=5)
    e = [x for x in man5.tensors if x.codec == "QUANT"][2]
    lo = S._parse_quant(memoryview(b5), e)[3]
    bad = bytearray(b5)
    bad[lo] = 0xF7
    from paper_2511_12376_b200.quantizer import QuantizerError
    with pytest.raises(QuantizerError, match="label 15 >= m=5"):
        S.decode_chain([(man0, b0), (man5, bytes(bad))])
    # the delta error of the same restore is reported first (model records
    # are replayed before the optimizer records)
    bad2 = bytearray(bad)
    e = [x for x in man5.tensors if x.codec == "DELTA" and x.name == "p6"][0]
    bad2[e.offset + hdr + (n + 7) // 8 - 1] |= 0x80
    with pytest.raises(DeltaError, match="padding"):
        S.decode_chain([(man0, b0), (man5, bytes(bad2))])


def test_planner_world1_with_gpu_encoder(dev, tmp_path):
    rng = np.random.default_rng(11)
    c0 = _random_ckpt(rng, 1)
    c1 = _random_ckpt(rng, 2, c0)
    specs = P.checkpoint_specs(c1)
    local = {t.name: t for t in c1.model_states + c1.optimizer_states}
    res = P.encode_sharded(specs, local, {t.name: t for t in c0.model_states}, "delta",
                           2, 1, 0, 1, S.CheckpointEncoder(dev, keep_prev=False))
    path = str(tmp_path / "tensors.bin")
    P.write_shard(path, res)
    man, want = S.encode_checkpoint(c1, c0, S.KIND_DELTA)
    assert open(path, "rb").read() == want
    assert res.manifest.to_bytes() == man.to_bytes()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gpu_worker(rank, world, port, path, q):
    """Two ranks sharing cuda:0 (independent kernels, no cross-rank waits);
    the size-table all-gather goes over gloo."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(11)
        c0 = _random_ckpt(rng, 1)
        c1 = _random_ckpt(rng, 2, c0)
        specs = P.checkpoint_specs(c1)
        plan = P.plan_shards([s.nbytes for s in specs], world)
        mine = {specs[i].name for i in plan.local_ids(rank)}
        local = {t.name: t for t in c1.model_states + c1.optimizer_states if t.name in mine}
        prev = {t.name: t for t in c0.model_states if t.name in mine}
        dev = torch.device("cuda:0")
        res = P.encode_sharded(specs, local, prev, "delta", 2, 1, rank, world,
                               S.CheckpointEncoder(dev, keep_prev=False),
                               device=torch.device("cpu"))
        P.write_shard(path, res, device=dev)
        dist.barrier()
        q.put(res.manifest.to_bytes())
    finally:
        dist.destroy_process_group()


def test_planner_two_ranks_one_gpu(dev, tmp_path):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    path = str(tmp_path / "tensors.bin")
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    mans = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rng = np.random.default_rng(11)
    c0 = _random_ckpt(rng, 1)
    c1 = _random_ckpt(rng, 2, c0)
    entries, want = _oracle(c1, c0, "delta")
    assert open(path, "rb").read() == want
    assert mans[0] == mans[1]
    assert [vars(e) for e in S.CheckpointManifest.from_bytes(mans[0]).tensors] == entries


def test_graph_replay_of_repeated_saves(dev, checkpoint_golden, golden_index):
    """Device-resident saves of the same tensors: the first runs eagerly, the
    second records the launch sequence as a CUDA graph, later ones replay it
    (after the inputs changed in place): every blob equals the reference's."""
    g, meta = checkpoint_golden, golden_index["checkpoint"]
    c0, c1 = _golden_ckpts(g, meta)

    def on_device(c):
        ms = [S.DeviceTensor(t.name, t.dtype, t.shape,
                             torch.from_numpy(np.frombuffer(t.data, np.int16).copy()).to(dev))
              for t in c.model_states]
        os_ = [S.DeviceTensor(t.name, t.dtype, t.shape,
                              torch.from_numpy(np.frombuffer(t.data, np.float32).copy()).to(dev))
               for t in c.optimizer_states]
        return Checkpoint(iteration=c.iteration, model_states=ms, optimizer_states=os_)

    d0, d1 = on_device(c0), on_device(c1)
    zero = on_device(c0)
    for t in zero.optimizer_states:
        t.data.zero_()
    enc = S.CheckpointEncoder(dev, clusters=16, keep_prev=False)
    for rep in range(4):
        if rep == 3:   # same addresses, new contents: the replay must see them
            for a, b in zip(d1.optimizer_states, zero.optimizer_states):
                a.data.copy_(b.data)
        man, out = enc.encode(d1, d0, S.KIND_DELTA)
        if rep < 3:
            assert out.numpy().tobytes() == g["blob1"].tobytes(), rep
            assert man.to_bytes() == g["manifest1"].tobytes()
        else:
            ref, _ = S.CheckpointEncoder(dev, clusters=16, keep_prev=False).encode(
                Checkpoint(iteration=110, model_states=c1.model_states,
                           optimizer_states=[t.to_blob() for t in zero.optimizer_states]),
                c0, S.KIND_DELTA)
            assert man.to_bytes() == ref.to_bytes()
    assert len(enc._graphs) == 1


@pytest.mark.parametrize("groups", [1, 2, 3, 8])
def test_pipelined_save_into_caller_buffer(dev, checkpoint_golden, golden_index, groups):
    """encode() into a pinned buffer that can hold any outcome overlaps the
    encode of one group of tensors with the copy-out of the previous one:
    same blob and manifest as the reference for any group count."""
    g, meta = checkpoint_golden, golden_index["checkpoint"]
    c0, c1 = _golden_ckpts(g, meta)
    enc = S.CheckpointEncoder(dev, clusters=16, keep_prev=False)
    enc.pipeline_groups = groups
    enc.pipeline_min_bytes = 0      # (the default) any size takes the pipelined path
    buf = torch.empty(S.blob_bound(c1) + 7, dtype=torch.uint8, pin_memory=True)
    for ck, prev, kind, bkey, mkey in ((c0, None, S.KIND_BASE, "blob0", "manifest0"),
                                       (c1, c0, S.KIND_DELTA, "blob1", "manifest1")):
        man, out = enc.encode(ck, prev, kind, out=buf)
        assert out.numpy().tobytes() == g[bkey].tobytes()
        assert man.to_bytes() == g[mkey].tobytes()


def test_chain_replay_uploads_only_needed_spans(dev, checkpoint_golden, golden_index):
    """Earlier links of a chain contribute only their model records: a base
    blob truncated after its model section decodes to the same checkpoint."""
    g = checkpoint_golden
    m0 = S.CheckpointManifest.from_bytes(g["manifest0"].tobytes())
    m1 = S.CheckpointManifest.from_bytes(g["manifest1"].tobytes())
    end = max(e.offset + e.length for e in m0.tensors if e.group == S.GROUP_MODEL)
    full = S.decode_chain([(m0, g["blob0"].tobytes()), (m1, g["blob1"].tobytes())])
    cut = S.decode_chain([(m0, g["blob0"].tobytes()[:end]), (m1, g["blob1"].tobytes())])
    assert [t.data for t in full.model_states] == [t.data for t in cut.model_states]
    assert [t.data for t in full.optimizer_states] == [t.data for t in cut.optimizer_states]


def test_copy_sm_into_pinned_host(dev):
    """bsnp_copy_sm: device bytes land in page-locked host memory by SM
    stores (aligned vector path and byte path), nothing outside the range."""
    from paper_2511_12376_b200 import _lib
    from paper_2511_12376_b200 import _runtime as rt
    src = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device=dev)
    want = src.cpu()
    for so, do, n in ((0, 0, 1 << 20), (16, 32, 4096), (3, 0, 77), (5, 7, 99997), (0, 0, 1)):
        dst = torch.zeros((1 << 20) + 64, dtype=torch.uint8, pin_memory=True)
        _lib.check(rt.lib().bsnp_copy_sm(src.data_ptr() + so, dst.data_ptr() + do, n,
                                         rt.stream_ptr(dev)), "bsnp_copy_sm")
        torch.cuda.current_stream(dev).synchronize()
        assert torch.equal(dst[do:do + n], want[so:so + n])
        assert int(dst[:do].sum()) == 0 and int(dst[do + n:].sum()) == 0


def test_multi_chunk_restore_vs_oracle(dev):
    """A chain whose links upload in 8 chunks, records straddling chunk
    boundaries: the grouped restore (one gather and one batched dequantize
    per chunk, deltas on side streams) rebuilds the weights bit for bit and
    the optimizer states as the oracle's dequantize, from host bytes and
    from pinned blobs alike."""
    rng = np.random.default_rng(7)
    sizes = [1, 7, 1000, 65535, 65537, 300001, 1 << 20, 777777, 3, 123457, 1 << 19, 2,
             999999, 4096, 250000]
    frac = [1.0, 0.0, 0.3, 0.01, 0.0, 0.05, 0.02, 1.0, 0.5, 0.001, 0.2, 1.0, 0.04, 0.6, 0.0]
    model0, model1, opt = [], [], []
    for i, (n, f) in enumerate(zip(sizes, frac)):
        a = rng.integers(0, 1 << 16, n, dtype=np.uint16)
        b = a.copy()
        k = int(n * f)
        if k:
            idx = rng.choice(n, k, replace=False)
            b[idx] ^= rng.integers(1, 1 << 16, k, dtype=np.uint16)
        model0.append(TensorBlob(f"w{i}", ElementType.F16, (n,), a.tobytes()))
        model1.append(TensorBlob(f"w{i}", ElementType.F16, (n,), b.tobytes()))
        if n > 1:
            opt.append(TensorBlob(f"m{i}", ElementType.F32, (n,),
                                  (rng.standard_normal(n) * 1e-3).astype(np.float32).tobytes()))
    c0 = Checkpoint(iteration=1, model_states=model0, optimizer_states=opt)
    c1 = Checkpoint(iteration=2, model_states=model1, optimizer_states=opt)
    enc = S.CheckpointEncoder(dev, clusters=16)
    m0, b0 = enc.encode(c0, None, S.KIND_BASE)
    m1, b1 = enc.encode(c1, None, S.KIND_DELTA)
    codecs = {e.codec for e in m1.tensors if e.group == S.GROUP_MODEL}
    assert codecs == {"RAW", "DELTA"}
    want_opt = []
    for t in opt:
        x = np.frombuffer(t.data, np.float32)
        tab = O.cluster_fit(x, 16)
        p, c, _ = O.cluster_quantize(x, tab)
        want_opt.append(O.cluster_dequantize(p, c, x.size, tab).astype("<f4").tobytes())
    for chain in ([(m0, b0.numpy().tobytes()), (m1, b1.numpy().tobytes())],
                  [(m0, b0), (m1, b1)]):
        rec = S.decode_chain(chain)
        assert [t.data for t in rec.model_states] == [t.data for t in model1]
        assert [t.data for t in rec.optimizer_states] == want_opt
    # a third link: the middle link now contributes only its model span
    model2 = []
    for t in model1:
        a = np.frombuffer(t.data, np.uint16).copy()
        k = a.size // 3
        if k:
            a[rng.choice(a.size, k, replace=False)] += 1
        model2.append(TensorBlob(t.name, ElementType.F16, t.shape, a.tobytes()))
    c2 = Checkpoint(iteration=3, model_states=model2, optimizer_states=opt)
    m2, b2 = enc.encode(c2, None, S.KIND_DELTA)
    rec = S.decode_chain([(m0, b0), (m1, b1.numpy().tobytes()), (m2, b2)])
    assert [t.data for t in rec.model_states] == [t.data for t in model2]
    assert [t.data for t in rec.optimizer_states] == want_opt


def test_save_and_restore_through_registered_host_memory(dev, checkpoint_golden, golden_index):
    """Landing buffers page-locked by registration (bsnp_host_register on a
    plain host allocation, as for tens-of-GB checkpoints) behave as pinned
    ones: same blobs as the reference, same restore."""
    from paper_2511_12376_b200 import _runtime as rt
    g, meta = checkpoint_golden, golden_index["checkpoint"]
    c0, c1 = _golden_ckpts(g, meta)
    enc = S.CheckpointEncoder(dev, clusters=16)
    arrs, bufs = [], []
    for ck in (c0, c1):
        a = np.zeros(S.blob_bound(ck) + 64, dtype=np.uint8)
        assert rt.lib().bsnp_host_register(a.ctypes.data, a.nbytes) == 0
        arrs.append(a)
        bufs.append(torch.from_numpy(a))
    try:
        assert all(b.is_pinned() for b in bufs)
        m0, b0 = enc.encode(c0, None, S.KIND_BASE, out=bufs[0])
        m1, b1 = enc.encode(c1, None, S.KIND_DELTA, out=bufs[1])
        assert b0.numpy().tobytes() == g["blob0"].tobytes()
        assert b1.numpy().tobytes() == g["blob1"].tobytes()
        rec = S.decode_chain([(m0, b0), (m1, b1)])
        assert [t.data for t in rec.model_states] == [t.data for t in c1.model_states]
    finally:
        torch.cuda.synchronize()
        for a in arrs:
            rt.lib().bsnp_host_unregister(a.ctypes.data)
