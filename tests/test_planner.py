"""Shard planner: LPT plan, one all-gather of the size table, global offsets.

The multi-rank path runs here on CPU with the gloo backend (world_size 2 and
3): every rank encodes only the tensors the plan gives it (with the CPU
oracle standing in for the GPU encoder, as the checker), exchanges its rows,
and pwrites its records at the global offsets.  The assembled tensors.bin
and the manifest must equal the single-process reference driver's
(store.py:214-272), byte for byte.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bitsnap_oracle as O
from paper_2511_12376_b200 import planner as P
from paper_2511_12376_b200.store import CheckpointManifest, EncodedRecord, ManifestEntry
from paper_2511_12376_b200.tensors import Checkpoint, ElementType, TensorBlob


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ckpt(seed: int, iteration: int, prev: Checkpoint | None = None, frac=0.05):
    """Small checkpoint: bf16-pattern model states (some identical, some
    heavily changed so RAW fallback is exercised) and F32 Adam-like states."""
    rng = np.random.default_rng(seed)
    shapes = [(64, 48), (7,), (33, 5), (1,), (96,), (0,)]
    model = []
    for i, shp in enumerate(shapes):
        n = int(np.prod(shp))
        if prev is None:
            a = rng.integers(0, 1 << 16, n, dtype=np.uint16)
        else:
            a = np.frombuffer(prev.model_states[i].data, np.uint16).copy()
            f = 0.97 if i == 2 else (0.0 if i == 3 else frac)
            k = int(round(f * n))
            idx = rng.choice(n, k, replace=False) if k else np.zeros(0, np.int64)
            a[idx] ^= rng.integers(1, 1 << 16, k, dtype=np.uint16)
        model.append(TensorBlob(f"w{i}", ElementType.F16, shp, a.tobytes()))
    opt = []
    for i, n in enumerate([1000, 37, 4096]):
        x = (rng.standard_normal(n) * 1e-3).astype(np.float32)
        if i == 1:
            x = x * x
        opt.append(TensorBlob(f"adam{i}", ElementType.F32, (n,), x.tobytes()))
    return Checkpoint(iteration=iteration, model_states=model, optimizer_states=opt)


def _oracle_blob(ckpt, prev, kind):
    conv = lambda ts, code: [(t.name, t.shape, code,
                              np.frombuffer(t.data, np.uint16 if code == 0 else np.float32))
                             for t in ts]
    entries, blob = O.encode_checkpoint(conv(ckpt.model_states, 0),
                                        conv(ckpt.optimizer_states, 1),
                                        conv(prev.model_states, 0) if prev else None, kind, 16)
    return entries, blob


class OracleEncoder:
    """Host encoder with the CheckpointEncoder.encode_records interface,
    built on the CPU oracle (test checker only)."""

    def encode_records(self, items, prev_map, kind):
        out = []
        for gid, group, t in items:
            if group == "model":
                raw = O.raw_record(t.name, 0, t.shape, t.data)
                if kind == "base":
                    out.append(EncodedRecord(gid, t.name, group, "RAW", t.num_elements, raw, []))
                    continue
                b = np.frombuffer(prev_map[t.name].data, np.uint16)
                mask, payload, n_c = O.delta_encode(b, np.frombuffer(t.data, np.uint16))
                enc = O.delta_record(t.name, t.shape, t.num_elements, n_c, mask, payload)
                if len(enc) < len(raw):
                    out.append(EncodedRecord(gid, t.name, group, "DELTA", n_c, enc, []))
                else:
                    out.append(EncodedRecord(gid, t.name, group, "RAW", t.num_elements, raw, []))
            else:
                x = np.frombuffer(t.data, np.float32)
                tab = O.cluster_fit(x, 16)
                packed, codes, _ = O.cluster_quantize(x, tab)
                out.append(EncodedRecord(gid, t.name, group, "QUANT", 16,
                                         O.quant_record(t.name, t.shape, tab, packed, codes), []))
        return out, {}


def _worker(rank, world, port, path, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c0 = _ckpt(0, 10)
        c1 = _ckpt(1, 11, prev=c0)
        ck, prev = (c0, None) if kind == "base" else (c1, c0)
        specs = P.checkpoint_specs(ck)
        plan = P.plan_shards([s.nbytes for s in specs], world)
        mine = {specs[g].name for g in plan.local_ids(rank)}
        # each rank holds only its own tensors (and their predecessors)
        local = {t.name: t for t in ck.model_states + ck.optimizer_states if t.name in mine}
        prev_local = ({t.name: t for t in prev.model_states if t.name in mine}
                      if prev else None)
        res = P.encode_sharded(specs, local, prev_local, kind, ck.iteration,
                               ck.iteration if kind == "base" else prev.iteration,
                               rank, world, OracleEncoder(), device=torch.device("cpu"))
        P.write_shard(path, res)
        dist.barrier()
        q.put((rank, res.manifest.to_bytes(), res.total_bytes))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["base", "delta"])
def test_sharded_encode_gloo_matches_single_process(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "tensors.bin")
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, path, kind, q))
                 for r in range(world)]
        for p in procs:
            p.start()
        res = [q.get(timeout=120) for _ in range(world)]
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        blob = open(path, "rb").read()
    c0 = _ckpt(0, 10)
    c1 = _ckpt(1, 11, prev=c0)
    ck, prev = (c0, None) if kind == "base" else (c1, c0)
    entries, want = _oracle_blob(ck, prev, kind)
    assert blob == want
    manifests = {m for _, m, _ in res}
    assert len(manifests) == 1      # identical on every rank
    man = CheckpointManifest.from_bytes(manifests.pop())
    assert [vars(e) for e in man.tensors] == entries
    assert all(t == len(want) for _, _, t in res)
    if kind == "delta":
        codecs = [e["codec"] for e in entries]
        assert "DELTA" in codecs and "RAW" in codecs   # w2 is 97 % changed


def test_plan_is_deterministic_and_balanced():
    sizes = [int(x) for x in np.random.default_rng(3).integers(1, 10 ** 6, 300)]
    a = P.plan_shards(sizes, 8)
    b = P.plan_shards(list(sizes), 8)
    assert a == b
    assert sorted(set(a.owner)) == list(range(8))
    assert a.imbalance < 1.01
    assert sum(a.load) == sum(sizes)
    assert P.plan_shards(sizes, 1).owner == (0,) * 300


def test_plan_llama70b_shapes_fit_8_gpus():
    """LPT of the C4 tensors (bf16 w + base, fp32 m, v)
    over 8 ranks is within 0.1 % of perfect balance."""
    d, ffn, kv, vocab = 8192, 28672, 1024, 32000
    per_layer = [d, d * d, d * kv, d * kv, d * d, ffn * d, ffn * d, d * ffn, d]
    numels = [vocab * d, vocab * d, d] + per_layer * 80
    bytes_ = [n * (2 + 2 + 4 + 4) for n in numels]
    plan = P.plan_shards(bytes_, 8)
    assert plan.imbalance < 1.001
    assert max(plan.load) < 110e9   # ~103.5 GB per GPU of 180 GB HBM


def test_global_offsets_rejects_bad_tables():
    rows = torch.tensor([[1, 0, 5, 10], [0, 1, 3, 7], [-1, -1, -1, -1]])
    out = P.global_offsets(rows, 2)
    assert out == [(1, 3, 0, 7), (0, 5, 7, 10)]
    with pytest.raises(ValueError):
        P.global_offsets(rows, 3)
    with pytest.raises(ValueError):
        P.global_offsets(torch.tensor([[0, 0, 1, 1], [0, 0, 1, 1]]), 2)


def test_manifest_json_byte_identical(checkpoint_golden):
    """store.py:154-171: the manifest JSON round-trips byte for byte."""
    for k in ("manifest0", "manifest1"):
        raw = checkpoint_golden[k].tobytes()
        m = CheckpointManifest.from_bytes(raw)
        assert m.to_bytes() == raw
    from paper_2511_12376_b200.store import StoreError
    with pytest.raises(StoreError, match="corrupt manifest"):
        CheckpointManifest.from_bytes(b"{not json")
    with pytest.raises(StoreError, match="older base"):
        CheckpointManifest(iteration=3, kind="delta", base_iteration=3)
    with pytest.raises(StoreError, match="codec"):
        CheckpointManifest(iteration=3, kind="base", base_iteration=3,
                           tensors=(ManifestEntry("w", "model", "QUANT", 0, 1),))


def _rows_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r holds global ids r, r + world (one row as a list, one as a tensor)
        rows_list = [(rank, 1, 10 + rank, 100 + rank)]
        rows_t = torch.tensor([[rank + world, 2, 20 + rank, 200 + rank]], dtype=torch.int64)
        a = P.exchange_sizes(rows_list, world, 2)
        b = P.exchange_sizes(rows_t, world, 2)
        q.put((rank, a.tolist(), b.tolist()))
    finally:
        dist.destroy_process_group()


def test_exchange_sizes_accepts_device_style_tensor_rows():
    """The size rows may be a tensor (the bench builds them on the GPU from
    the encoder's status word): same all-gather, same padding, at world 2."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rows_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, a, b in res:
        assert a == [[0, 1, 10, 100], [-1, -1, -1, -1], [1, 1, 11, 101], [-1, -1, -1, -1]]
        assert b == [[2, 2, 20, 200], [-1, -1, -1, -1], [3, 2, 21, 201], [-1, -1, -1, -1]]
    # without a process group: the local rows, padded
    t = P.exchange_sizes(torch.tensor([[0, 1, 5, 9]]), 1, 3)
    assert t.tolist() == [[0, 1, 5, 9], [-1, -1, -1, -1], [-1, -1, -1, -1]]
