"""The reference store's save / load entry points over the B200 codec
(fsstore.py; reference store.py:84-111, 306-474) and the async agent
(engine.py:235-306): same on-disk layout, same tracker and base-refresh
policy, byte-identical tensors.bin (the golden checkpoint the reference's own
store wrote, tests/golden/make_golden.py)."""

import os
import sys

import numpy as np
import pytest

from paper_2511_12376_b200 import engine as E
from paper_2511_12376_b200 import store as S
from paper_2511_12376_b200.tensors import Checkpoint, ElementType, TensorBlob

REF_SRC = "/root/reference/pkg/src"


def _golden(g):
    return [(S.CheckpointManifest.from_bytes(g[f"manifest{i}"].tobytes()), g[f"blob{i}"].tobytes())
            for i in (0, 1)]


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


def test_commit_layout_and_policy(tmp_path, checkpoint_golden, monkeypatch):
    monkeypatch.delenv("MAX_CACHED_ITERATION", raising=False)
    cfg = S.StoreConfig(tmp_path / "store", max_cached_iteration=2)
    assert S.decide_kind(cfg, 100) == S.KIND_BASE
    (m0, b0), (m1, b1) = _golden(checkpoint_golden)
    S.commit(cfg, m0, b0)
    assert S.decide_kind(cfg, 110) == S.KIND_DELTA
    S.commit(cfg, m1, b1)
    assert S.decide_kind(cfg, 120) == S.KIND_BASE      # max_cached_iteration = 2
    d = cfg.iter_dir(110)
    assert d.name == "iter_0000110"
    assert (d / "tensors.bin").read_bytes() == b1
    assert (d / "manifest.bin").read_bytes() == m1.to_bytes()
    assert (d / "type.txt").read_text() == "delta\n"
    assert cfg.tracker_path().read_text() == "110\n100\n"
    assert S.list_iterations(cfg) == [100, 110]
    assert S.read_manifest(cfg, 110) == m1
    with pytest.raises(S.MissingLinkError):
        S.read_manifest(cfg, 105)
    (cfg.root / ".needs_base").touch()
    assert S.decide_kind(cfg, 120) == S.KIND_BASE
    monkeypatch.setenv("MAX_CACHED_ITERATION", "5")
    os.unlink(cfg.root / ".needs_base")
    assert S.decide_kind(cfg, 120) == S.KIND_DELTA
    with pytest.raises(S.StoreError):
        S.StoreConfig(tmp_path / "x", redundancy_depth=0)
    # the tracker API and error types of the reference (store.py:66-121,
    # 181-207): TrackerState, TrackerError / MissingLinkError are StoreErrors
    assert S.read_tracker(cfg) == S.TrackerState(110, 100)
    S.write_tracker(cfg, S.TrackerState(120, 120))
    assert cfg.tracker_path().read_text() == "120\n120\n"
    with pytest.raises(S.TrackerError):
        S.TrackerState(1, 2)
    cfg.tracker_path().write_text("garbage\n")
    with pytest.raises(S.StoreError, match="malformed tracker"):
        S.read_tracker(cfg)
    assert S.try_read_tracker(cfg) is None
    with pytest.raises(S.StoreError, match="checkpoint chain broken: iteration 105 missing"):
        S.read_manifest(cfg, 105)


def test_checkpoint_file_roundtrip(tmp_path, checkpoint_golden, golden_index):
    """tensors.py:217-224: write_checkpoint_file / read_checkpoint_file."""
    from paper_2511_12376_b200 import tensors as T
    c0, _ = _golden_ckpts(checkpoint_golden, golden_index["checkpoint"])
    T.write_checkpoint_file(tmp_path / "c.bsck", c0)
    back = T.read_checkpoint_file(tmp_path / "c.bsck")
    assert back == c0
    assert (tmp_path / "c.bsck").read_bytes() == T.serialize_checkpoint(c0)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
def test_reference_store_reads_our_commit(tmp_path, checkpoint_golden, golden_index):
    """Interoperability: the reference's own load_checkpoint replays a store
    our commit wrote (and our read_manifest reads the reference's)."""
    sys.path.insert(0, REF_SRC)
    try:
        from bitsnap import store as RS
    finally:
        sys.path.remove(REF_SRC)
    cfg = S.StoreConfig(tmp_path / "store", max_cached_iteration=2)
    for m, b in _golden(checkpoint_golden):
        S.commit(cfg, m, b)
    out = RS.load_checkpoint(RS.StoreConfig(tmp_path / "store", max_cached_iteration=2))
    _, c1 = _golden_ckpts(checkpoint_golden, golden_index["checkpoint"])
    assert out.iteration == 110
    assert [t.data for t in out.model_states] == [t.data for t in c1.model_states]
    rcfg = RS.StoreConfig(tmp_path / "ref", max_cached_iteration=2)
    (m0, b0), _ = _golden(checkpoint_golden)
    RS.commit(rcfg, RS.CheckpointManifest.from_bytes(m0.to_bytes()), b0)
    assert S.read_manifest(S.StoreConfig(tmp_path / "ref"), 100) == m0


def test_async_agent_persists_staged_blobs(tmp_path, checkpoint_golden):
    (m0, b0), (m1, b1) = _golden(checkpoint_golden)
    region = E.SlotRegion.create(tmp_path / "r.bssl", ranks=2, redundancy=2,
                                 capacity=len(b0) + 4096)
    region.stage(0, S.pack_blob(m0, b0), 100)
    region.stage(0, S.pack_blob(m1, b1), 110)
    region.stage(1, S.pack_blob(m0, b0), 100)
    agent = E.AsyncAgent(region, tmp_path / "stores", max_cached_iteration=2)
    assert agent.persist_once() == 3
    assert agent.errors == []
    assert all(s.state == E.STATE_PERSISTED for s in region.all_slots() if s.iteration)
    c0 = agent.rank_config(0)
    assert (c0.iter_dir(110) / "tensors.bin").read_bytes() == b1
    assert c0.tracker_path().read_text() == "110\n100\n"
    assert (agent.rank_config(1).iter_dir(100) / "tensors.bin").read_bytes() == b0
    # a corrupted slot stays VALID and is reported
    region.stage(1, S.pack_blob(m1, b1), 110)
    idx = [s.index for s in region.slots(1) if s.iteration == 110][0]
    off = region._slot_offset(1, idx) + E.SLOT_HEADER.size + 100
    region._mm[off] ^= 0xFF
    assert agent.persist_once() == 0
    assert "checksum mismatch" in agent.errors[-1]
    agent.start()
    agent.stop()
    region.close()


@pytest.mark.gpu
def test_save_and_load_through_store(dev, tmp_path, checkpoint_golden, golden_index):
    """save_checkpoint (GPU encode + commit) writes the reference store's
    bytes; load_checkpoint replays the chain on the GPU."""
    from oracle import bitsnap_oracle as O
    c0, c1 = _golden_ckpts(checkpoint_golden, golden_index["checkpoint"])
    (m0, b0), (m1, b1) = _golden(checkpoint_golden)
    for use_encoder in (False, True):
        root = tmp_path / f"s{int(use_encoder)}"
        cfg = S.StoreConfig(root, max_cached_iteration=2)
        enc = S.CheckpointEncoder(dev, clusters=16) if use_encoder else None
        assert S.save_checkpoint(cfg, c0, None, encoder=enc) == m0
        # with the resident encoder the delta needs no prev
        assert S.save_checkpoint(cfg, c1, None if use_encoder else c0, encoder=enc) == m1
        assert (cfg.iter_dir(100) / "tensors.bin").read_bytes() == b0
        assert (cfg.iter_dir(110) / "tensors.bin").read_bytes() == b1
        out = S.load_checkpoint(cfg)
        assert out.iteration == 110
        assert [t.data for t in out.model_states] == [t.data for t in c1.model_states]
        for a, b in zip(out.optimizer_states, c1.optimizer_states):
            x = np.frombuffer(b.data, np.float32)
            tab = O.cluster_fit(x, 16)
            p, c, _ = O.cluster_quantize(x, tab)
            assert a.data == O.cluster_dequantize(p, c, x.size, tab).astype("<f4").tobytes()
        assert [t.data for t in S.load_checkpoint(cfg, 100).model_states] == \
            [t.data for t in c0.model_states]
    # a failed delta save forces the next save to be a base (store.py:386-391)
    cfg = S.StoreConfig(tmp_path / "fail", max_cached_iteration=3)
    S.save_checkpoint(cfg, c0)
    with pytest.raises(S.MissingPreviousError):
        S.save_checkpoint(cfg, c1)          # delta without prev
    assert (cfg.root / ".needs_base").exists()
    assert S.save_checkpoint(cfg, c1).kind == S.KIND_BASE
    assert not (cfg.root / ".needs_base").exists()


@pytest.mark.gpu
def test_failed_commit_with_resident_encoder(dev, tmp_path, checkpoint_golden, golden_index,
                                             monkeypatch):
    """A resident encoder retains each saved checkpoint as its next delta
    base.  When the COMMIT of a base fails (disk full, ...), that base is on
    no disk, so the next save must be a base again — not a delta naming the
    uncommitted iteration as its base (load would hit MissingLinkError)."""
    c0, c1 = _golden_ckpts(checkpoint_golden, golden_index["checkpoint"])
    c2 = Checkpoint(iteration=120, model_states=c0.model_states,
                    optimizer_states=c0.optimizer_states)
    cfg = S.StoreConfig(tmp_path / "s", max_cached_iteration=1)   # every save a base
    enc = S.CheckpointEncoder(dev, clusters=16)
    assert S.save_checkpoint(cfg, c0, encoder=enc).kind == S.KIND_BASE

    def boom(*a, **k):
        raise OSError("no space left on device")
    with monkeypatch.context() as mp:
        mp.setattr(S, "write_tensors_bin", boom)
        with pytest.raises(OSError):
            S.save_checkpoint(cfg, c1, encoder=enc)       # base 110: encoded, not committed
    assert enc.prev is None
    assert (cfg.root / ".needs_base").exists()
    monkeypatch.setenv("MAX_CACHED_ITERATION", "3")       # the policy would now pick a delta
    m = S.save_checkpoint(cfg, c2, encoder=enc)
    assert m.kind == S.KIND_BASE and m.base_iteration == 120
    out = S.load_checkpoint(cfg)
    assert out.iteration == 120
    assert [t.data for t in out.model_states] == [t.data for t in c0.model_states]


@pytest.mark.gpu
@pytest.mark.parametrize("point", ["store.dir.tensors-written", "store.dir.manifest-written",
                                   "store.dir.type-written", "store.dir.renamed",
                                   "store.tracker.temp-written"])
def test_crash_during_save_leaves_store_loadable(dev, tmp_path, checkpoint_golden, golden_index,
                                                 point):
    """faults.py crash points in the save pipeline (store.py:339-371,
    181-187): a delta save crashing at any of them, then recover_scan, leaves
    the store loading the last committed checkpoint bit for bit."""
    from paper_2511_12376_b200 import faults
    c0, c1 = _golden_ckpts(checkpoint_golden, golden_index["checkpoint"])
    cfg = S.StoreConfig(tmp_path / "s", max_cached_iteration=3)
    S.save_checkpoint(cfg, c0)
    faults.crash_at(point)
    try:
        with pytest.raises(faults.CrashPoint):
            S.save_checkpoint(cfg, c1, prev=c0)
    finally:
        faults.clear()
    actions = S.recover_scan(cfg)
    assert all(a.startswith(("removed temp", "pruned uncommitted")) for a in actions)
    out = S.load_checkpoint(cfg)
    assert out.iteration == 100
    assert [t.data for t in out.model_states] == [t.data for t in c0.model_states]


@pytest.mark.gpu
def test_inspect_and_prune_above(dev, tmp_path, checkpoint_golden, golden_index):
    """store.py:480-503, 533-553 over a three-link chain saved by the GPU
    encoder: inspect lists it, prune_above removes the newest link and
    repairs the tracker, the store then loads the middle link."""
    c0, c1 = _golden_ckpts(checkpoint_golden, golden_index["checkpoint"])
    c2 = Checkpoint(iteration=120, model_states=c0.model_states,
                    optimizer_states=c0.optimizer_states)
    cfg = S.StoreConfig(tmp_path / "s", max_cached_iteration=5)
    enc = S.CheckpointEncoder(dev, clusters=16)
    assert [S.save_checkpoint(cfg, c, encoder=enc).kind for c in (c0, c1, c2)] == \
        [S.KIND_BASE, S.KIND_DELTA, S.KIND_DELTA]
    info = S.inspect(cfg)
    assert info["tracker"] == {"latest_iteration": 120, "latest_base_iteration": 100}
    assert [(c["iteration"], c["kind"], c["base_iteration"]) for c in info["checkpoints"]] == \
        [(100, "base", 100), (110, "delta", 100), (120, "delta", 110)]
    assert all(c["tensors_bytes"] == (cfg.iter_dir(c["iteration"]) / "tensors.bin").stat().st_size
               for c in info["checkpoints"])
    assert S.prune_above(cfg, 110) == [120]
    assert S.read_tracker(cfg) == S.TrackerState(110, 100)
    out = S.load_checkpoint(cfg)
    assert out.iteration == 110
    assert [t.data for t in out.model_states] == [t.data for t in c1.model_states]
