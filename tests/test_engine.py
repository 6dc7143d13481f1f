"""Staging slot region and recovery consensus
against the reference's own engine, run here by
tests/golden/make_engine_golden.py: the same scripted SlotRegion calls must
give the same outcomes, slot table, status report and region file bytes;
the staging blob of the golden checkpoint must give the same file; the
recovery decisions (consensus and cold start) must match, and the
torch.distributed consensus (gloo, world 2) must agree with them.  GPU: the
device hand-off (encoder output DMA'd into the mapped slot) must write the
same file as staging the reference's blob."""

import hashlib
import json
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_12376_b200 import engine as E
from paper_2511_12376_b200 import store as S

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def eg():
    with open(os.path.join(GOLDEN, "engine_golden.json")) as f:
        return json.load(f)


def run_script(region, script):
    out = []
    for op, *a in script:
        try:
            if op == "stage":
                s = region.stage(a[0], bytes.fromhex(a[1]), a[2])
                out.append(["ok", s.rank, s.index, s.state, s.iteration, s.length,
                            str(s.checksum)])
            elif op == "set_state":
                region.set_state(*a)
                out.append(["ok"])
            elif op == "clear":
                region.clear_slot(*a)
                out.append(["ok"])
            elif op == "verify":
                out.append(["ok", bool(region.verify(*a))])
        except E.EngineError as exc:
            out.append(["raise", type(exc).__name__])
    return out


def test_slot_region_script_matches_reference(eg, tmp_path):
    path = tmp_path / "script.bssl"
    region = E.SlotRegion.create(path, **eg["region"])
    got = run_script(region, eg["script"])
    want = eg["script_out"]
    assert got == want["results"]
    assert [[s.rank, s.index, s.state, s.iteration, s.length, str(s.checksum)]
            for s in region.all_slots()] == want["slots"]
    assert E.status_report(region).split("\n")[1:] == want["status"]
    region.close()
    assert path.read_bytes().hex() == want["file_hex"]
    # reopen: header parsed back
    with E.SlotRegion.open(path) as r2:
        assert (r2.ranks, r2.redundancy, r2.capacity) == (2, 2, 48)
        assert r2.verify(0, 0) and r2.payload(0, 0) == b"third"


def test_region_checks(eg, tmp_path):
    assert str(E.EMPTY_CHECKSUM) == eg["empty_checksum"]
    with pytest.raises(E.EngineError, match=">= 1"):
        E.SlotRegion.create(tmp_path / "a", 0, 1, 1)
    bad = tmp_path / "bad"
    bad.write_bytes(b"XXXX" + bytes(40))
    with pytest.raises(E.EngineError, match="magic"):
        E.SlotRegion.open(bad)
    ver = tmp_path / "ver"
    ver.write_bytes(E.REGION_HEADER.pack(b"BSSL", 9, 1, 1, 4) + bytes(64))
    with pytest.raises(E.EngineError, match="version"):
        E.SlotRegion.open(ver)


def test_staging_blob_matches_reference(eg, checkpoint_golden, tmp_path):
    g = checkpoint_golden
    man = S.CheckpointManifest.from_bytes(g["manifest1"].tobytes())
    blob = S.pack_blob(man, g["blob1"].tobytes())
    cs = eg["checkpoint_stage"]
    assert len(blob) == cs["blob_len"]
    m2, t2 = S.unpack_blob(blob)
    assert m2 == man and bytes(t2) == g["blob1"].tobytes()
    path = tmp_path / "ckpt.bssl"
    with E.SlotRegion.create(path, 1, 2, cs["capacity"]) as region:
        s = region.stage(0, blob, man.iteration)
        assert str(s.checksum) == cs["checksum"]
    assert hashlib.sha256(path.read_bytes()).hexdigest() == cs["file_sha256"]
    with pytest.raises(S.StoreError, match="truncated"):
        S.unpack_blob(blob[:-1])
    with pytest.raises(S.StoreError, match="magic"):
        S.unpack_blob(b"NOPE" + blob[4:])


def test_blob_bound_covers_reference_blobs(checkpoint_golden, golden_index):
    """store.blob_bound (the caller-buffer size of a pipelined save) is an
    upper bound of the reference's base and delta blobs of the golden
    checkpoint, and tight for the quantized optimizer records."""
    from test_store_gpu import _golden_ckpts
    g = checkpoint_golden
    c0, c1 = _golden_ckpts(g, golden_index["checkpoint"])
    for ck, blob in ((c0, g["blob0"]), (c1, g["blob1"])):
        bound = S.blob_bound(ck)
        assert blob.size <= bound
        opt = sum(t.num_elements for t in ck.optimizer_states)
        assert bound < sum(t.nbytes for t in ck.model_states) + 1.5 * opt + 600 * (
            len(ck.model_states) + len(ck.optimizer_states))


def _consensus_region(path):
    region = E.SlotRegion.create(path, ranks=2, redundancy=3, capacity=16)
    region.stage(0, b"r0-it3", 3)
    region.stage(0, b"r0-it4", 4)
    region.stage(1, b"r1-it3", 3)
    s = region.stage(1, b"r1-it4", 4)
    off = region._slot_offset(1, s.index) + E.SLOT_HEADER.size
    region._mm[off] ^= 0xFF          # a corrupt copy: fails verify
    return region


def test_recovery_decision_matches_reference(eg, tmp_path):
    want = eg["recovery"]["consensus"]
    region = _consensus_region(tmp_path / "r1.bssl")
    root = tmp_path / "stores"            # the ranks' on-disk stores: empty
    # the reference's single-process entry points (engine.py:309-380)
    reports = E.gather_reports(region, root)
    assert [(r.rank, r.latest_valid_iteration) for r in reports] == [(0, 4), (1, 3)]
    d = E.recover(reports, region, root)
    assert d.chosen_iteration == want["chosen"]
    assert [list(p) for p in sorted(set(d.pruned))] == want["pruned"]
    assert d.trace == want["trace"]
    assert [[x.rank, x.index, x.state, x.iteration] for x in region.all_slots()] == want["slots"]
    region.close()
    cold = eg["recovery"]["cold"]
    with pytest.raises(E.ColdStartError, match=cold["message"]):
        E.decide([{5}, {6}])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _recover_worker(rank, world, port, path, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        region = E.SlotRegion.open(path)
        d = E.recover_dist(region, rank)
        q.put((rank, d.chosen_iteration, d.pruned, d.trace,
               [[x.index, x.state, x.iteration] for x in region.slots(rank)]))
        region.close()
        try:
            E.decide(E.gather_valid({10 + rank}))
            q.put((rank, "no-raise"))
        except E.ColdStartError:
            q.put((rank, "cold"))
    finally:
        dist.destroy_process_group()


def test_recover_over_torch_distributed(eg, tmp_path):
    """Two ranks (gloo) share the region file; each gathers the valid sets,
    agrees on iteration 3 and clears its own newer slot."""
    want = eg["recovery"]["consensus"]
    path = str(tmp_path / "shared.bssl")
    _consensus_region(path).close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_recover_worker, args=(r, 2, port, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(4)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dec = {r[0]: r for r in res if len(r) == 5}
    cold = {r[0]: r[1] for r in res if len(r) == 2}
    assert cold == {0: "cold", 1: "cold"}
    for rank in (0, 1):
        _, chosen, pruned, trace, slots = dec[rank]
        assert chosen == want["chosen"]
        assert pruned == [(rank, 4)]
        assert trace[:2] == want["trace"][:2]
        assert trace[-1] == want["trace"][-1]
        assert f"pruned iteration 4 on rank {rank}" in trace
    with E.SlotRegion.open(path) as region:
        assert [[x.rank, x.index, x.state, x.iteration] for x in region.all_slots()] == \
            want["slots"]


@pytest.mark.gpu
def test_device_stage_checkpoint_matches_reference(eg, dev, checkpoint_golden, golden_index,
                                                   tmp_path):
    """The encoder's records DMA'd into the page-locked slot: the region
    file equals the one the reference writes when staging its own blob."""
    from test_store_gpu import _golden_ckpts
    g, meta = checkpoint_golden, golden_index["checkpoint"]
    c0, c1 = _golden_ckpts(g, meta)
    cs = eg["checkpoint_stage"]
    # tmpfs mappings can be page-locked (DMA); a disk-backed one cannot, and
    # the copies then go through the driver's staging (same bytes)
    shm = os.path.isdir("/dev/shm")
    path = (tmp_path if not shm else
            __import__("pathlib").Path(tempfile.mkdtemp(dir="/dev/shm"))) / "ckpt.bssl"
    enc = S.CheckpointEncoder(dev, clusters=16)
    enc.encode(c0, None, S.KIND_BASE)              # c0 stays resident as the delta base
    with E.SlotRegion.create(path, 1, 2, cs["capacity"]) as region:
        if shm:
            assert region.dma_ready
        info, man = region.stage_checkpoint(0, enc, c1, None, S.KIND_DELTA)
        assert info.state == E.STATE_VALID and info.length == cs["blob_len"]
        assert str(info.checksum) == cs["checksum"] and region.verify(0, info.index)
        m2, tb = S.unpack_blob(region.payload(0, info.index))
        assert m2.to_bytes() == g["manifest1"].tobytes() and bytes(tb) == g["blob1"].tobytes()
        with pytest.raises(E.StaleIterationError):
            region.stage_checkpoint(0, enc, c1, c0, S.KIND_DELTA)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == cs["file_sha256"]
    path.unlink()
    if shm:
        path.parent.rmdir()
    # a disk-backed region: no page-locking, same bytes
    with E.SlotRegion.create(tmp_path / "disk.bssl", 1, 2, cs["capacity"]) as region:
        info, _ = region.stage_checkpoint(0, enc, c1, c0, S.KIND_DELTA)
        m2, tb = S.unpack_blob(region.payload(0, info.index))
        assert bytes(tb) == g["blob1"].tobytes()


def _store_recovery_setup(root, region_path, checkpoint_golden):
    """Rank 0's store holds the golden base (100) and delta (110), rank 1's
    only the base; rank 0 also stages 120 in memory."""
    from paper_2511_12376_b200 import store as S
    g = checkpoint_golden
    links = [(S.CheckpointManifest.from_bytes(g[f"manifest{i}"].tobytes()), g[f"blob{i}"].tobytes())
             for i in (0, 1)]
    for rank, n in ((0, 2), (1, 1)):
        cfg = E.rank_store(root, rank)
        for m, b in links[:n]:
            S.commit(cfg, m, b)
    region = E.SlotRegion.create(region_path, ranks=2, redundancy=2, capacity=16)
    region.stage(0, b"r0-it120", 120)
    return region


def test_recover_prunes_disk_like_reference(tmp_path, checkpoint_golden):
    """engine.recover with on-disk stores (engine.py:319-380 + store.py:533-553):
    the consensus counts each rank's committed iterations, and everything
    newer is cleared from the slots AND pruned from the stores, the tracker
    repaired to the newest remaining checkpoint and its base."""
    root = tmp_path / "ours"
    region = _store_recovery_setup(root, tmp_path / "ours.bssl", checkpoint_golden)
    reports = E.gather_reports(region, root)
    assert [(r.rank, r.latest_valid_iteration) for r in reports] == [(0, 120), (1, 100)]
    d = E.recover(reports, region, root)
    assert d.chosen_iteration == 100
    assert d.pruned == [(0, 110), (0, 120)]
    assert d.trace[-3:] == ["pruned iteration 110 on rank 0", "pruned iteration 120 on rank 0",
                            "recovering from iteration 100"]
    cfg0 = E.rank_store(root, 0)
    assert cfg0.tracker_path().read_text() == "100\n100\n"
    assert [p.name for p in sorted(cfg0.root.iterdir()) if p.name.startswith("iter_")] == \
        ["iter_0000100"]
    assert all(s.state == E.STATE_EMPTY for s in region.slots(0))
    region.close()
    if not os.path.isdir("/root/reference/pkg/src"):
        return
    # the reference's own recover on the same setup: same decision and trace
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from bitsnap import engine as RE
    rroot = tmp_path / "ref"
    _store_recovery_setup(rroot, tmp_path / "ref.bssl", checkpoint_golden).close()
    rregion = RE.SlotRegion.open(tmp_path / "ref.bssl")
    rd = RE.recover(RE.gather_reports(rregion, rroot), rregion, rroot)
    assert rd.chosen_iteration == d.chosen_iteration
    assert [tuple(p) for p in rd.pruned] == d.pruned
    assert rd.trace == d.trace
    assert (rroot / "rank_00" / "latest_checkpointed_iteration.txt").read_text() == "100\n100\n"
    rregion.close()
