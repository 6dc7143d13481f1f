"""Staging slot region and recovery consensus.

Mirrors the producer half of /root/reference/pkg/src/bitsnap/engine.py:

  * `SlotRegion` — the memory-mapped BSSL file holding K fixed-capacity slots
    per rank (engine.py:27-37 layout, 96-244 behaviour): same header structs,
    slot states, eviction policy (first EMPTY slot, else the oldest PERSISTED
    one, else BackpressureError), stale-iteration and capacity checks, and the
    blake2b-64 checksum (engine.py:60-64) recorded when a slot turns VALID.
    A region written here is byte-identical to the reference's for the same
    sequence of calls, so the reference's AsyncAgent can drain it.
  * `SlotRegion.stage_checkpoint` — the B200 hand-off: the GPU encoder's
    output (store.CheckpointEncoder) lands straight in the slot's payload
    bytes, in the staging-blob layout of store.py:275-286 (header, manifest,
    tensors.bin); no host-side copy of the blob is made.  A tmpfs mapping
    (/dev/shm) is page-locked with cudaHostRegister so the copies are DMA; a
    disk-backed mapping cannot be registered and the copies go through the
    driver's staging buffer (same bytes, ~4x slower).  Only the checksum
    runs on the host, over the mapped bytes, as the format requires.
  * `gather_valid` / `recover` — the recovery consensus of engine.py:291-380
    with the simulated all-gather replaced by torch.distributed all-gathers
    of every rank's valid-iteration set (NCCL on GPUs, gloo on CPU): the
    newest iteration valid on every rank, else ColdStartError.  Each rank
    clears its own slots newer than the chosen iteration; pruning the
    on-disk store is the store's lifecycle (out of scope).
"""

from __future__ import annotations

import hashlib
import mmap
import struct
import threading
from dataclasses import dataclass, field
from pathlib import Path

import torch

from . import faults

REGION_MAGIC = b"BSSL"
REGION_VERSION = 1
REGION_HEADER = struct.Struct("<4sHIIQ")  # magic, version, ranks, K, capacity
SLOT_HEADER = struct.Struct("<BQQQ")  # state, iteration, length, checksum

STATE_EMPTY = 0
STATE_WRITING = 1
STATE_VALID = 2
STATE_PERSISTED = 3
STATE_NAMES = {0: "EMPTY", 1: "WRITING", 2: "VALID", 3: "PERSISTED"}


class EngineError(RuntimeError):
    """engine.py:40."""


class StaleIterationError(EngineError):
    """engine.py:44."""


class BackpressureError(EngineError):
    """engine.py:48: all slots are pending persist; caller must wait."""


class PayloadTooLargeError(EngineError):
    """engine.py:52."""


class ColdStartError(EngineError):
    """engine.py:56: no iteration is valid on every rank."""


def checksum(payload) -> int:
    """engine.py:60-64: 64-bit blake2b digest of a staged payload."""
    return int.from_bytes(hashlib.blake2b(payload, digest_size=8).digest(), "little")


EMPTY_CHECKSUM = checksum(b"")


@dataclass(frozen=True)
class SlotInfo:
    """engine.py:72-84."""

    rank: int
    index: int
    state: int
    iteration: int
    length: int
    checksum: int

    @property
    def state_name(self) -> str:
        return STATE_NAMES.get(self.state, f"?{self.state}")


@dataclass(frozen=True)
class RankReport:
    """engine.py:87-90."""

    rank: int
    latest_valid_iteration: int | None


def _host_register(ptr: int, nbytes: int) -> bool:
    """Page-lock an existing host range for DMA (bsnp_host_register: a
    refusal leaves no pending CUDA error behind for later launches)."""
    if nbytes == 0 or not torch.cuda.is_available():
        return False
    from . import _runtime as rt
    return rt.lib().bsnp_host_register(ptr, nbytes) == 0


def _host_unregister(ptr: int) -> None:
    from . import _runtime as rt
    rt.lib().bsnp_host_unregister(ptr)


class SlotRegion:
    """K fixed-capacity checkpoint slots per rank in a memory-mapped file
    (engine.py:96-244)."""

    def __init__(self, path: Path, file, mm, ranks: int, redundancy: int, capacity: int):
        self.path = Path(path)
        self._file = file
        self._mm = mm
        self.ranks = ranks
        self.redundancy = redundancy
        self.capacity = capacity
        self._lock = threading.Lock()
        self._view = None        # uint8 tensor over the mapping (device staging)
        self._registered = None  # base address page-locked with cudaHostRegister

    # ---- lifecycle (engine.py:109-143)
    @classmethod
    def create(cls, path, ranks: int, redundancy: int, capacity: int) -> "SlotRegion":
        if ranks < 1 or redundancy < 1 or capacity < 1:
            raise EngineError("ranks, redundancy and capacity must be >= 1")
        path = Path(path)
        slot_bytes = SLOT_HEADER.size + capacity
        total = REGION_HEADER.size + ranks * redundancy * slot_bytes
        with open(path, "wb") as f:
            f.write(REGION_HEADER.pack(REGION_MAGIC, REGION_VERSION, ranks, redundancy,
                                       capacity))
            f.truncate(total)  # zero-filled, like the reference's explicit zeros
        return cls.open(path)

    @classmethod
    def open(cls, path) -> "SlotRegion":
        path = Path(path)
        f = open(path, "r+b")
        mm = mmap.mmap(f.fileno(), 0)
        magic, version, ranks, redundancy, capacity = REGION_HEADER.unpack_from(mm, 0)
        if magic != REGION_MAGIC:
            mm.close()
            f.close()
            raise EngineError(f"bad slot-region magic {magic!r}")
        if version != REGION_VERSION:
            mm.close()
            f.close()
            raise EngineError(f"unsupported slot-region version {version}")
        return cls(path, f, mm, ranks, redundancy, capacity)

    def close(self) -> None:
        if self._registered is not None:
            _host_unregister(self._registered)
            self._registered = None
        self._view = None
        self._mm.close()
        self._file.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- slot addressing (engine.py:147-187)
    def _slot_offset(self, rank: int, index: int) -> int:
        slot_bytes = SLOT_HEADER.size + self.capacity
        return REGION_HEADER.size + (rank * self.redundancy + index) * slot_bytes

    def slot(self, rank: int, index: int) -> SlotInfo:
        state, iteration, length, digest = SLOT_HEADER.unpack_from(
            self._mm, self._slot_offset(rank, index))
        return SlotInfo(rank, index, state, iteration, length, digest)

    def slots(self, rank: int) -> list:
        return [self.slot(rank, i) for i in range(self.redundancy)]

    def all_slots(self) -> list:
        return [s for r in range(self.ranks) for s in self.slots(r)]

    def payload(self, rank: int, index: int) -> bytes:
        info = self.slot(rank, index)
        off = self._slot_offset(rank, index) + SLOT_HEADER.size
        return bytes(self._mm[off:off + info.length])

    def payload_view(self, rank: int, index: int) -> memoryview:
        """The slot's payload bytes without a copy."""
        info = self.slot(rank, index)
        off = self._slot_offset(rank, index) + SLOT_HEADER.size
        return memoryview(self._mm)[off:off + info.length]

    def _write_header(self, rank, index, state, iteration, length, digest) -> None:
        SLOT_HEADER.pack_into(self._mm, self._slot_offset(rank, index), state, iteration,
                              length, digest)

    def set_state(self, rank: int, index: int, state: int) -> None:
        info = self.slot(rank, index)
        self._write_header(rank, index, state, info.iteration, info.length, info.checksum)

    def clear_slot(self, rank: int, index: int) -> None:
        self._write_header(rank, index, STATE_EMPTY, 0, 0, 0)

    def verify(self, rank: int, index: int) -> bool:
        info = self.slot(rank, index)
        if info.state not in (STATE_VALID, STATE_PERSISTED):
            return False
        return checksum(self.payload_view(rank, index)) == info.checksum

    # ---- producer side (engine.py:191-235)
    def _claim(self, rank: int, length: int, iteration: int) -> int:
        """Slot choice of engine.py:204-226 (caller holds the lock): marks the
        slot WRITING and returns its index."""
        if length > self.capacity:
            raise PayloadTooLargeError(
                f"payload of {length} bytes exceeds slot capacity {self.capacity}")
        slots = self.slots(rank)
        staged = [s for s in slots if s.state != STATE_EMPTY]
        if staged and iteration <= max(s.iteration for s in staged):
            raise StaleIterationError(
                f"rank {rank}: iteration {iteration} is not newer than "
                f"staged {max(s.iteration for s in staged)}")
        empty = [s for s in slots if s.state == STATE_EMPTY]
        if empty:
            target = empty[0]
        else:
            persisted = [s for s in slots if s.state == STATE_PERSISTED]
            if not persisted:
                raise BackpressureError(
                    f"rank {rank}: all {self.redundancy} slots pending persist")
            target = min(persisted, key=lambda s: s.iteration)
        self._write_header(rank, target.index, STATE_WRITING, iteration, length, 0)
        return target.index

    def _seal(self, rank: int, idx: int, iteration: int, length: int) -> SlotInfo:
        faults.trip("engine.stage.slot-written")
        digest = checksum(self.payload_view(rank, idx)[:length])
        self._write_header(rank, idx, STATE_VALID, iteration, length, digest)
        faults.trip("engine.stage.slot-valid")
        return self.slot(rank, idx)

    def stage(self, rank: int, payload: bytes, iteration: int) -> SlotInfo:
        """engine.py:191-235: copy a compressed checkpoint into a slot and mark
        it VALID (with its checksum)."""
        if len(payload) > self.capacity:
            raise PayloadTooLargeError(
                f"payload of {len(payload)} bytes exceeds slot capacity {self.capacity}")
        with self._lock:
            idx = self._claim(rank, len(payload), iteration)
            off = self._slot_offset(rank, idx) + SLOT_HEADER.size
            self._mm[off:off + len(payload)] = payload
            return self._seal(rank, idx, iteration, len(payload))

    def _tensor_view(self) -> torch.Tensor:
        """uint8 tensor over the whole mapping, page-locked when possible so
        device-to-host copies land in it by DMA."""
        if self._view is None:
            view = torch.frombuffer(self._mm, dtype=torch.uint8)
            if self._registered is None and _host_register(view.data_ptr(), view.numel()):
                self._registered = view.data_ptr()
            self._view = view
        return self._view

    @property
    def dma_ready(self) -> bool:
        """True once the mapping is page-locked (copies into it are DMA)."""
        self._tensor_view()
        return self._registered is not None

    def stage_checkpoint(self, rank: int, encoder, ckpt, prev, kind: str):
        """Encode `ckpt` on the GPU (store.CheckpointEncoder) and stage it as
        the staging blob of store.py:275-286 — identical bytes to
        `stage(rank, pack_blob(*encode_checkpoint(...)), ckpt.iteration)`.
        The encoded records land straight in the slot; the slot is WRITING
        until the checksum is recorded.  Returns (SlotInfo, manifest)."""
        from . import store as S
        view = self._tensor_view()
        claimed = {}

        def dest(manifest, nbytes):
            mbytes = manifest.to_bytes()
            head = S.blob_header(manifest, mbytes, nbytes) + mbytes
            total = len(head) + nbytes
            with self._lock:
                idx = self._claim(rank, total, ckpt.iteration)
            claimed.update(idx=idx, total=total)
            off = self._slot_offset(rank, idx) + SLOT_HEADER.size
            self._mm[off:off + len(head)] = head
            return view[off + len(head):off + total]

        try:
            manifest, _ = encoder.encode_into(ckpt, prev, kind, dest)
        except BaseException:
            # a failed copy (e.g. out of device memory) must not leave the
            # slot WRITING for good: _claim never reuses such a slot
            if "idx" in claimed:
                with self._lock:
                    self.clear_slot(rank, claimed["idx"])
            raise
        with self._lock:
            info = self._seal(rank, claimed["idx"], ckpt.iteration, claimed["total"])
        return info, manifest


def rank_store(parent_root, rank: int, **cfg_kwargs):
    """engine.py:230-232: each rank persists into its own store root."""
    from .fsstore import StoreConfig
    return StoreConfig(root=Path(parent_root) / f"rank_{rank:02d}", **cfg_kwargs)


class AsyncAgent:
    """engine.py:235-306: the background consumer that persists VALID slots
    through the store (unpack_blob + commit, oldest iteration first per rank;
    a failed commit keeps the slot VALID for a retry and is recorded in
    `errors`).  Pure host work: the codec ran when the slot was staged."""

    def __init__(self, region: SlotRegion, store_root, poll_interval: float = 0.01,
                 **store_kwargs):
        self.region = region
        self.store_root = Path(store_root)
        self.poll_interval = poll_interval
        self.store_kwargs = store_kwargs
        self.errors: list = []
        self._stop = threading.Event()
        self._thread = None

    def rank_config(self, rank: int):
        return rank_store(self.store_root, rank, **self.store_kwargs)

    def persist_once(self) -> int:
        from . import store as S
        done = 0
        for rank in range(self.region.ranks):
            pending = sorted((s for s in self.region.slots(rank) if s.state == STATE_VALID),
                             key=lambda s: s.iteration)
            for info in pending:
                if not self.region.verify(rank, info.index):
                    self.errors.append(f"rank {rank} iteration {info.iteration}: "
                                       "checksum mismatch")
                    continue
                try:
                    manifest, tensors = S.unpack_blob(self.region.payload(rank, info.index))
                    S.commit(self.rank_config(rank), manifest, tensors)
                    faults.trip("engine.persist.committed")
                except faults.CrashPoint:
                    raise
                except Exception as exc:  # keep the slot VALID for a retry
                    self.errors.append(f"rank {rank} iteration {info.iteration}: {exc}")
                    continue
                self.region.set_state(rank, info.index, STATE_PERSISTED)
                done += 1
        return done

    def persist_loop(self) -> None:
        while not self._stop.is_set():
            if self.persist_once() == 0:
                self._stop.wait(self.poll_interval)

    def start(self) -> None:
        self._stop.clear()
        self._thread = threading.Thread(target=self.persist_loop, daemon=True)
        self._thread.start()

    def stop(self) -> None:
        self._stop.set()
        if self._thread is not None:
            self._thread.join()
            self._thread = None

    def drain(self, timeout: float = 30.0) -> None:
        import time
        deadline = time.monotonic() + timeout
        while time.monotonic() < deadline:
            if not any(s.state == STATE_VALID for s in self.region.all_slots()):
                return
            time.sleep(0.002)
        raise EngineError("timed out waiting for agent to drain slots")


def status_report(region: SlotRegion) -> str:
    """engine.py:383-393."""
    lines = [f"slot region {region.path}: {region.ranks} ranks x "
             f"{region.redundancy} slots, capacity {region.capacity} bytes"]
    for s in region.all_slots():
        lines.append(f"rank {s.rank} slot {s.index}: {s.state_name:9s} "
                     f"iteration={s.iteration} length={s.length}")
    return "\n".join(lines)


# ---------------------------------------------------------------------------
# recovery consensus over torch.distributed (engine.py:291-380)
# ---------------------------------------------------------------------------

def region_valid_iterations(region: SlotRegion, rank: int) -> set:
    """The memory half of engine.py:302-317: iterations of this rank's VALID or
    PERSISTED slots whose checksum verifies."""
    return {s.iteration for s in region.slots(rank)
            if s.state in (STATE_VALID, STATE_PERSISTED) and region.verify(rank, s.index)}


def gather_valid(valid, group=None) -> list:
    """All-gather every rank's set of valid iterations (the reference's
    simulated all-gather, engine.py:291-299): two collectives — the counts,
    then the sets padded to the largest count.  NCCL gathers device tensors,
    gloo host tensors.  Returns a list of sets indexed by rank."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    mine = sorted(int(v) for v in valid)
    cnt = torch.tensor([len(mine)], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    width = max(1, max(int(c.item()) for c in counts))
    row = torch.full((width,), -1, dtype=torch.int64, device=dev)
    if mine:
        row[:len(mine)] = torch.tensor(mine, dtype=torch.int64, device=dev)
    rows = torch.empty(world * width, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(rows, row, group=group)
    rows = rows.view(world, width).cpu().tolist()
    return [set(r[:int(c.item())]) for r, c in zip(rows, counts)]


@dataclass
class RecoveryDecision:
    """engine.py:320-325."""

    chosen_iteration: int
    reports: list
    pruned: list = field(default_factory=list)  # (rank, iteration)
    trace: list = field(default_factory=list)


def decide(per_rank: list) -> RecoveryDecision:
    """The consensus of engine.py:328-351 from every rank's valid set: the
    newest iteration valid on all ranks, else ColdStartError.  Trace lines as
    the reference's."""
    reports = [RankReport(r, max(v) if v else None) for r, v in enumerate(per_rank)]
    trace = ["all-gather reports: " + " ".join(
        f"rank{r.rank}=" + ("none" if r.latest_valid_iteration is None
                            else str(r.latest_valid_iteration))
        for r in reports)]
    common = set.intersection(*per_rank) if per_rank else set()
    if not common:
        trace.append("no iteration valid on all ranks: cold start")
        raise ColdStartError("no iteration is valid on every rank")
    chosen = max(common)
    trace.append(f"consensus iteration: {chosen}")
    return RecoveryDecision(chosen, reports, [], trace)


def valid_iterations(region: SlotRegion, store_root, rank: int) -> set:
    """engine.py:319-333: this rank's verified VALID / PERSISTED slots plus
    the iterations its on-disk store holds up to the tracker's latest."""
    from . import fsstore as F
    valid = region_valid_iterations(region, rank)
    cfg = rank_store(store_root, rank)
    tracker = F.try_read_tracker(cfg)
    if tracker is not None:
        valid.update(it for it in F.list_iterations(cfg) if it <= tracker.latest_iteration)
    return valid


def gather_reports(region: SlotRegion, store_root) -> list:
    """engine.py:309-316: the reference's simulated all-gather in one process
    (every rank's newest valid iteration); `gather_valid` is the real one."""
    reports = []
    for rank in range(region.ranks):
        valid = valid_iterations(region, store_root, rank)
        reports.append(RankReport(rank, max(valid) if valid else None))
    return reports


def recover(reports: list, region: SlotRegion, store_root) -> RecoveryDecision:
    """engine.py:344-380 (same signature, decision, pruning and trace): the
    newest iteration every rank holds, everything newer cleared from every
    rank's slots and pruned from its store.  ColdStartError without one."""
    from . import fsstore as F
    per_rank = [valid_iterations(region, store_root, r) for r in range(region.ranks)]
    d = decide(per_rank)
    d.reports = list(reports)
    d.trace[0] = "all-gather reports: " + " ".join(
        f"rank{r.rank}=" + ("none" if r.latest_valid_iteration is None
                            else str(r.latest_valid_iteration))
        for r in sorted(reports, key=lambda r: r.rank))
    pruned = []
    for rank in range(region.ranks):
        for sl in region.slots(rank):
            if sl.state != STATE_EMPTY and sl.iteration > d.chosen_iteration:
                region.clear_slot(rank, sl.index)
                pruned.append((rank, sl.iteration))
        for it in F.prune_above(rank_store(store_root, rank), d.chosen_iteration):
            pruned.append((rank, it))
    d.pruned = sorted(set(pruned))
    for rank, it in d.pruned:
        d.trace.append(f"pruned iteration {it} on rank {rank}")
    d.trace.append(f"recovering from iteration {d.chosen_iteration}")
    return d


def recover_dist(region: SlotRegion, rank: int, group=None, store_root=None,
                 extra_valid=()) -> RecoveryDecision:
    """`recover` for one rank of a torch.distributed job (one process per
    GPU): gather the valid sets over the process group (`gather_valid`: this
    rank's verified slots, its on-disk store when `store_root` is given, and
    `extra_valid`), decide, and clear this rank's slots (and prune its store)
    newer than the chosen iteration."""
    from . import fsstore as F
    valid = (valid_iterations(region, store_root, rank) if store_root is not None
             else region_valid_iterations(region, rank))
    valid |= set(int(v) for v in extra_valid)
    d = decide(gather_valid(valid, group))
    for sl in region.slots(rank):
        if sl.state != STATE_EMPTY and sl.iteration > d.chosen_iteration:
            region.clear_slot(rank, sl.index)
            d.pruned.append((rank, sl.iteration))
    if store_root is not None:
        for it in F.prune_above(rank_store(store_root, rank), d.chosen_iteration):
            d.pruned.append((rank, it))
    for r, it in sorted(set(d.pruned)):
        d.trace.append(f"pruned iteration {it} on rank {r}")
    d.trace.append(f"recovering from iteration {d.chosen_iteration}")
    return d
