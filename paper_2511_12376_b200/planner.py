"""Shard planner: each GPU encodes its own parameter shard; one all-gather
of a small int64 size table gives every rank the global record offsets.

The reference has no planner: its closest analogues are the
per-tensor offset accumulation of store.encode_checkpoint (store.py:236-247),
the per-rank stores (engine.py:230-232) and the simulated all-gather
(engine.py:309-316).  Here:

  1. `plan_shards` — deterministic LPT bin-packing of tensors by raw bytes
     onto G ranks (every rank computes the same plan locally, no traffic);
  2. each rank encodes its tensors on its own GPU (no data-path collective);
  3. `exchange_sizes` — ONE `all_gather_into_tensor` of rows
     (global_id, codec, count, encoded_bytes), padded to the plan's maximum
     row count per rank (NCCL over NVLink on the box, gloo in CPU tests);
  4. `global_offsets` — exclusive prefix of encoded bytes in checkpoint
     order, i.e. exactly the offsets the single-process driver assigns, so the
     concatenated tensors.bin is byte-identical to store.encode_checkpoint's.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

import torch

CODEC_RAW, CODEC_DELTA, CODEC_QUANT = 0, 1, 2
CODEC_NAMES = {CODEC_RAW: "RAW", CODEC_DELTA: "DELTA", CODEC_QUANT: "QUANT"}
ROW = 4  # (global_id, codec, count, encoded_bytes)


@dataclass(frozen=True)
class ShardPlan:
    world: int
    owner: tuple          # owner[global_id] = rank
    load: tuple           # raw bytes per rank

    def local_ids(self, rank: int) -> list:
        return [i for i, r in enumerate(self.owner) if r == rank]

    @property
    def max_rows(self) -> int:
        counts = [0] * self.world
        for r in self.owner:
            counts[r] += 1
        return max(counts) if counts else 0

    @property
    def imbalance(self) -> float:
        mean = sum(self.load) / max(1, self.world)
        return max(self.load) / mean if mean else 1.0


def plan_shards(raw_bytes, world: int) -> ShardPlan:
    """Longest-processing-time-first: biggest tensor to the least-loaded rank
    (ties: lower rank, then lower tensor index) — deterministic on all ranks."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(raw_bytes)), key=lambda i: (-int(raw_bytes[i]), i))
    heap = [(0, r) for r in range(world)]
    owner = [0] * len(raw_bytes)
    load = [0] * world
    for i in order:
        ld, r = heapq.heappop(heap)
        owner[i] = r
        load[r] = ld + int(raw_bytes[i])
        heapq.heappush(heap, (load[r], r))
    return ShardPlan(world=world, owner=tuple(owner), load=tuple(load))


def exchange_sizes(rows, world: int, max_rows: int | None = None, group=None,
                   device: torch.device | None = None) -> torch.Tensor:
    """All-gather this rank's (global_id, codec, count, bytes) rows (a list,
    or an int64 [k, 4] tensor, e.g. on the GPU).

    Returns an int64 tensor [world * max_rows, 4] on `device` (rows padded
    with global_id = -1).  Without a process group (a single-process save)
    no collective is issued; with one, the all-gather runs at any world size.
    """
    import torch.distributed as dist
    nrows = rows.shape[0] if isinstance(rows, torch.Tensor) else len(rows)
    max_rows = max(nrows, 1) if max_rows is None else max(max_rows, 1)
    if nrows > max_rows:
        raise ValueError("more rows than the plan allows")
    if device is None:
        if dist.is_initialized() and dist.get_backend(group) == "nccl":
            device = torch.device("cuda", torch.cuda.current_device())
        else:
            device = torch.device("cpu")
    if isinstance(rows, torch.Tensor):
        # rows already on the device (e.g. counts the encoder left there):
        # no host round trip before the all-gather
        local = torch.full((max_rows, ROW), -1, dtype=torch.int64, device=device)
        local[:nrows] = rows.to(device=device, dtype=torch.int64)
    else:
        local = torch.full((max_rows, ROW), -1, dtype=torch.int64)
        if rows:
            local[:nrows] = torch.tensor(rows, dtype=torch.int64)
        local = local.to(device)
    if world == 1 and not dist.is_initialized():
        return local
    out = torch.empty((world * max_rows, ROW), dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, local, group=group)
    return out


def global_offsets(gathered: torch.Tensor, n_total: int):
    """Rows from all ranks -> per-global-id (codec, count, offset, length),
    offsets = exclusive prefix sum in global_id order (store.py:240-247)."""
    g = gathered.cpu()
    g = g[g[:, 0] >= 0]
    if g.shape[0] != n_total:
        raise ValueError(f"size table has {g.shape[0]} rows, expected {n_total}")
    g = g[torch.argsort(g[:, 0])]
    if not torch.equal(g[:, 0], torch.arange(n_total)):
        raise ValueError("size table ids are not a permutation of the tensors")
    lengths = g[:, 3]
    offsets = torch.cumsum(lengths, 0) - lengths
    return [(int(c), int(k), int(o), int(l))
            for c, k, o, l in zip(g[:, 1], g[:, 2], offsets, lengths)]


# ---------------------------------------------------------------------------
# sharded checkpoint encode (one process per GPU)
# ---------------------------------------------------------------------------

CODEC_CODES = {"RAW": CODEC_RAW, "DELTA": CODEC_DELTA, "QUANT": CODEC_QUANT}


@dataclass(frozen=True)
class TensorSpec:
    """What every rank knows about every tensor (no data): enough to plan."""

    name: str
    group: str            # "model" | "optimizer"
    nbytes: int


def checkpoint_specs(ckpt) -> list:
    return ([TensorSpec(t.name, "model", t.nbytes) for t in ckpt.model_states]
            + [TensorSpec(t.name, "optimizer", t.nbytes) for t in ckpt.optimizer_states])


@dataclass
class ShardResult:
    manifest: object            # store.CheckpointManifest, identical on every rank
    records: list               # this rank's EncodedRecords
    offsets: list               # their global offsets in tensors.bin
    total_bytes: int            # length of the whole tensors.bin
    local: object = None        # host buffer holding the records back to back (`out`)
    local_offsets: list = None  # their offsets in `local` (+ the end)


def encode_sharded(specs, local, prev_local, kind: str, iteration: int, base_iteration: int,
                   rank: int, world: int, encoder, group=None, device=None,
                   plan: ShardPlan | None = None, out=None) -> ShardResult:
    """store.encode_checkpoint (store.py:214-272) across `world` ranks.

    specs: [TensorSpec] of the whole checkpoint in checkpoint order (model
    states, then optimizer states).  local: {name: tensor} holding at least
    the tensors the plan assigns to this rank (TensorBlob or DeviceTensor);
    prev_local: {name: previous model state} for those tensors (delta saves).
    encoder: an object with `encode_records(items, prev_map, kind)` — the
    store.CheckpointEncoder on a GPU.  The only communication is ONE
    all-gather of (global_id, codec, count, encoded_bytes) rows; every rank
    then derives the same manifest, whose offsets equal the single-process
    driver's, so the records written at their offsets form a byte-identical
    tensors.bin.

    out: a pinned (or registered) host uint8 buffer large enough for any
    encoding of this rank's tensors: the records are then encoded in groups
    and land back to back in it while later groups are encoded (the device
    arenas of a group or two at a time: a rank's share of a 7B-70B
    checkpoint fits beside its inputs), before the size-table exchange.
    """
    from .store import CheckpointManifest, ManifestEntry
    if plan is None:
        plan = plan_shards([s.nbytes for s in specs], world)
    mine = plan.local_ids(rank)
    items = [(gid, specs[gid].group, local[specs[gid].name]) for gid in mine]
    prev_map = None
    if kind == "delta":
        prev_map = {specs[gid].name: prev_local[specs[gid].name]
                    for gid in mine if specs[gid].group == "model"}
    local_offs = None
    if out is not None and items and hasattr(encoder, "encode_groups"):
        recs, local_offs, _ = encoder.encode_groups(items, prev_map, kind, out)
    else:
        recs, _ = encoder.encode_records(items, prev_map, kind) if items else ([], {})
    rows = [(r.gid, CODEC_CODES[r.codec], r.count, r.length) for r in recs]
    gathered = exchange_sizes(rows, world, plan.max_rows, group=group, device=device)
    table = global_offsets(gathered, len(specs))
    names = {v: k for k, v in CODEC_CODES.items()}
    entries = tuple(ManifestEntry(specs[i].name, specs[i].group, names[c], o, l)
                    for i, (c, _, o, l) in enumerate(table))
    manifest = CheckpointManifest(iteration=iteration, kind=kind,
                                  base_iteration=base_iteration, tensors=entries)
    total = (table[-1][2] + table[-1][3]) if table else 0
    return ShardResult(manifest, recs, [table[r.gid][2] for r in recs], total,
                       out if local_offs is not None else None, local_offs)


def write_shard(path: str, res: ShardResult, device=None) -> int:
    """pwrite this rank's records at their global offsets of `path` (a
    tensors.bin every rank opens; the file is sized to the full length).
    Returns the bytes written."""
    import os
    import torch
    from .store import sequential_offsets
    if res.local is not None:       # landed already (encode_sharded(out=...))
        local_offs, buf = res.local_offsets, res.local
    else:
        local_offs = sequential_offsets(res.records)
        buf = torch.empty(max(local_offs[-1], 1), dtype=torch.uint8,
                          pin_memory=torch.cuda.is_available())
        if res.records:
            if device is None and torch.cuda.is_available():
                device = torch.device("cuda", torch.cuda.current_device())
            _place(res.records, local_offs, buf, device)
    fd = os.open(path, os.O_WRONLY | os.O_CREAT, 0o644)
    try:
        if os.fstat(fd).st_size < res.total_bytes:
            os.ftruncate(fd, res.total_bytes)
        mv = memoryview(buf.numpy())
        for r, lo, go in zip(res.records, local_offs, res.offsets):
            _pwrite_all(fd, mv[lo:lo + r.length], go)
    finally:
        os.close(fd)
    return local_offs[-1]


def _pwrite_all(fd: int, mv: memoryview, offset: int) -> None:
    """pwrite until every byte landed: Linux moves at most 0x7ffff000 bytes
    per call, so a record of 2 GiB or more needs several."""
    import os
    done = 0
    while done < len(mv):
        k = os.pwrite(fd, mv[done:], offset + done)
        if k <= 0:
            raise OSError(f"pwrite wrote {k} bytes at offset {offset + done}")
        done += k


def _place(recs, offsets, buf, device):
    from .store import place_records
    if device is not None:
        place_records(recs, offsets, buf, device)
        return
    # host-only records (CPU tests with a host encoder)
    import numpy as np
    b = buf.numpy()
    for r, o in zip(recs, offsets):
        b[o:o + len(r.header)] = np.frombuffer(r.header, np.uint8)
        o += len(r.header)
        for p in r.parts:
            b[o:o + len(p)] = np.frombuffer(p, np.uint8)
            o += len(p)
