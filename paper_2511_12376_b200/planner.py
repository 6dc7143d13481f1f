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
    """All-gather this rank's (global_id, codec, count, bytes) rows.

    Returns an int64 tensor [world * max_rows, 4] on `device` (rows padded
    with global_id = -1).  With world == 1 no collective is issued.
    """
    import torch.distributed as dist
    max_rows = max(len(rows), 1) if max_rows is None else max(max_rows, 1)
    if len(rows) > max_rows:
        raise ValueError("more rows than the plan allows")
    if device is None:
        if dist.is_initialized() and dist.get_backend(group) == "nccl":
            device = torch.device("cuda", torch.cuda.current_device())
        else:
            device = torch.device("cpu")
    local = torch.full((max_rows, ROW), -1, dtype=torch.int64)
    if rows:
        local[:len(rows)] = torch.tensor(rows, dtype=torch.int64)
    local = local.to(device)
    if world == 1:
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
