"""One rank's share of the bench's sharded checkpoint line on ONE GPU
(bench.run_ckpt_sharded for rank R of W, no process group): the size-table
all-gather is replaced by a stand-in that fills the other ranks' rows with
placeholder sizes, so everything the rank itself does — generating its LPT
share, the grouped encode landing in registered host memory, the restore of
its records, the bit-exact weight check — runs as in the W-GPU job.  A
memory-fit check for configurations whose multi-GPU run needs a node this
session does not have (C4 at 8 ranks: ~103 GB of states per GPU).  Dev tool.

usage: python tools/dryrun_shard.py C4 0 8
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench
from paper_2511_12376_b200 import planner as PL

config, rank, world = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
real = PL.exchange_sizes
_specs = {}


def stand_in(rows, world_, max_rows=None, group=None, device=None):
    local = real(rows, 1, max_rows, group=None, device=torch.device("cpu"))
    have = {int(r[0]) for r in local if r[0] >= 0}
    n = _specs["n"]
    fill = [(g, PL.CODEC_RAW, 0, 1) for g in range(n) if g not in have]
    out = torch.full((world_ * local.shape[0] + len(fill), PL.ROW), -1, dtype=torch.int64)
    out[:local.shape[0]] = local
    if fill:
        out[local.shape[0]:local.shape[0] + len(fill)] = torch.tensor(fill, dtype=torch.int64)
    return out


orig_encode_sharded = PL.encode_sharded


def encode_sharded(specs, *a, **k):
    _specs["n"] = len(specs)
    return orig_encode_sharded(specs, *a, **k)


PL.exchange_sizes = stand_in
PL.encode_sharded = encode_sharded
# no process group: barriers are no-ops, the stats gather sees this rank only
import torch.distributed as dist
dist.barrier = lambda *a, **k: None
dist.get_backend = lambda *a, **k: "gloo"


def _gather(out_list, t, *a, **k):
    for o in out_list:
        o.copy_(t)


dist.all_gather = _gather
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
line = bench.run_ckpt_sharded(config, dev, rank, world)
line["dryrun"] = f"rank {rank} of {world} on one GPU; other ranks' size rows are placeholders"
line["peak_allocated_gb"] = round(torch.cuda.max_memory_allocated(dev) / 1e9, 2)
print(json.dumps(line))
