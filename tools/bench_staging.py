#!/usr/bin/env python
"""Staging hand-off benchmark: a whole checkpoint
encoded on the GPU and staged into a BSSL slot region (engine.SlotRegion).

  direct   region.stage_checkpoint: records DMA'd straight into the
           page-locked mapped slot, then the blake2b-64 checksum on the host
  bounce   CheckpointEncoder.encode into a reused pinned buffer, then
           region.stage(pack_blob(...)) — the copy-through-host hand-off the
           reference's stage() implies

Times are host wall clock around each call (device work included: the
encoder synchronises before returning); `checksum_s` is the blake2b share,
which the format fixes on the host.  C0 (GPT-2-small) by default; the region
file lives under --dir (page cache).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C0", choices=["C0", "C3"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dir", default=tempfile.gettempdir())
    args = ap.parse_args()
    import torch
    from bench_checkpoint import generate
    from paper_2511_12376_b200 import engine as E
    from paper_2511_12376_b200 import store as S
    dev = torch.device("cuda:0")
    c0, c1 = generate(args.config, dev)
    raw = sum(t.nbytes for t in c1.model_states + c1.optimizer_states)
    enc = S.CheckpointEncoder(dev, clusters=16)
    man, out = enc.encode(c0, None, S.KIND_BASE)
    man1, out1 = enc.encode(c1, c0, S.KIND_DELTA)
    blob_len = S.BLOB_HEADER.size + len(man1.to_bytes()) + out1.numel()
    cap = blob_len + (1 << 20)
    path = os.path.join(args.dir, f"bsnp_stage_{os.getpid()}.bssl")
    res = {}
    try:
        region = E.SlotRegion.create(path, 1, 2 * args.reps + 2, cap)
        dma = region.dma_ready
        it = 1000
        for _ in range(args.reps):
            ck = type(c1)(iteration=it, model_states=c1.model_states,
                          optimizer_states=c1.optimizer_states)
            torch.cuda.synchronize()
            t = time.perf_counter()
            info, m = region.stage_checkpoint(0, enc, ck, c0, S.KIND_DELTA)
            t_direct = time.perf_counter() - t
            t = time.perf_counter()
            E.checksum(region.payload_view(0, info.index))
            t_sum = time.perf_counter() - t
            it += 1
            ck = type(c1)(iteration=it, model_states=c1.model_states,
                          optimizer_states=c1.optimizer_states)
            torch.cuda.synchronize()
            t = time.perf_counter()
            mb, ob = enc.encode(ck, c0, S.KIND_DELTA, out=out1)
            region.stage(0, S.pack_blob(mb, ob), it)
            t_bounce = time.perf_counter() - t
            it += 1
            for k, v in (("direct_s", t_direct), ("bounce_s", t_bounce), ("checksum_s", t_sum)):
                res[k] = min(res.get(k, 1e9), v)
            assert region.verify(0, info.index)
        region.close()
    finally:
        if os.path.exists(path):
            os.unlink(path)
    line = {"config": args.config, "raw_bytes": raw, "blob_bytes": blob_len,
            "dma_into_mapping": dma,
            "direct_s": round(res["direct_s"], 4), "bounce_s": round(res["bounce_s"], 4),
            "checksum_s": round(res["checksum_s"], 4),
            "direct_gbs_raw": round(raw / res["direct_s"] / 1e9, 2),
            "direct_excl_checksum_gbs_raw":
                round(raw / max(res["direct_s"] - res["checksum_s"], 1e-9) / 1e9, 2),
            "note": "delta save of iteration 1 against the resident iteration-0 model "
                    "states; times include device work, D2H and the host checksum"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
