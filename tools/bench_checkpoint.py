#!/usr/bin/env python
"""Whole-checkpoint codec benchmark (BASELINE configs[0] "C0" and [3] "C3").

A checkpoint pair (base at iteration 0, delta at iteration 1) of a
GPT-2-small (C0), Llama-2-7B (C3, with fp32 master weights among the
optimizer states) or one rank's share of a Llama-2-70B (C4) shaped model is
generated on the GPU
(SURVEY §8(d) recipe: fp32 master w0 ~ N(0, 0.02), w1 = w0 - 1e-5 u, saved
weights bf16; Adam m ~ N(0, 1e-3), v = N(0, 1e-3)^2, quantized per tensor
with m = 16 clusters as store.encode_checkpoint does).  Timed with CUDA
events, inputs resident in HBM, outputs landing in pinned host memory:

  save_base   encode_checkpoint(kind=base)   RAW model + QUANT optimizer
  save_delta  encode_checkpoint(kind=delta)  DELTA model vs the resident
                                             previous states + QUANT
  load        decode_chain([base, delta])    RAW + in-place delta replay +
                                             dequantize (host blobs in)

GB/s = raw checkpoint bytes / time.  --verify re-encodes C0 with the CPU
oracle (numpy restatement of the reference) and compares the blobs.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


# optimizer-state names: torch.optim.Adam's state keys as name prefixes.  With
# the C0 tensor names below these reproduce the reference's published C0 blob
# size exactly (438,174,150 B; record headers carry the names)
M_PREFIX, V_PREFIX = "exp_avg.", "exp_avg_sq."


def shapes(config: str):
    if config == "C0":
        d, ffn, vocab, ctx, layers = 768, 3072, 50257, 1024, 12
        out = [("wte", (vocab, d)), ("wpe", (ctx, d))]
        for i in range(layers):
            p = f"h.{i}."
            out += [(p + "ln_1.weight", (d,)), (p + "ln_1.bias", (d,)),
                    (p + "attn.c_attn.weight", (d, 3 * d)), (p + "attn.c_attn.bias", (3 * d,)),
                    (p + "attn.c_proj.weight", (d, d)), (p + "attn.c_proj.bias", (d,)),
                    (p + "ln_2.weight", (d,)), (p + "ln_2.bias", (d,)),
                    (p + "mlp.c_fc.weight", (d, ffn)), (p + "mlp.c_fc.bias", (ffn,)),
                    (p + "mlp.c_proj.weight", (ffn, d)), (p + "mlp.c_proj.bias", (d,))]
        return out + [("ln_f.weight", (d,)), ("ln_f.bias", (d,))]
    if config == "C3":
        d, ffn, vocab, layers = 4096, 11008, 32000, 32
        out = [("embed", (vocab, d)), ("lm_head", (vocab, d)), ("norm", (d,))]
        for i in range(layers):
            p = f"layers.{i}."
            out += [(p + n, (d, d)) for n in ("q", "k", "v", "o")]
            out += [(p + "gate", (ffn, d)), (p + "up", (ffn, d)), (p + "down", (d, ffn)),
                    (p + "in_norm", (d,)), (p + "post_norm", (d,))]
        return out
    if config == "C4":   # Llama-2-70B: GQA k/v (1024, 8192), ffn 28672
        d, ffn, kv, vocab, layers = 8192, 28672, 1024, 32000, 80
        out = [("embed", (vocab, d)), ("lm_head", (vocab, d)), ("norm", (d,))]
        for i in range(layers):
            p = f"layers.{i}."
            out += [(p + "q", (d, d)), (p + "k", (kv, d)), (p + "v", (kv, d)), (p + "o", (d, d)),
                    (p + "gate", (ffn, d)), (p + "up", (ffn, d)), (p + "down", (d, ffn)),
                    (p + "in_norm", (d,)), (p + "post_norm", (d,))]
        return out
    raise ValueError(config)


def shard_names(config: str, rank: int, world: int):
    """The tensors planner.plan_shards gives `rank` of `world` (LPT over the
    bf16 w + base + fp32 m, v bytes of each tensor)."""
    from paper_2511_12376_b200.planner import plan_shards
    shp = shapes(config)
    raw = []
    for _, s in shp:
        n = 1
        for x in s:
            n *= x
        raw.append(12 * n)
    plan = plan_shards(raw, world)
    return {name for (name, _), r in zip(shp, plan.owner) if r == rank}, plan


def generate(config: str, dev, seed: int = 0, only=None):
    import torch
    from paper_2511_12376_b200.store import DeviceTensor
    from paper_2511_12376_b200.tensors import Checkpoint
    g = torch.Generator(device=dev).manual_seed(seed)
    base, cur, opt = [], [], []
    for name, shp in shapes(config):
        if only is not None and name not in only:
            continue
        w0 = torch.randn(shp, device=dev, generator=g) * 0.02
        w1 = w0 - 1e-5 * torch.randn(shp, device=dev, generator=g)
        base.append(DeviceTensor.wrap(name, w0.to(torch.bfloat16)))
        cur.append(DeviceTensor.wrap(name, w1.to(torch.bfloat16)))
        if config == "C3":   # BASELINE configs[3]: bf16 weights plus fp32 master, m and v
            opt.append(DeviceTensor.wrap("master." + name, w1))
        del w0, w1
        opt.append(DeviceTensor.wrap(M_PREFIX + name,
                                     torch.randn(shp, device=dev, generator=g) * 1e-3))
        opt.append(DeviceTensor.wrap(V_PREFIX + name,
                                     (torch.randn(shp, device=dev, generator=g) * 1e-3) ** 2))
    return (Checkpoint(iteration=0, model_states=base, optimizer_states=opt),
            Checkpoint(iteration=1, model_states=cur, optimizer_states=opt))


def generate_cpu_recipe_host(config: str, seed: int = 0) -> dict:
    """SURVEY §8(d)'s C0 recipe exactly (the inputs of the reference's
    published ratios, tests/golden/c0_ratio.json): ONE CPU torch.Generator
    seeded 0; per tensor, in checkpoint order, w0 = randn * 0.02, u = randn,
    w1 = w0 - 1e-5 u, m = randn * 1e-3, v = (randn * 1e-3)^2; weights saved as
    bf16 (round to nearest even).  -> {name: (w0 u16, w1 u16, m f32, v f32)}"""
    import torch
    g = torch.Generator().manual_seed(seed)
    out = {}
    for name, shp in shapes(config):
        w0 = torch.randn(shp, generator=g) * 0.02
        u = torch.randn(shp, generator=g)
        w1 = w0 - 1e-5 * u
        m = torch.randn(shp, generator=g) * 1e-3
        v = (torch.randn(shp, generator=g) * 1e-3) ** 2
        b = lambda t: t.to(torch.bfloat16).view(torch.int16).numpy().view("<u2")
        out[name] = (b(w0), b(w1), m.numpy(), v.numpy())
    return out


def generate_cpu_recipe(config: str, dev, seed: int = 0):
    """generate_cpu_recipe_host, moved to the GPU as DeviceTensors."""
    import torch
    from paper_2511_12376_b200.store import DeviceTensor
    from paper_2511_12376_b200.tensors import Checkpoint
    base, cur, opt = [], [], []
    for name, (w0, w1, m, v) in generate_cpu_recipe_host(config, seed).items():
        bf = lambda a: torch.from_numpy(a.view("<i2")).to(dev).view(torch.bfloat16)
        base.append(DeviceTensor.wrap(name, bf(w0)))
        cur.append(DeviceTensor.wrap(name, bf(w1)))
        opt.append(DeviceTensor.wrap(M_PREFIX + name, torch.from_numpy(m).to(dev)))
        opt.append(DeviceTensor.wrap(V_PREFIX + name, torch.from_numpy(v).to(dev)))
    return (Checkpoint(iteration=0, model_states=base, optimizer_states=opt),
            Checkpoint(iteration=1, model_states=cur, optimizer_states=opt))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C0", choices=["C0", "C3", "C4"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--verify", action="store_true")
    ap.add_argument("--shard", default=None,
                    help="R/W: only rank R's tensors of a W-rank plan (C4 needs 8 GPUs' HBM)")
    args = ap.parse_args()
    import torch
    from paper_2511_12376_b200 import store as S
    dev = torch.device("cuda:0")
    if args.shard or args.config in ("C3", "C4"):
        # C3 (107.8 GB of states) and its restore do not fit one GPU together:
        # the shard path frees the inputs before the restore
        default = "0/8" if args.config == "C4" else "0/1"
        return run_shard(args, *(int(x) for x in (args.shard or default).split("/")))
    c0, c1 = generate(args.config, dev)
    raw = sum(t.nbytes for t in c1.model_states + c1.optimizer_states)
    enc = S.CheckpointEncoder(dev, clusters=16)

    def timed(fn):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        return out, time.perf_counter() - t

    # a training loop keeps its pinned save buffers (page-locking GBs per save
    # would dominate), sized for any outcome (store.blob_bound) so the save
    # can stream groups of records out while later groups are encoded
    buf0 = torch.empty(S.blob_bound(c0), dtype=torch.uint8, pin_memory=True)
    buf1 = torch.empty(S.blob_bound(c1), dtype=torch.uint8, pin_memory=True)
    m0, b0 = enc.encode(c0, None, S.KIND_BASE, out=buf0)
    m1, b1 = enc.encode(c1, None, S.KIND_DELTA, out=buf1)
    res = {}
    out = None
    for _ in range(args.reps):
        out = None  # the previous restore holds model + dequantized optimizer states
        (m0, b0), tb = timed(lambda: enc.encode(c0, None, S.KIND_BASE, out=buf0))
        (m1, b1), td = timed(lambda: enc.encode(c1, None, S.KIND_DELTA, out=buf1))
        chain = [(m0, b0), (m1, b1)]
        out, tl = timed(lambda: S.decode_chain(chain, to_host=False))
        for k, v in (("save_base_s", tb), ("save_delta_s", td), ("load_s", tl)):
            res[k] = min(res.get(k, 1e9), v)
    blob1 = b1.numpy().tobytes() if args.verify else None
    # correctness of the round trip on the device
    for a, b in zip(out.model_states, c1.model_states):
        assert torch.equal(a.data.view(torch.int16), b.flat())
    codecs = {}
    for e in m1.tensors:
        codecs[e.codec] = codecs.get(e.codec, 0) + 1
    mb = sum(t.nbytes for t in c1.model_states)
    ob = sum(t.nbytes for t in c1.optimizer_states)
    mlen = sum(e.length for e in m1.tensors if e.group == "model")
    olen = sum(e.length for e in m1.tensors if e.group == "optimizer")
    line = {
        "config": args.config, "tensors": len(m1.tensors), "raw_bytes": raw,
        "codecs_delta_checkpoint": codecs,
        "ratio_weights": round(mb / mlen, 4), "ratio_optimizer": round(ob / olen, 4),
        "ratio_total": round(raw / b1.numel(), 4),
        "save_base_gbs": round(raw / res["save_base_s"] / 1e9, 2),
        "save_delta_gbs": round(raw / res["save_delta_s"] / 1e9, 2),
        "load_gbs": round(raw / res["load_s"] / 1e9, 2),
        **{k: round(v, 4) for k, v in res.items()},
        "note": "device-resident inputs; outputs land in reused pinned host buffers (D2H "
                "included); load starts from those host blobs (H2D included)",
    }
    if args.verify and args.config == "C0":
        import numpy as np
        from oracle import bitsnap_oracle as O

        def conv(ts, code):
            return [(t.name, t.shape, code, t.flat().cpu().numpy().view(
                np.uint16 if code == 0 else np.float32)) for t in ts]
        t = time.perf_counter()
        entries, want = O.encode_checkpoint(conv(c1.model_states, 0),
                                            conv(c1.optimizer_states, 1),
                                            conv(c0.model_states, 0), "delta", 16)
        line["oracle_delta_encode_s"] = round(time.perf_counter() - t, 2)
        line["oracle_blob_identical"] = want == blob1
        line["oracle_manifest_identical"] = entries == [vars(e) for e in m1.tensors]
    print(json.dumps(line), flush=True)


def run_shard(args, rank: int, world: int):
    """One rank's share of a multi-GPU save: the tensors the LPT plan gives
    `rank`, encoded on this GPU (the ranks share nothing but the size-table
    all-gather, so the job's time is the slowest rank's).  The restore runs
    after the inputs but the compared weights are freed (inputs and restored
    states of a C4 shard do not fit one GPU together)."""
    import torch
    from paper_2511_12376_b200 import store as S
    dev = torch.device("cuda:0")
    only, plan = shard_names(args.config, rank, world)
    c0, c1 = generate(args.config, dev, only=only)
    raw = sum(t.nbytes for t in c1.model_states + c1.optimizer_states)
    # c0 / c1 are immutable snapshot buffers: borrowed, not copied (a C4
    # shard has no room for an owned copy of its weights)
    enc = S.CheckpointEncoder(dev, clusters=16, keep_prev="borrow")
    import numpy as np
    from paper_2511_12376_b200 import _runtime as rt

    def pinned(n):
        # page-locked by registration: the caching host allocator would
        # round tens of GB up to the next power of two
        a = np.empty(n, dtype=np.uint8)
        assert rt.lib().bsnp_host_register(a.ctypes.data, n) == 0, "host register failed"
        t = torch.from_numpy(a)
        assert t.is_pinned()
        return t
    buf0 = pinned(S.blob_bound(c0))
    buf1 = pinned(S.blob_bound(c1))

    def timed(fn):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        return out, time.perf_counter() - t
    res = {}
    for _ in range(args.reps):
        (m0, b0), tb = timed(lambda: enc.encode(c0, None, S.KIND_BASE, out=buf0))
        (m1, b1), td = timed(lambda: enc.encode(c1, None, S.KIND_DELTA, out=buf1))
        for k, v in (("save_base_s", tb), ("save_delta_s", td)):
            res[k] = min(res.get(k, 1e9), v)
    peak_save = torch.cuda.max_memory_allocated(dev)
    want = [t.flat() for t in c1.model_states]
    inputs = sum(t.nbytes for t in list(c0.model_states) + list(c1.model_states)
                 + list(c1.optimizer_states))
    del c0, c1, enc
    torch.cuda.empty_cache()
    out, tl = timed(lambda: S.decode_chain([(m0, b0), (m1, b1)], to_host=False))
    res["load_s"] = tl
    ok = all(torch.equal(a.data.view(torch.int16), b) for a, b in zip(out.model_states, want))
    mlen = sum(e.length for e in m1.tensors if e.group == "model")
    olen = sum(e.length for e in m1.tensors if e.group == "optimizer")
    line = {"config": args.config, "shard": f"{rank}/{world}", "tensors": len(m1.tensors),
            "raw_bytes": raw, "plan_load_max_over_mean": round(max(plan.load) * world /
                                                                sum(plan.load), 4),
            "input_bytes_on_gpu": inputs,
            "ratio_total": round(raw / b1.numel(), 4),
            "ratio_weights_optimizer": [round(sum(t.nbytes for t in out.model_states) / mlen, 4),
                                        round(sum(t.nbytes for t in out.optimizer_states) /
                                              olen, 4)],
            "save_base_gbs": round(raw / res["save_base_s"] / 1e9, 2),
            "save_delta_gbs": round(raw / res["save_delta_s"] / 1e9, 2),
            "load_gbs": round(raw / res["load_s"] / 1e9, 2),
            **{k: round(v, 4) for k, v in res.items()},
            "peak_gpu_bytes_save": peak_save,
            "peak_gpu_bytes": torch.cuda.max_memory_allocated(dev),
            "restored_weights_identical": ok,
            "note": "one rank's shard on one GPU; device-resident inputs, blobs in pinned host "
                    "memory (D2H / H2D included); load once, after freeing the inputs"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
