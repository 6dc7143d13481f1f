#!/usr/bin/env python
"""BitSnap B200 codec benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], "C1"): one flat bf16 tensor of 2^30
elements, base ~ N(0, 0.02) in bf16, current = base with k = round(p*n)
distinct uniformly-random elements moved by +-1 ulp (p = 1 % by default).
A step = bitmask encode of (base, current) followed by the decode of that
record back onto base, i.e. the save + restore pair of one delta checkpoint.

  value  = whole-job algorithmic GB/s, inputs resident in HBM
           (encode 4n + n/8 + 2n_c, decode n/8 + 2n_c + 4n bytes)
  e2e    = the same through pinned host buffers: H2D of the inputs and D2H of
           the encoded record / decoded tensor inside the timed region
  --impl reference : the reference algorithm (CPU oracle port, numpy, all host
           cores) on a bounded sample of the same workload.

Multi-GPU (torchrun): every rank encodes/decodes its own 2^30 shard (weak
scaling); the shard planner's NCCL all-gather of the per-rank size table is
part of every step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "bitmask delta encode+decode throughput (C1: 2^30 bf16, p changed)"
FALLBACK_HBM_GBS = 6650.0
NOMINAL_HBM_GBS = 8000.0   # the north star's nominal per-GPU HBM peak (reported beside "frac")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--log2n", type=int, default=30)
    ap.add_argument("--p", type=float, default=0.01)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-elems-per-core", type=int, default=1 << 23)
    ap.add_argument("--no-c2", action="store_true",
                    help="skip the C2 cluster-quantizer measurement")
    ap.add_argument("--no-c0", action="store_true",
                    help="skip the whole-checkpoint line (BASELINE configs[0], GPT-2-small)")
    ap.add_argument("--c2-log2n", type=int, default=30)
    ap.add_argument("--c2-block", type=int, default=1 << 20)
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the C1 change-fraction sweep (p = 0.1 / 1 / 6.25 / 25 %%)")
    ap.add_argument("--no-ckpt", action="store_true",
                    help="skip the sharded whole-checkpoint line (planner over all ranks)")
    ap.add_argument("--ckpt-config", default=None, choices=["C0", "C3", "C4"],
                    help="checkpoint of the sharded line (default C3; C4 at 8 ranks)")
    return ap.parse_args()


def max_over_ranks(values, dev):
    """Element-wise max over the job (NCCL on device tensors, gloo on host)."""
    import torch
    import torch.distributed as dist
    on = dev if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor(values, dtype=torch.float64, device=on)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu().tolist()]


def algo_bytes(n: int, n_c: int) -> tuple[int, int]:
    mask = (n + 7) // 8
    return 4 * n + mask + 2 * n_c, mask + 2 * n_c + 4 * n


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# clocks sampling during the timed region
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
         "clocks.mem,temperature.gpu,temperature.memory")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9 and parts[1].isdigit():
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = sorted(int(r[1]) for r in rows)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for name, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        out = {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": int(rows[0][2]),
               "samples": len(rows), "reasons": sorted(reasons)}

        def num(i):
            vals = []
            for r in rows:
                try:
                    vals.append(float(r[i]))
                except (IndexError, ValueError):
                    pass
            return vals
        mem, tg, tm, pw = num(9), num(10), num(11), num(3)
        if mem:
            out["mem_mhz"] = int(sorted(mem)[len(mem) // 2])
        if tg:
            out["gpu_temp_c_max"] = max(tg)
        if tm:
            out["hbm_temp_c_max"] = max(tm)
        if pw:
            out["power_w_max"] = max(pw)
        return out


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (oracle port) on all host cores
# ---------------------------------------------------------------------------
def _cpu_worker(args):
    seed, n, p, barrier = args
    import numpy as np
    from oracle import bitsnap_oracle as O
    rng = np.random.default_rng(seed)
    f = (rng.standard_normal(n, dtype=np.float32) * 0.02).view(np.uint32).astype(np.uint64)
    base = ((f + ((f >> 16) & 1) + 0x7FFF) >> 16).astype(np.uint16)
    cur = base.copy()
    k = int(round(p * n))
    idx = rng.choice(n, k, replace=False)
    cur[idx] += 1
    bb, cb = base.tobytes(), cur.tobytes()   # TensorBlob.data, as the reference holds it
    barrier.wait()
    t0 = time.perf_counter()
    mask, payload, n_c = O.ref_encode_bytes(bb, cb)
    out = O.ref_decode_bytes(bb, mask, payload, n, n_c)
    dt = time.perf_counter() - t0
    assert out == cb
    e, d = algo_bytes(n, n_c)
    return e + d, dt, t0


def cpu_baseline(p: float, per_core: int, cores: int | None = None, reps: int = 1):
    import multiprocessing as mp
    cores = cores or len(os.sched_getaffinity(0))
    ctx = mp.get_context("fork")
    best = None
    with ctx.Manager() as mgr:
        for r in range(reps):
            barrier = mgr.Barrier(cores)
            with ctx.Pool(cores) as pool:
                res = pool.map(_cpu_worker, [(1000 * r + i, per_core, p, barrier)
                                             for i in range(cores)])
            total = sum(x[0] for x in res)
            start = min(x[2] for x in res)
            end = max(x[2] + x[1] for x in res)
            gbs = total / (end - start) / 1e9
            best = gbs if best is None else max(best, gbs)
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                 if l.startswith("model name")][0]
    except Exception:
        model = "unknown"
    return {"value": round(best, 3), "unit": "GB/s", "cores": cores,
            "kind": "port",
            "sample": f"{cores} x {per_core} bf16 elements (one per core), p={p}, "
                      f"the reference's encode_delta + decode_delta step for step on bytes "
                      f"(oracle ref_encode_bytes / ref_decode_bytes), best of {reps}; "
                      f"cpu: {model}"}


def _cpu_model():
    try:
        return [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                if l.startswith("model name")][0]
    except Exception:
        return "unknown"


def _c2_cpu_worker(args):
    seed, block, blocks, dist, barrier = args
    import numpy as np
    from oracle import bitsnap_oracle as O
    rng = np.random.default_rng(seed)
    xs = []
    for _ in range(blocks):
        x = rng.standard_normal(block, dtype=np.float32) * np.float32(1e-3)
        xs.append(x * x if dist == "adam_v" else x)
    barrier.wait()
    t0 = time.perf_counter()
    for x in xs:
        tab = O.cluster_fit(x, 16)
        packed, codes, _ = O.cluster_quantize(x, tab)
        O.cluster_dequantize(packed, codes, x.size, tab)
    return len(xs) * block, time.perf_counter() - t0, t0


def cpu_baseline_c2(block: int = 1 << 20, blocks_per_core: int = 2, cores: int | None = None,
                    dist: str = "adam_m"):
    """the reference's per-block cluster codec (oracle port:
    build_clusters + quantize + dequantize, quantizer.py:100-204) on whole
    2^20-element blocks, one process per core."""
    import multiprocessing as mp
    cores = cores or len(os.sched_getaffinity(0))
    ctx = mp.get_context("fork")
    with ctx.Manager() as mgr:
        barrier = mgr.Barrier(cores)
        with ctx.Pool(cores) as pool:
            res = pool.map(_c2_cpu_worker, [(100 + i, block, blocks_per_core, dist, barrier)
                                            for i in range(cores)])
    elems = sum(r[0] for r in res)
    wall = max(r[2] + r[1] for r in res) - min(r[2] for r in res)
    # encode + decode algorithmic bytes (5.5 B per element each way)
    return {"value": round(2 * 5.5 * elems / wall / 1e9, 4), "unit": "GB/s", "cores": cores,
            "kind": "port",
            "sample": f"{cores} x {blocks_per_core} blocks of {block} fp32 ({dist}), m = 16, "
                      f"numpy oracle fit + quantize + dequantize; cpu: {_cpu_model()}"}


def _c0_cpu_worker(args):
    names, barrier = args
    import numpy as np
    from oracle import bitsnap_oracle as O
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bench_checkpoint as BC
    data = _C0_CPU["data"]
    model = [(n, data[n][0].shape, 0, data[n][1]) for n in names]
    prev = [(n, data[n][0].shape, 0, data[n][0]) for n in names]
    opt = [(k + n, data[n][2].shape, 1, data[n][2 + i]) for n in names
           for i, k in enumerate((BC.M_PREFIX, BC.V_PREFIX))]
    barrier.wait()
    t0 = time.perf_counter()
    O.encode_checkpoint(model, opt, prev, "delta", 16)
    return sum(10 * data[n][0].size for n in names), time.perf_counter() - t0, t0


_C0_CPU: dict = {}


def cpu_baseline_c0(cores: int | None = None, max_elems: int | None = None):
    """the reference's whole-checkpoint encode (oracle port of
    store.encode_checkpoint, store.py:214-272) on the C0 delta pair, tensors
    spread over the cores (LPT); `max_elems` bounds the sample (1-core)."""
    import multiprocessing as mp
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from bench_checkpoint import generate_cpu_recipe_host
    data = generate_cpu_recipe_host("C0")
    names = list(data)
    if max_elems:
        picked, tot = [], 0
        for nm in names:
            if tot + data[nm][0].size > max_elems and picked:
                continue
            picked.append(nm)
            tot += data[nm][0].size
        names = picked
    _C0_CPU["data"] = data
    cores = cores or len(os.sched_getaffinity(0))
    bins = [[] for _ in range(cores)]
    loads = [0] * cores
    for nm in sorted(names, key=lambda k: -data[k][0].size):
        i = loads.index(min(loads))
        bins[i].append(nm)
        loads[i] += data[nm][0].size
    bins = [b for b in bins if b]
    ctx = mp.get_context("fork")
    with ctx.Manager() as mgr:
        barrier = mgr.Barrier(len(bins))
        with ctx.Pool(len(bins)) as pool:
            res = pool.map(_c0_cpu_worker, [(b, barrier) for b in bins])
    _C0_CPU.clear()
    raw = sum(r[0] for r in res)
    wall = max(r[2] + r[1] for r in res) - min(r[2] for r in res)
    return {"value": round(raw / wall / 1e9, 4), "unit": "GB/s (raw checkpoint bytes / s)",
            "cores": len(bins), "kind": "port",
            "sample": f"{len(names)} of the C0 delta pair's tensors ({raw / 1e9:.3f} GB raw), "
                      f"numpy oracle encode_checkpoint(kind=delta); cpu: {_cpu_model()}"}


def c1_config(n: int, p: float, world: int) -> dict:
    """The C1 workload of the bench line — the same dict on both arms."""
    return {"workload": "C1", "n_per_gpu": n, "p": p, "n_c": int(round(p * n)),
            "dtype": "bf16 (raw u16 patterns)", "parallelism": f"shard x{world}",
            "l2": "inputs 4 GiB >> 126 MB L2 (no flush needed)"}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    per_core = args.cpu_elems_per_core
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(args.p, per_core, reps=1)
        if i >= args.warmup:
            vals.append(r["value"])
    v = sorted(vals)[len(vals) // 2]
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "impl": "reference",
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u16", "data": "synthetic",
            # the B200 arm's workload; each step times a bounded sample of it
            # (cpu_baseline.sample says which)
            "config": c1_config(1 << args.log2n, args.p, world),
            "cpu_baseline": {**r, "value": v},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def make_c1(n: int, p: float, seed: int, dev):
    """Seeded C1 generator: exactly k = round(p n) changes."""
    import torch
    g = torch.Generator(device=dev).manual_seed(seed)
    base = (torch.randn(n, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    base = base.view(torch.int16)
    k = int(round(p * n))
    idx = torch.randperm(n, device=dev, generator=g)[:k]
    sgn = torch.randint(0, 2, (k,), device=dev, generator=g, dtype=torch.int32) * 2 - 1
    vals = base[idx].to(torch.int32) & 0xFFFF
    sgn = torch.where((vals & 0x7FFF) == 0, torch.ones_like(sgn), sgn)
    cur = base.clone()
    v = (vals + sgn) & 0xFFFF
    cur[idx] = torch.where(v > 32767, v - 65536, v).to(torch.int16)
    del idx, sgn, vals
    torch.cuda.synchronize(dev)
    return base, cur, k


def run_b200(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist
    from paper_2511_12376_b200 import bitmask as B
    from paper_2511_12376_b200 import _runtime as rt
    from paper_2511_12376_b200 import planner

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n = 1 << args.log2n
    base, cur, k = make_c1(n, args.p, args.seed + rank, dev)
    mask = torch.empty((n + 7) // 8, dtype=torch.uint8, device=dev)
    payload = torch.empty(n, dtype=torch.int16, device=dev)
    out = torch.empty_like(base)
    st = rt.new_status(dev, 2)
    stream = torch.cuda.current_stream(dev)

    # the step never waits for the host: the decode reads n_c from the
    # encode's status word on the device, and the size row of the
    # multi-GPU exchange is built there too
    row = torch.tensor([[0, 1, 0, (n + 7) // 8]], dtype=torch.int64, device=dev)

    def step(timing=None):
        if timing:
            timing[0].record(stream)
        B.encode_delta_async(base, cur, mask, payload, st[0])
        if timing:
            timing[1].record(stream)
        if world > 1:
            row[0, 2:3].copy_(st[0, 0:1])
            row[0, 3:4].copy_(st[0, 0:1] * 2 + (n + 7) // 8)
            planner.exchange_sizes(row, world)
        if timing:
            timing[2].record(stream)
        B.decode_delta_async_dn(base, mask, payload, st[0], out, st[1])
        if timing:
            timing[3].record(stream)

    for _ in range(args.warmup):
        step()
    (n_c, flags), (pc, dflags) = rt.read_status(st)
    assert n_c == k and flags == 0 and pc == k and dflags == 0, (n_c, k, flags, pc, dflags)
    torch.cuda.synchronize(dev)
    # correctness of the timed configuration: decode(encode(cur)) == cur
    assert torch.equal(out, cur)

    joined = None
    if world > 1:
        # which GPUs the ranks run on (one process per GPU): rank, device
        # name and PCI bus id, gathered once over the job's backend
        props = torch.cuda.get_device_properties(dev)
        me = {"rank": rank, "local_rank": local_rank, "host": os.uname().nodename,
              "device": props.name,
              "pci_bus_id": f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:"
                            f"{props.pci_device_id:02x}"}
        joined = [None] * world
        dist.all_gather_object(joined, me)
        if rank == 0:
            # stdout carries only the JSON line; the join record goes to stderr too
            print(f"[bench] {dist.get_backend()} process group: {world} ranks joined: "
                  + ", ".join(f"rank {j['rank']} {j['device']} {j['pci_bus_id']}@{j['host']}"
                              for j in joined), file=sys.stderr, flush=True)
    clocks = Clocks(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        step(evs[i])
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    (n_c, flags), (pc, dflags) = rt.read_status(st)
    assert n_c == k and flags == 0 and pc == k and dflags == 0, (n_c, k, flags, pc, dflags)
    ms = t_start.elapsed_time(t_end) / args.steps
    enc_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    dec_ms = sum(e[2].elapsed_time(e[3]) for e in evs) / args.steps
    if world > 1:
        ms, = max_over_ranks([ms], dev)
        dist.barrier()

    eb, db = algo_bytes(n, k)
    value = world * (eb + db) / (ms * 1e-3) / 1e9

    # ---------------- e2e through pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, base, cur, k, dev, world)
    del base, cur, mask, payload, out
    sweep = None if args.no_sweep else run_c1_sweep(args, dev, world)
    c2 = None if args.no_c2 else run_c2(args, dev, world)
    c2_modes = None if args.no_c2 else run_c2_modes(args, dev, world)
    c0 = None if (args.no_c0 or world > 1) else run_c0(dev)
    ckpt = None
    if not args.no_ckpt:
        cfg = args.ckpt_config or ("C4" if world == 8 else "C3")
        ckpt = run_ckpt_sharded(cfg, dev, rank, world)

    if rank != 0:
        return
    hbm, peak_kind = peaks()
    dom = "delta_encode" if enc_ms >= dec_ms else "delta_decode"
    dom_ms = max(enc_ms, dec_ms)
    dom_bytes = eb if dom == "delta_encode" else db
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = ncu_traffic().get(dom)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u16", "data": "synthetic",
        "config": c1_config(n, args.p, world),
        "ops": {"encode_gbs": round(eb / (enc_ms * 1e-3) / 1e9, 1),
                "decode_gbs": round(db / (dec_ms * 1e-3) / 1e9, 1),
                "encode_ms": round(enc_ms, 4), "decode_ms": round(dec_ms, 4),
                "compression_ratio": round(2 * n / (B.delta_size_bytes(n, k) + 1), 4)},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                     "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4),
                     "frac_of_nominal_8000": round(achieved / NOMINAL_HBM_GBS, 4),
                     "algorithmic_bytes": dom_bytes,
                     "traffic": traffic["bytes"] if traffic else None,
                     "traffic_detail": traffic},
        # the whole job's rate against N GPUs' measured HBM bandwidth
        "box": {"gbs": round(value, 2), "gpus": world, "peak_gbs": round(world * hbm, 1),
                "frac_of_hbm": round(value / (world * hbm), 4)},
        # per step: zero + encode; zero, count, scan, offsets table, decode
        "gpu_launches": 7 * args.steps,
        "clocks": clk,
    }
    if joined:
        line["dist"] = {"backend": dist.get_backend(), "world": world, "ranks": joined}
    if e2e:
        line["e2e"] = e2e
    if sweep:
        line["c1_sweep"] = sweep
    if c2:
        line["c2_cluster_quant"] = c2
    if c2_modes:
        line["c2_modes"] = c2_modes
    if c0:
        line["c0_checkpoint"] = c0
    if ckpt:
        line[ckpt.pop("key")] = ckpt
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.p, args.cpu_elems_per_core)
        # the 1-core figure beside the all-core one
        one = cpu_baseline(args.p, args.cpu_elems_per_core, cores=1)
        line["cpu_baseline"]["value_1core"] = one["value"]
        if not args.no_c2:
            c2cpu = cpu_baseline_c2()
            c2cpu["value_1core"] = cpu_baseline_c2(blocks_per_core=2, cores=1)["value"]
            line["cpu_baseline_c2"] = c2cpu
        if not args.no_c0:
            c0cpu = cpu_baseline_c0()
            c0cpu["value_1core"] = cpu_baseline_c0(cores=1, max_elems=3_000_000)["value"]
            line["cpu_baseline_c0"] = c0cpu
            # C3 / C4 on the CPU by extrapolation from a timed
            # sample — here the C0 whole-checkpoint rate (the same codec mix:
            # bf16 deltas + quantized fp32 states) scaled by raw bytes
            for key in ("c3_sharded", "c4_sharded"):
                if key in line and c0cpu["value"] > 0:
                    raw = line[key]["raw_bytes"]
                    line[key]["cpu_extrapolated"] = {
                        "save_delta_s": round(raw / (c0cpu["value"] * 1e9), 1),
                        "cores": c0cpu["cores"], "kind": "port, extrapolated",
                        "basis": "cpu_baseline_c0 rate (numpy oracle encode_checkpoint, "
                                 "all host cores) x this checkpoint's raw bytes"}
    print(json.dumps(line), flush=True)


C0_PUBLISHED_BLOB = 438_174_150   # 1,244,398,080 -> 438,174,150 B


def run_c0(dev, reps: int = 3):
    """BASELINE configs[0]: a GPT-2-small checkpoint pair (bf16 weights, fp32
    Adam m/v) generated by SURVEY §8(d)'s CPU recipe — the inputs the
    reference's own store encoded for tests/golden/c0_ratio.json — saved as
    base + delta through store.CheckpointEncoder into reused pinned buffers
    and restored with decode_chain (blobs H2D, chain replay, dequantize).
    The delta blob must be the reference's byte for byte (size and sha256).
    GB/s = raw bytes / wall time per call (device work and PCIe copies
    inside)."""
    import hashlib
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from bench_checkpoint import generate_cpu_recipe
    from paper_2511_12376_b200 import store as S
    c0, c1 = generate_cpu_recipe("C0", dev)
    raw = sum(t.nbytes for t in c1.model_states + c1.optimizer_states)
    enc = S.CheckpointEncoder(dev, clusters=16)
    bufs = [torch.empty(S.blob_bound(c), dtype=torch.uint8, pin_memory=True) for c in (c0, c1)]
    best = {}
    for _ in range(reps + 1):
        t = []
        for fn in (lambda: enc.encode(c0, None, S.KIND_BASE, out=bufs[0]),
                   lambda: enc.encode(c1, None, S.KIND_DELTA, out=bufs[1])):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            res = fn()
            torch.cuda.synchronize(dev)
            t.append((time.perf_counter() - t0, res))
        chain = [t[0][1], t[1][1]]
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        out = S.decode_chain(chain, to_host=False)
        torch.cuda.synchronize(dev)
        tl = time.perf_counter() - t0
        del out
        for k, v in (("save_base_s", t[0][0]), ("save_delta_s", t[1][0]), ("load_s", tl)):
            best[k] = min(best.get(k, 1e9), v)
    blob = chain[1][1].numel()
    try:
        with open(os.path.join(ROOT, "tests", "golden", "c0_ratio.json")) as f:
            ref = json.load(f)
    except Exception:
        ref = {}
    digest = hashlib.sha256(chain[1][1].numpy().tobytes()).hexdigest()
    return {"workload": "C0: GPT-2-small checkpoint (124.4M params, 148 tensors; bf16 weights, "
                        "fp32 Adam m/v, m = 16), base + delta save, chain restore",
            "raw_bytes": raw, "delta_blob_bytes": blob,
            "compression_ratio": round(raw / blob, 4),
            "reference": {"delta_blob_bytes": ref.get("delta_blob_bytes"),
                          "ratio": round(ref["ratio"], 4) if ref else None,
                          "blob_identical": digest == ref.get("blob_sha256"),
                          "source": "reference store.encode_checkpoint on the same inputs "
                                    "(tests/golden/make_c0_ratio.py)"},
            "published": {"delta_blob_bytes": C0_PUBLISHED_BLOB,
                          "reproduced": blob == C0_PUBLISHED_BLOB,
                          "source": "BASELINE.md §2 / SURVEY §6 (2.8400x)"},
            "save_delta_gbs": round(raw / best["save_delta_s"] / 1e9, 2),
            "save_base_gbs": round(raw / best["save_base_s"] / 1e9, 2),
            "load_gbs": round(raw / best["load_s"] / 1e9, 2),
            **{k: round(v, 4) for k, v in best.items()},
            "timing": "host wall clock per call, device-resident inputs, pinned host "
                      "outputs, best of 3 after one untimed pair"}


def run_c1_sweep(args, dev, world, reps: int = 3):
    """BASELINE configs[1] at every change fraction it names: encode, decode
    (out of place) and the in-place apply of chain replay, CUDA events per
    op, inputs resident in HBM (4 GiB >> L2)."""
    import torch
    from paper_2511_12376_b200 import bitmask as B
    from paper_2511_12376_b200 import _runtime as rt
    n = 1 << args.log2n
    hbm, kind = peaks()
    out = {}
    for p in (0.001, 0.01, 0.0625, 0.25):
        base, cur, k = make_c1(n, p, args.seed + 3, dev)
        mask = torch.empty((n + 7) // 8, dtype=torch.uint8, device=dev)
        pay = torch.empty(n, dtype=torch.int16, device=dev)
        res = torch.empty_like(base)
        work = base.clone()
        st = rt.new_status(dev, 3)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        t = [0.0, 0.0, 0.0]
        for r in range(reps + 1):
            work.copy_(base)
            torch.cuda.synchronize(dev)
            ev[0].record()
            B.encode_delta_async(base, cur, mask, pay, st[0])
            ev[1].record()
            B.decode_delta_async(base, mask, pay[:k], k, res, st[1])
            ev[2].record()
            B.decode_delta_async(work, mask, pay[:k], k, work, st[2])
            ev[3].record()
            torch.cuda.synchronize(dev)
            if r:
                for i in range(3):
                    t[i] += ev[i].elapsed_time(ev[i + 1]) / reps
        assert torch.equal(res, cur) and torch.equal(work, cur)
        mb = (n + 7) // 8
        nbytes = (4 * n + mb + 2 * k, mb + 2 * k + 4 * n, mb + 4 * k)
        row = {"n_c": k, "compression_ratio": round(2 * n / B.delta_size_bytes(n, k), 4)}
        for name, ms, b in zip(("encode", "decode", "apply_in_place"), t, nbytes):
            row[name + "_ms"] = round(ms, 4)
            row[name + "_gbs"] = round(b / (ms * 1e-3) / 1e9, 1)
            row[name + "_frac"] = round(b / (ms * 1e-3) / 1e9 / hbm, 4)
        out[f"p={p}"] = row
        del base, cur, mask, pay, res, work
    return {"workload": f"C1 sweep: 2^{args.log2n} bf16, p = 0.1 / 1 / 6.25 / 25 %",
            "bytes": "encode 4n + n/8 + 2n_c; decode n/8 + 2n_c + 4n; in-place n/8 + 4n_c "
                     "(SURVEY §8(d))", "peak": hbm, "peak_kind": kind, "points": out}


def run_c2_modes(args, dev, world, reps: int = 5):
    """BASELINE configs[2] in every form the bench quotes: Adam-m and Adam-v
    (v = |N(0,1e-3)|^2, one-sided, heavy-tailed), per 2^20 block and per
    tensor (the store's layout), m = 16; and the m sweep of SURVEY §8(d)
    (m = 2 / 4 / 8, Adam-m per block); encode and dequantize."""
    import torch
    from paper_2511_12376_b200 import quantizer as Q
    from paper_2511_12376_b200 import _runtime as rt
    n = 1 << args.c2_log2n
    hbm, kind = peaks()
    algo = 4 * n + n + (n + 1) // 2
    out = {}
    clocks = Clocks(dev.index or 0)
    clocks.start()
    for dist in ("adam_m", "adam_v"):
        g = torch.Generator(device=dev).manual_seed(args.seed + (7 if dist == "adam_m" else 8))
        x = torch.randn(n, device=dev, generator=g) * 1e-3
        if dist == "adam_v":
            x.mul_(x)
        runs = [(args.c2_block, 16), (0, 16)]
        if dist == "adam_m":
            runs += [(args.c2_block, mm) for mm in (2, 4, 8)]
        for block, m in runs:
            tables = Q.new_tables(n, block, dev)
            labels = torch.empty(Q.unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
            codes = torch.empty(n, dtype=torch.uint8, device=dev)
            res = torch.empty_like(x)
            st = rt.new_status(dev)
            # each op in its own loop (a save encodes, a restore dequantizes):
            # one untimed launch, then `reps` launches back to back between
            # two CUDA events (steady state, no host sync between launches)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            t = {}
            for op in ("encode", "dequantize"):
                def launch():
                    if op == "encode":
                        Q.cluster_encode_async(x, m, block, tables, labels, codes)
                    else:
                        Q.cluster_dequantize_async(labels, codes, n, block, tables, res, st)
                launch()
                torch.cuda.synchronize(dev)
                ev[0].record()
                for _ in range(reps):
                    launch()
                ev[1].record()
                torch.cuda.synchronize(dev)
                t[op] = ev[0].elapsed_time(ev[1]) / reps
            te, td = t["encode"], t["dequantize"]
            (maxlab, flags), = rt.read_status(st)
            assert flags == 0 and maxlab < m
            units = Q.num_units(n, block)
            enc_bytes = Q.serialized_quant_size("t", 1, block or n, m) * units
            key = f"{dist},block={block or 'tensor'}" + ("" if m == 16 else f",m={m}")
            out[key] = {
                "encode_ms": round(te, 4), "decode_ms": round(td, 4),
                "encode_gbs": round(algo / (te * 1e-3) / 1e9, 1),
                "decode_gbs": round(algo / (td * 1e-3) / 1e9, 1),
                "encode_frac": round(algo / (te * 1e-3) / 1e9 / hbm, 4),
                "decode_frac": round(algo / (td * 1e-3) / 1e9 / hbm, 4),
                "compression_ratio": round(4 * n / enc_bytes, 4),
                "max_abs_err": float((res - x).abs().max())}
            del tables, labels, codes, res
        del x
    clk = clocks.stop()
    return {"workload": f"C2 modes: 2^{args.c2_log2n} fp32, m = 16 (and m = 2 / 4 / 8 for "
                        "Adam-m per block)", "algorithmic_bytes": algo,
            "peak": hbm, "peak_kind": kind, "points": out, "clocks": clk}


def run_ckpt_sharded(config, dev, rank, world, reps: int = 2):
    """A whole checkpoint sharded over the job: every rank
    generates ITS share of the planner's LPT plan (bf16 w0 / w1 and the fp32
    optimizer states, tools/bench_checkpoint.py shapes), saves a base and a
    delta with planner.encode_sharded (its own GPU's encode + ONE all-gather
    of the size table) landing its records in pinned host memory at their
    global offsets, and restores its share with decode_chain (bit-exact
    check of the weights).  Box GB/s = the checkpoint's raw bytes / the
    slowest rank's time (barrier to completion)."""
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bench_checkpoint as BC
    from bench_checkpoint import generate, shapes, shard_names
    from paper_2511_12376_b200 import planner as PL
    from paper_2511_12376_b200 import store as S
    from paper_2511_12376_b200.tensors import ElementType
    only, lplan = shard_names(config, rank, world)
    torch.cuda.empty_cache()
    # specs of the WHOLE checkpoint in checkpoint order; every state of a
    # layer tensor goes to the rank the LPT plan gave the tensor
    shp = shapes(config)
    owner_of = dict(zip((nm for nm, _ in shp), lplan.owner))
    numel = {nm: int(torch.Size(sz).numel()) for nm, sz in shp}
    specs, owner = [], []
    for nm, _ in shp:
        specs.append(PL.TensorSpec(nm, "model", 2 * numel[nm]))
        owner.append(owner_of[nm])
    pre = ["master.", BC.M_PREFIX, BC.V_PREFIX] if config == "C3" else [BC.M_PREFIX, BC.V_PREFIX]
    for nm, _ in shp:
        for p in pre:
            specs.append(PL.TensorSpec(p + nm, "optimizer", 4 * numel[nm]))
            owner.append(owner_of[nm])
    load = [0] * world
    for sp, r in zip(specs, owner):
        load[r] += sp.nbytes
    plan = PL.ShardPlan(world=world, owner=tuple(owner), load=tuple(load))
    raw_total = sum(sp.nbytes for sp in specs)
    mine = plan.local_ids(rank)
    # any encoding fits: a model state at most raw, an fp32 optimizer state
    # always quantized (1.5 B per element), plus headers (store.blob_bound)
    bound = sum(sp.nbytes if sp.group == "model" else 3 * sp.nbytes // 8
                for sp in (specs[i] for i in mine)) + 512 * (len(mine) + 1)
    import numpy as np
    from paper_2511_12376_b200 import _runtime as rt
    # two registered landing buffers per rank: check the node's free host
    # memory first (every rank must agree, or the collectives below hang)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = None
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    need = 2 * bound * local_world
    # and this GPU's free HBM for its share: the base and current states
    # plus the encoder's arenas and the restore (a C4 rank of 8: 103.5 GB of
    # states, 129 GB peak, profiles/r02_dryrun_c4_rank2of8.json)
    model_mine = sum(specs[i].nbytes for i in mine if specs[i].group == "model")
    dev_need = int(1.3 * (plan.load[rank] + model_mine)) + (4 << 30)   # w0 and w1 both resident
    dev_free = torch.cuda.mem_get_info(dev)[0]
    host_ok = avail is None or need < 0.85 * avail
    ok = torch.tensor([1 if host_ok else 0, 1 if dev_need < dev_free else 0], dtype=torch.int64)
    if world > 1:
        if dist.get_backend() == "nccl":
            ok = ok.to(dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if int(ok[0].item()) == 0 or int(ok[1].item()) == 0:
        why = (f"host memory: {need / 1e9:.0f} GB of landing buffers for {local_world} "
               f"rank(s), {(avail or 0) / 1e9:.0f} GB available" if int(ok[0].item()) == 0 else
               f"device memory: a rank's share needs ~{dev_need / 1e9:.0f} GB of HBM, "
               f"{dev_free / 1e9:.0f} GB free on rank {rank}'s GPU (or another rank's)")
        return {"key": f"{config.lower()}_sharded", "skipped": why}
    c0, c1 = generate(config, dev, only=only)
    enc = S.CheckpointEncoder(dev, clusters=16, keep_prev="borrow")
    loc0 = {t.name: t for t in list(c0.model_states) + list(c0.optimizer_states)}
    loc1 = {t.name: t for t in list(c1.model_states) + list(c1.optimizer_states)}
    prev = {t.name: t for t in c0.model_states}
    host = [np.empty(bound, dtype=np.uint8) for _ in range(2)]
    for a in host:   # page-locked by registration (the caching allocator rounds up to 2^k)
        assert rt.lib().bsnp_host_register(a.ctypes.data, bound) == 0, "host register failed"
    bufs = [torch.from_numpy(a) for a in host]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def save(kind, local, it, buf):
        res = PL.encode_sharded(specs, local, prev if kind == "delta" else None, kind, it,
                                0, rank, world, enc, plan=plan, out=buf)
        return res, res.local_offsets

    times = {}
    for _ in range(reps):
        for key, kind, it, buf in (("save_base_s", "base", 0, bufs[0]),
                                   ("save_delta_s", "delta", 1, bufs[1])):
            barrier()
            t0 = time.perf_counter()
            r = save(kind, loc0 if kind == "base" else loc1, it, buf)
            torch.cuda.synchronize(dev)
            times[key] = min(times.get(key, 1e9), time.perf_counter() - t0)
            if kind == "base":
                rb = r
            else:
                rd = r
    del r
    # restore this rank's share: its records form a chain of local blobs
    def local_link(res, offs, buf):
        ents = tuple(S.ManifestEntry(rec.name, rec.group, rec.codec, o, rec.length)
                     for rec, o in zip(res.records, offs))
        man = S.CheckpointManifest(iteration=res.manifest.iteration, kind=res.manifest.kind,
                                   base_iteration=res.manifest.base_iteration, tensors=ents)
        return man, buf[:offs[-1]]
    chain = [local_link(*rb, bufs[0]), local_link(*rd, bufs[1])]
    # the restore needs the HBM the inputs hold (a C3 rank: 108 GB of states
    # + 75 GB of dequantized optimizer states): keep only the weights to
    # compare with
    def digest(flat):  # position-weighted sum of the bit patterns (exact, in int64)
        v = flat.reshape(-1).view(torch.int16).to(torch.int64)
        i = torch.arange(v.numel(), device=v.device, dtype=torch.int64) % 1000003 + 1
        return int(v.sum()), int(((v + 40000) * i).sum())

    want = {t.name: digest(t.flat()) for t in c1.model_states}
    del c0, c1, loc0, loc1, prev, enc
    torch.cuda.empty_cache()
    barrier()
    t0 = time.perf_counter()
    restored = S.decode_chain(chain, device=dev, to_host=False)
    torch.cuda.synchronize(dev)
    times["load_s"] = time.perf_counter() - t0
    exact = all(digest(t.data) == want[t.name] for t in restored.model_states) and \
        len(restored.model_states) == len(want)
    blob = rd[1][-1] if rd[1] else 0
    del restored, want, chain, rb, rd
    torch.cuda.synchronize(dev)
    for a in host:
        rt.lib().bsnp_host_unregister(a.ctypes.data)
    del bufs, host
    stats = torch.tensor([times["save_base_s"], times["save_delta_s"], times["load_s"],
                          float(blob), 0.0 if exact else 1.0], dtype=torch.float64)
    if world > 1:
        if dist.get_backend() == "nccl":
            stats = stats.to(dev)
        gathered = [torch.zeros_like(stats) for _ in range(world)]
        dist.all_gather(gathered, stats)
        stats_all = torch.stack([g.cpu() for g in gathered])
    else:
        stats_all = stats[None]
    mx = stats_all.max(dim=0).values.tolist()
    blob_total = int(stats_all[:, 3].sum())
    return {"key": f"{config.lower()}_sharded",
            "workload": f"{config} whole checkpoint sharded over {world} rank(s): base + delta "
                        "save (planner.encode_sharded, one size-table all-gather, records landed "
                        "in pinned host memory), restore of each rank's share (decode_chain)",
            "ranks": world, "raw_bytes": raw_total, "delta_blob_bytes": blob_total,
            "compression_ratio": round(raw_total / max(blob_total, 1), 4),
            "plan_imbalance": round(plan.imbalance, 4),
            "save_base_s": round(mx[0], 4), "save_delta_s": round(mx[1], 4),
            "load_s": round(mx[2], 4),
            "save_delta_box_gbs": round(raw_total / mx[1] / 1e9, 2),
            "save_base_box_gbs": round(raw_total / mx[0] / 1e9, 2),
            "load_box_gbs": round(raw_total / mx[2] / 1e9, 2),
            "restored_bit_exact": mx[4] == 0.0,
            "timing": "host wall clock per rank from a barrier, max over ranks; best of "
                      f"{reps} saves, one restore"}


def run_c2(args, dev, world):
    """BASELINE configs[2] on the same GPU: 2^30 fp32 Adam-m-shaped state,
    one cluster table per 2^20-element block, m = 16 (4-bit labels + u8
    codes).  encode = build_clusters + quantize of every block,
    decode = dequantize; both 5.5 bytes/element algorithmic."""
    import torch
    import torch.distributed as dist
    from paper_2511_12376_b200 import quantizer as Q
    from paper_2511_12376_b200 import _runtime as rt
    n, block, m = 1 << args.c2_log2n, args.c2_block, 16
    g = torch.Generator(device=dev).manual_seed(args.seed + 7)
    x = torch.randn(n, device=dev, generator=g) * 1e-3
    tables = Q.new_tables(n, block, dev)
    labels = torch.empty(Q.unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
    codes = torch.empty(n, dtype=torch.uint8, device=dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    st = rt.new_status(dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(3, args.warmup)):
        Q.cluster_encode_async(x, m, block, tables, labels, codes)
        Q.cluster_dequantize_async(labels, codes, n, block, tables, out, st)
    torch.cuda.synchronize(dev)
    (maxlab, flags), = rt.read_status(st)
    assert flags == 0 and maxlab < m
    err = float((out - x).abs().max())
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    if world > 1:
        dist.barrier()
    te = td = 0.0
    clocks = Clocks(dev.index or 0)
    clocks.start()
    for _ in range(args.steps):
        ev[0].record(stream)
        Q.cluster_encode_async(x, m, block, tables, labels, codes)
        ev[1].record(stream)
        Q.cluster_dequantize_async(labels, codes, n, block, tables, out, st)
        ev[2].record(stream)
        torch.cuda.synchronize(dev)
        te += ev[0].elapsed_time(ev[1])
        td += ev[1].elapsed_time(ev[2])
    clk = clocks.stop()
    te /= args.steps
    td /= args.steps
    if world > 1:
        te, td = max_over_ranks([te, td], dev)
    units = Q.num_units(n, block)
    algo = 4 * n + n + (n + 1) // 2            # read x, write codes + labels
    enc_bytes = Q.serialized_quant_size("t", 1, block, m) * units
    hbm, kind = peaks()
    enc_gbs = world * algo / (te * 1e-3) / 1e9
    dec_gbs = world * algo / (td * 1e-3) / 1e9
    traffic = ncu_traffic().get("cluster_encode")
    return {"workload": "C2: 2^%d fp32 ~N(0,1e-3), block %d, m=%d" % (args.c2_log2n, block, m),
            "encode_ms": round(te, 4), "decode_ms": round(td, 4),
            "encode_gbs": round(enc_gbs, 1), "decode_gbs": round(dec_gbs, 1),
            "roofline_encode": {"bound": "hbm", "achieved": round(enc_gbs / world, 1),
                                "peak": hbm, "peak_kind": kind, "unit": "GB/s",
                                "frac": round(enc_gbs / world / hbm, 4),
                                "frac_of_nominal_8000": round(enc_gbs / world / NOMINAL_HBM_GBS, 4),
                                "algorithmic_bytes": algo,
                                "traffic": traffic["bytes"] if traffic else None,
                                "traffic_detail": traffic},
            "roofline_decode": {"bound": "hbm", "achieved": round(dec_gbs / world, 1),
                                "peak": hbm, "peak_kind": kind, "unit": "GB/s",
                                "frac": round(dec_gbs / world / hbm, 4),
                                "frac_of_nominal_8000": round(dec_gbs / world / NOMINAL_HBM_GBS, 4),
                                "algorithmic_bytes": algo,
                                "traffic": (ncu_traffic().get("cluster_dequantize") or {})
                                .get("bytes"),
                                "traffic_detail": ncu_traffic().get("cluster_dequantize")},
            "compression_ratio": round(4 * n / enc_bytes, 4),
            "max_abs_err": err, "clocks": clk}


def run_e2e(args, base, cur, k, dev, world):
    """Encode + decode through pinned host memory (H2D inputs, D2H results)."""
    import torch
    import torch.distributed as dist
    from paper_2511_12376_b200 import hostpath

    n = base.numel()
    base_h = base.cpu().pin_memory()
    cur_h = cur.cpu().pin_memory()
    codec = hostpath.HostDeltaCodec(dev, n)
    for _ in range(max(1, args.warmup)):
        rec, out_h = codec.roundtrip(base_h, cur_h)
    assert rec.n_c == k and torch.equal(out_h, cur_h)
    # the record that reached the host is complete: its mask holds k changes
    import numpy as np
    assert int(np.bitwise_count(rec.mask.numpy()).sum()) == k
    steps = max(2, args.steps // 2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(steps):
        rec, out_h = codec.roundtrip(base_h, cur_h)
    torch.cuda.synchronize(dev)
    dt = (time.perf_counter() - t0) / steps
    if world > 1:
        dt, = max_over_ranks([dt], dev)
    eb, db = algo_bytes(n, k)
    mask = (n + 7) // 8
    return {"value": round(world * (eb + db) / dt / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": 4 * n + mask + 2 * k,
            "d2h_bytes_per_step": mask + 2 * k + 2 * n,
            "ms_per_step": round(dt * 1e3, 3), "steps": steps,
            "path": "hostpath.HostDeltaCodec.roundtrip: pinned host base+current H2D once, "
                    "encode, record D2H, decode onto the resident base, restored tensor D2H "
                    "(32 chunks; 3 encode + 2 decode streams, decode 4 chunks behind)"}


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # BSNP_DIST_BACKEND=gloo (test only): exercise the multi-rank code path
    # with several ranks sharing fewer GPUs; the driver's runs use NCCL
    backend = os.environ.get("BSNP_DIST_BACKEND", "nccl")
    if backend != "nccl":
        import torch
        local_rank %= max(1, torch.cuda.device_count())
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1 or os.environ.get("BSNP_FORCE_PG"):
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        run_b200(args, rank, world, local_rank)
    finally:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
