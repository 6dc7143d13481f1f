"""Randomised whole-checkpoint stress (dev tool): random checkpoints (1-60
tensors, shapes from empty to a few hundred thousand elements, random change
fractions and cluster counts) saved as chains through store.CheckpointEncoder
in every keep_prev mode, with host TensorBlobs or device-resident
DeviceTensors (the recorded-graph path when addresses repeat), into fresh or
reused pinned buffers; every blob and manifest is compared with the oracle's
encode_checkpoint and every chain is restored with decode_chain.

    python tools/stress_store.py [seconds]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import bitsnap_oracle as O
from paper_2511_12376_b200 import store as S
from paper_2511_12376_b200.tensors import Checkpoint, ElementType, TensorBlob

dev = torch.device("cuda:0")
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(os.environ.get("SEED", "3")))


def shape():
    kind = rng.integers(0, 6)
    if kind == 0:
        return (0,)
    if kind == 1:
        return (int(rng.integers(1, 9)),)
    if kind == 2:
        return (int(rng.integers(1, 300)), int(rng.integers(1, 300)))
    if kind == 3:
        return (int(rng.integers(8000, 9000)),)
    return (int(rng.integers(1, 400_000)),)


def make(spec, prev=None, it=0):
    model, opt = [], []
    for i, (shp, frac) in enumerate(spec["model"]):
        n = int(np.prod(shp))
        if prev is None:
            a = rng.integers(0, 1 << 16, n, dtype=np.uint16)
        else:
            a = np.frombuffer(prev.model_states[i].data, np.uint16).copy()
            k = int(n * frac)
            if k:
                a[rng.choice(n, k, replace=False)] ^= rng.integers(1, 1 << 16, k, dtype=np.uint16)
        model.append(TensorBlob(f"m{i}", ElementType.F16, shp, a.tobytes()))
    for i, (shp, scale) in enumerate(spec["opt"]):
        n = int(np.prod(shp))
        x = (rng.standard_normal(n) * scale).astype(np.float32)
        if i % 3 == 1:
            x = x * x
        opt.append(TensorBlob(f"o{i}", ElementType.F32, shp, x.tobytes()))
    return Checkpoint(iteration=it, model_states=model, optimizer_states=opt)


def oracle(ck, prev, kind, clusters):
    conv = lambda ts, code: [(t.name, t.shape, code,
                              np.frombuffer(t.data, np.uint16 if code == 0 else np.float32))
                             for t in ts]
    return O.encode_checkpoint(conv(ck.model_states, 0), conv(ck.optimizer_states, 1),
                               conv(prev.model_states, 0) if prev else None, kind, clusters)


def on_device(ck, bufs):
    """DeviceTensors over persistent buffers (same addresses every save)."""
    out = []
    for t in ck.model_states + ck.optimizer_states:
        dt = torch.int16 if t.dtype is ElementType.F16 else torch.float32
        src = torch.frombuffer(bytearray(t.data), dtype=dt) if t.nbytes else torch.empty(0, dtype=dt)
        b = bufs.get(t.name)
        if b is None or b.numel() != src.numel():
            b = bufs[t.name] = torch.empty(src.numel(), dtype=dt, device=dev)
        b.copy_(src)
        out.append(S.DeviceTensor(t.name, t.dtype, t.shape, b))
    nm = len(ck.model_states)
    return Checkpoint(iteration=ck.iteration, model_states=out[:nm], optimizer_states=out[nm:])


t_end = time.time() + budget
cases = bad = 0
while time.time() < t_end:
    cases += 1
    clusters = int(rng.integers(2, 17))
    nm, no = int(rng.integers(1, 40)), int(rng.integers(0, 20))
    spec = {"model": [(shape(), float(rng.choice([0.0, 1e-3, 0.02, 0.3, 1.0]))) for _ in range(nm)],
            # (an empty optimizer state is rejected, as by the reference: quantizer.py:110-111)
            "opt": [(s if int(np.prod(s)) else (1,), float(10.0 ** rng.uniform(-6, 1)))
                    for s in (shape() for _ in range(no))]}
    links = int(rng.integers(2, 5))
    cks = [make(spec, it=10)]
    for j in range(1, links):
        cks.append(make(spec, cks[-1], 10 + j))
    keep = [True, "copy", "borrow", False][cases % 4]
    device_inputs = bool(rng.integers(0, 2)) and keep != "borrow"
    reuse_out = bool(rng.integers(0, 2))
    enc = S.CheckpointEncoder(dev, clusters=clusters, keep_prev=keep)
    bufs, chain, outbuf = {}, [], None
    try:
        for j, ck in enumerate(cks):
            kind = S.KIND_BASE if j == 0 else S.KIND_DELTA
            prev = cks[j - 1] if j else None
            arg = on_device(ck, bufs) if device_inputs else ck
            prev_arg = None
            if kind == S.KIND_DELTA and keep is False:
                prev_arg = prev
            if reuse_out:
                need = S.blob_bound(ck)
                if outbuf is None or outbuf.numel() < need:
                    outbuf = torch.empty(need, dtype=torch.uint8, pin_memory=True)
                man, blob = enc.encode(arg, prev_arg, kind, out=outbuf)
            else:
                man, blob = enc.encode(arg, prev_arg, kind)
            entries, want = oracle(ck, prev, kind, clusters)
            got = blob.numpy().tobytes()
            if got != want or [vars(e) for e in man.tensors] != entries:
                raise AssertionError(f"link {j} blob/manifest differs from the oracle")
            chain.append((man, got))
        rec = S.decode_chain(chain)
        for a, b in zip(rec.model_states, cks[-1].model_states):
            if a.data != b.data:
                raise AssertionError(f"restored {b.name} differs")
    except Exception as e:
        bad += 1
        print(f"MISMATCH case {cases}: clusters={clusters} tensors={nm}+{no} links={links} "
              f"keep={keep} device={device_inputs} reuse_out={reuse_out}: {e!r}", flush=True)
print(f"stress_store: {cases} cases, {bad} mismatches", flush=True)
