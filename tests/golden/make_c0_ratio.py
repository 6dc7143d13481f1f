"""Run the REFERENCE store's encode_checkpoint (store.py:214-272) on the C0
checkpoint pair of SURVEY §8(d)'s recipe (tools/bench_checkpoint.py
generate_cpu_recipe: one CPU torch.Generator seeded 0) and record the blob
sizes, so the GPU bench can check it reproduces the reference's compression
ratio on the same inputs byte for byte.  Needs /root/reference (this
container only); writes tests/golden/c0_ratio.json."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np
import torch

from bitsnap import store as RS
from bitsnap.tensors import Checkpoint, ElementType, TensorBlob
from bench_checkpoint import M_PREFIX, V_PREFIX, shapes

g = torch.Generator().manual_seed(0)
m0, m1, opt = [], [], []
for name, shp in shapes("C0"):
    w0 = torch.randn(shp, generator=g) * 0.02
    u = torch.randn(shp, generator=g)
    w1 = w0 - 1e-5 * u
    m = torch.randn(shp, generator=g) * 1e-3
    v = (torch.randn(shp, generator=g) * 1e-3) ** 2
    b = lambda t: t.to(torch.bfloat16).view(torch.int16).numpy().astype("<i2").tobytes()
    m0.append(TensorBlob(name, ElementType.F16, tuple(shp), b(w0)))
    m1.append(TensorBlob(name, ElementType.F16, tuple(shp), b(w1)))
    opt.append(TensorBlob(M_PREFIX + name, ElementType.F32, tuple(shp), m.numpy().astype("<f4").tobytes()))
    opt.append(TensorBlob(V_PREFIX + name, ElementType.F32, tuple(shp), v.numpy().astype("<f4").tobytes()))
c0 = Checkpoint(iteration=0, model_states=tuple(m0), optimizer_states=tuple(opt))
c1 = Checkpoint(iteration=1, model_states=tuple(m1), optimizer_states=tuple(opt))
t = time.time()
man, blob = RS.encode_checkpoint(c1, c0, RS.KIND_DELTA, 16)
el = time.time() - t
raw = sum(len(x.data) for x in list(c1.model_states) + list(c1.optimizer_states))
wb = sum(e.length for e in man.tensors if e.group == "model")
ob = sum(e.length for e in man.tensors if e.group != "model")
out = {"config": "C0 (GPT-2-small), SURVEY §8(d) CPU-generator recipe, seed 0",
       "raw_bytes": raw, "delta_blob_bytes": len(blob), "ratio": raw / len(blob),
       "weights_ratio": sum(len(x.data) for x in c1.model_states) / wb,
       "optimizer_ratio": sum(len(x.data) for x in c1.optimizer_states) / ob,
       "blob_sha256": hashlib.sha256(blob).hexdigest(),
       "manifest_sha256": hashlib.sha256(man.to_bytes()).hexdigest(),
       "reference_encode_s": round(el, 1)}
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "c0_ratio.json"), "w"), indent=1)
print(out)
