"""Quantizer lab: build a variant of _bsnp.so with EXTRA nvcc flags (e.g.
"-DBSNP_WDELTA=160") and time the C2 encode and dequantize (Adam-m and Adam-v,
per 2^20 block and per tensor; CUDA events, 5 reps) — dev tool."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2511_12376_b200 import _build, _lib
tag = os.environ["TAG"]; extra = os.environ.get("EXTRA", "").split()
so = _build.build(out=f"/tmp/_bsnp_{tag}.so", extra=extra)
_lib.SO_PATH = so
from paper_2511_12376_b200 import quantizer as Q, _runtime as rt
dev = torch.device("cuda:0"); n = 1 << 30
for dist in ("adam_m", "adam_v"):
    g = torch.Generator(device=dev).manual_seed(7)
    x = torch.randn(n, device=dev, generator=g) * 1e-3
    if dist == "adam_v":
        x.mul_(x)
    for block in (1 << 20, 0):
        tables = Q.new_tables(n, block, dev)
        labels = torch.empty(Q.unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
        for _ in range(2):
            Q.cluster_encode_async(x, 16, block, tables, labels, codes)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            Q.cluster_encode_async(x, 16, block, tables, labels, codes)
        e1.record(); torch.cuda.synchronize()
        te = e0.elapsed_time(e1) / 5
        out = torch.empty_like(x)
        st = torch.zeros(4, dtype=torch.int64, device=dev)
        for _ in range(2):
            Q.cluster_dequantize_async(labels, codes, n, block, tables, out, st)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            Q.cluster_dequantize_async(labels, codes, n, block, tables, out, st)
        e1.record(); torch.cuda.synchronize()
        print(f"{tag} {dist} block={block or 'tensor'}: encode {te:.4f} ms | dequantize "
              f"{e0.elapsed_time(e1) / 5:.4f} ms", flush=True)
        del tables, labels, codes, out
    del x
