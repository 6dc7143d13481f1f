"""Dequantize A/B lab: time the C2 dequantize (Adam-m / Adam-v, m = 16 / 8,
per 2^20 block; CUDA events, 10 reps after 2) with the library SO (default:
the in-tree _bsnp.so) and print a digest of the output — run once per
library and compare; dev tool."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_12376_b200 import _lib

if os.environ.get("SO"):
    _lib.SO_PATH = os.path.abspath(os.environ["SO"])
from paper_2511_12376_b200 import quantizer as Q

tag = os.environ.get("TAG", os.path.basename(_lib.SO_PATH))
dev = torch.device("cuda:0")
n, block = 1 << 30, 1 << 20
for dist in ("adam_m", "adam_v"):
    g = torch.Generator(device=dev).manual_seed(7)
    x = torch.randn(n, device=dev, generator=g) * 1e-3
    if dist == "adam_v":
        x.mul_(x)
    for m in (16, 8):
        tables = Q.new_tables(n, block, dev)
        labels = torch.empty(Q.unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
        Q.cluster_encode_async(x, m, block, tables, labels, codes)
        out = torch.empty_like(x)
        st = torch.zeros(4, dtype=torch.int64, device=dev)
        for _ in range(2):
            Q.cluster_dequantize_async(labels, codes, n, block, tables, out, st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            Q.cluster_dequantize_async(labels, codes, n, block, tables, out, st)
        e1.record()
        torch.cuda.synchronize()
        dig = hashlib.sha256(out.view(torch.int32).cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"{tag} {dist} m={m}: dequantize {e0.elapsed_time(e1) / 10:.4f} ms digest {dig}",
              flush=True)
        del tables, labels, codes, out
    del x
