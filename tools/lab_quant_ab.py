"""Quantizer A/B lab: time the C2 encode + dequantize (Adam-m / Adam-v, per
2^20 block and per tensor; CUDA events, 5 reps after 2) with the library
SO (default: the in-tree _bsnp.so) — run once per library and compare; dev
tool."""
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
n = 1 << 30
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
        e1.record()
        torch.cuda.synchronize()
        import hashlib
        dig = hashlib.sha256(labels.cpu().numpy().tobytes() + codes.cpu().numpy().tobytes()
                             + tables.cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"{tag} {dist} block={block or 'tensor'}: encode {e0.elapsed_time(e1) / 5:.4f} ms "
              f"digest {dig}", flush=True)
        del tables, labels, codes
    del x
