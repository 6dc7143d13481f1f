"""Quantizer lab: ONE C2-shaped encode after a warm-up (for ncu launch lists
and full captures of the encode kernels; DEQ=1 adds one dequantize; dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_12376_b200 import quantizer as Q

dev = torch.device("cuda:0")
n = 1 << int(os.environ.get("LOG2N", "30"))
block = 1 << int(os.environ.get("LOG2B", "20"))
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(n, device=dev, generator=g) * 1e-3
if os.environ.get("DIST") == "adam_v":
    x = x * x
tables = Q.new_tables(n, block, dev)
labels = torch.empty(Q.unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
codes = torch.empty(n, dtype=torch.uint8, device=dev)
for _ in range(int(os.environ.get("REPS", "2"))):
    Q.cluster_encode_async(x, int(os.environ.get("M", "16")), block, tables, labels, codes)
if os.environ.get("DEQ") == "1":  # and one dequantize of the result
    out = torch.empty_like(x)
    status = torch.zeros(4, dtype=torch.int64, device=dev)
    Q.cluster_dequantize_async(labels, codes, n, block, tables, out, status)
torch.cuda.synchronize()
print("ok")
