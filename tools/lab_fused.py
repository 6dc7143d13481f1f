"""Fused per-block encoder timing (C2 shape) + optional single run for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_12376_b200 import quantizer as Q, _runtime as rt
dev = torch.device("cuda:0")
n = 1 << int(os.environ.get("LOG2N", "30")); block = 1 << 20
x = torch.randn(n, device=dev) * 1e-3
tables = Q.new_tables(n, block, dev)
labels = torch.empty(Q.unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
codes = torch.empty(n, dtype=torch.uint8, device=dev)
reps = int(os.environ.get("REPS", "5"))
for _ in range(2):
    Q.cluster_encode_async(x, 16, block, tables, labels, codes)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    Q.cluster_encode_async(x, 16, block, tables, labels, codes)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"fused encode n=2^{n.bit_length()-1}: {ms:.3f} ms  {5.5*n/ms/1e6:.0f} GB/s", flush=True)
