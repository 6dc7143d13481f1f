"""Quantizer lab: C2 encode (2^30 fp32, block 2^20, m=16) through
cluster_encode_async, CUDA events; prints a digest of the outputs so that
kernel variants can be compared for bit-identical results (dev tool).
M="2 4 8 16" sweeps the cluster count and adds the dequantize
time, the max abs error and the compression ratio of each."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_12376_b200 import quantizer as Q

dev = torch.device("cuda:0")
n = 1 << int(os.environ.get("LOG2N", "30"))
block = 1 << int(os.environ.get("LOG2B", "20"))
g = torch.Generator(device=dev).manual_seed(0)
ms = [int(v) for v in os.environ.get("M", "16").split()]
sweep = "M" in os.environ
for dist, m in [(d, m) for d in ("adam_m", "adam_v") for m in ms]:
    g = torch.Generator(device=dev).manual_seed(0 if dist == "adam_m" else 1)
    x = torch.randn(n, device=dev, generator=g) * 1e-3
    if dist == "adam_v":
        x = x * x
    tables = Q.new_tables(n, block, dev)
    labels = torch.empty(Q.unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
    codes = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(3):
        Q.cluster_encode_async(x, m, block, tables, labels, codes)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 10
    e0.record()
    for _ in range(R):
        Q.cluster_encode_async(x, m, block, tables, labels, codes)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / R
    h = hashlib.sha1()
    for a in (tables, labels, codes):
        h.update(a.cpu().numpy().tobytes())
    extra = ""
    if sweep:
        from paper_2511_12376_b200 import _runtime as rt
        out = torch.empty_like(x)
        st = rt.new_status(dev)
        Q.cluster_dequantize_async(labels, codes, n, block, tables, out, st)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(R):
            Q.cluster_dequantize_async(labels, codes, n, block, tables, out, st)
        e1.record()
        torch.cuda.synchronize()
        td = e0.elapsed_time(e1) / R
        units = (n + block - 1) // block
        rec = units * Q.serialized_quant_size("t", 1, block, m)
        ratio = f" ratio {4 * n / rec:.4f}x"
        extra = (f" | dequant {td:.3f} ms {5.5 * n / td / 1e6:.0f} GB/s | max|err| "
                 f"{float((out - x).abs().max()):.2e}{ratio}")
    print(f"{dist} m={m} block={block}: encode {t:.3f} ms -> {5.5 * n / t / 1e6:.0f} GB/s "
          f"({5.5 * n / t / 1e6 / 6458:.1%} of measured HBM){extra}  digest {h.hexdigest()[:16]}",
          flush=True)
