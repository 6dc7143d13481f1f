"""Quantizer lab: C2 timings (2^30 fp32, block 2^20, m=16) per kernel phase."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_12376_b200 import quantizer as Q, _runtime as rt
dev = torch.device("cuda:0")
log2n = int(os.environ.get("LOG2N", "30"))
n = 1 << log2n
g = torch.Generator(device=dev).manual_seed(0)
for dist in ("adam_m", "adam_v"):
    x = torch.randn(n, device=dev, generator=g) * 1e-3
    if dist == "adam_v":
        x = x * x
    for block in (1 << 20, 0):
        tables = Q.new_tables(n, block, dev)
        labels = torch.empty(Q.unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
        out = torch.empty(n, dtype=torch.float32, device=dev)
        st = rt.new_status(dev)
        def ev(): return torch.cuda.Event(enable_timing=True)
        for _ in range(2):
            Q.cluster_encode_async(x, 16, block, tables, labels, codes)
            Q.cluster_dequantize_async(labels, codes, n, block, tables, out, st)
        torch.cuda.synchronize()
        R = 5
        e = [ev() for _ in range(5)]
        t_fit = t_q = t_dq = 0
        for _ in range(R):
            e[0].record(); Q.cluster_fit_async(x, 16, block, tables); e[1].record()
            Q.cluster_quantize_async(x, block, tables, labels, codes); e[2].record()
            Q.cluster_dequantize_async(labels, codes, n, block, tables, out, st); e[3].record()
            torch.cuda.synchronize()
            t_fit += e[0].elapsed_time(e[1]); t_q += e[1].elapsed_time(e[2]); t_dq += e[2].elapsed_time(e[3])
        t_fit /= R; t_q /= R; t_dq /= R
        enc = t_fit + t_q
        print(f"{dist} block={block}: fit {t_fit:.3f} ms quant {t_q:.3f} ms -> encode {5.5*n/enc/1e6:.0f} GB/s; "
              f"dequant {t_dq:.3f} ms -> {5.5*n/t_dq/1e6:.0f} GB/s; max|err|={float((out-x).abs().max()):.3e}", flush=True)
