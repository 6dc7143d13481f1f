"""Bitmask lab: encode / decode / in-place apply (chain replay) timings over
the C1 change fractions (dev tool; CUDA events, inputs in HBM)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2511_12376_b200 import bitmask as B, _runtime as rt

dev = torch.device("cuda:0")
n = 1 << int(os.environ.get("LOG2N", "30"))
for p in (0.001, 0.01, 0.0625, 0.25):
    base, cur, k = bench.make_c1(n, p, 0, dev)
    mask = torch.empty((n + 7) // 8, dtype=torch.uint8, device=dev)
    pay = torch.empty(n, dtype=torch.int16, device=dev)
    out = torch.empty_like(base)
    work = base.clone()
    st = rt.new_status(dev, 3)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t = [0.0, 0.0, 0.0]
    R = 5
    for r in range(R + 1):
        work.copy_(base)
        torch.cuda.synchronize()
        ev[0].record()
        B.encode_delta_async(base, cur, mask, pay, st[0])
        ev[1].record()
        B.decode_delta_async(base, mask, pay[:k], k, out, st[1])
        ev[2].record()
        B.decode_delta_async(work, mask, pay[:k], k, work, st[2])   # in place
        ev[3].record()
        torch.cuda.synchronize()
        if r:
            for i in range(3):
                t[i] += ev[i].elapsed_time(ev[i + 1]) / R
    assert torch.equal(out, cur) and torch.equal(work, cur)
    mb = (n + 7) // 8
    enc_b, dec_b, app_b = 4 * n + mb + 2 * k, mb + 2 * k + 4 * n, mb + 4 * k
    print(f"p={p}: encode {t[0]:.3f} ms {enc_b / t[0] / 1e6:.0f} GB/s | decode {t[1]:.3f} ms "
          f"{dec_b / t[1] / 1e6:.0f} GB/s | in-place apply {t[2]:.3f} ms "
          f"{app_b / t[2] / 1e6:.0f} GB/s (algorithmic n/8 + 4 n_c)", flush=True)
