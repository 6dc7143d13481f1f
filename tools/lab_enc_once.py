"""One C1 encode at P (default 0.25) after a warm-up (for ncu; dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2511_12376_b200 import bitmask as B, _runtime as rt

dev = torch.device("cuda:0")
n = 1 << 30
base, cur, k = bench.make_c1(n, float(os.environ.get("P", "0.25")), 0, dev)
mask = torch.empty(n // 8, dtype=torch.uint8, device=dev)
pay = torch.empty(n, dtype=torch.int16, device=dev)
st = rt.new_status(dev)
for _ in range(2):
    B.encode_delta_async(base, cur, mask, pay, st)
torch.cuda.synchronize()
print("ok")
