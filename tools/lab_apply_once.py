"""C1 in-place apply (chain replay) at P after an encode (for ncu; dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2511_12376_b200 import bitmask as B, _runtime as rt

dev = torch.device("cuda:0")
n = 1 << 30
base, cur, k = bench.make_c1(n, float(os.environ.get("P", "0.01")), 0, dev)
mask = torch.empty(n // 8, dtype=torch.uint8, device=dev)
pay = torch.empty(n, dtype=torch.int16, device=dev)
st = rt.new_status(dev, 2)
B.encode_delta_async(base, cur, mask, pay, st[0])
work = base.clone()
for _ in range(2):
    B.decode_delta_async(work, mask, pay[:k], k, work, st[1])
torch.cuda.synchronize()
assert torch.equal(work, cur)
print("ok")
