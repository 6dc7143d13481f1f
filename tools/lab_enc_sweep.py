import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2511_12376_b200 import _build, _lib
tag = os.environ["TAG"]; extra = os.environ.get("EXTRA", "").split()
so = _build.build(out=f"/tmp/_bsnp_{tag}.so", extra=extra)
_lib.SO_PATH = so
from paper_2511_12376_b200 import bitmask as B, _runtime as rt
dev = torch.device("cuda:0"); n = 1 << 30
for p in [float(x) for x in os.environ.get("PS", "0.01 0.0625 0.25").split()]:
    base, cur, k = bench.make_c1(n, p, 0, dev)
    mask = torch.empty(n // 8, dtype=torch.uint8, device=dev); pay = torch.empty(n, dtype=torch.int16, device=dev)
    st = rt.new_status(dev)
    for _ in range(2): B.encode_delta_async(base, cur, mask, pay, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): B.encode_delta_async(base, cur, mask, pay, st)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10; eb, _ = bench.algo_bytes(n, k)
    print(f"{tag} p={p}: encode {ms:.3f} ms {eb/ms/1e6:.0f} GB/s", flush=True)
    del base, cur, mask, pay
