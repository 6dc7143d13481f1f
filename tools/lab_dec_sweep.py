"""Bitmask decode lab: build a variant of _bsnp.so with EXTRA nvcc flags and
time the out-of-place decode and the in-place (validated) chain-replay apply
over PS (dev tool; CUDA events, 10 reps, results checked)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2511_12376_b200 import _build, _lib
tag = os.environ["TAG"]; extra = os.environ.get("EXTRA", "").split()
so = _build.build(out=f"/tmp/_bsnp_{tag}.so", extra=extra)
_lib.SO_PATH = so
from paper_2511_12376_b200 import bitmask as B, _runtime as rt
dev = torch.device("cuda:0"); n = 1 << 30
for p in [float(x) for x in os.environ.get("PS", "0.001 0.01").split()]:
    base, cur, k = bench.make_c1(n, p, 0, dev)
    mask = torch.empty(n // 8, dtype=torch.uint8, device=dev); pay = torch.empty(n, dtype=torch.int16, device=dev)
    st = rt.new_status(dev, 2)
    B.encode_delta_async(base, cur, mask, pay, st[0])
    out = torch.empty_like(base); work = base.clone()
    td = ta = 0.0
    for r in range(11):
        work.copy_(base)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        e[0].record()
        B.decode_delta_async(base, mask, pay[:k], k, out, st[1])
        e[1].record()
        B.decode_delta_async(work, mask, pay[:k], k, work, st[1])
        e[2].record(); torch.cuda.synchronize()
        if r:
            td += e[0].elapsed_time(e[1]) / 10
            ta += e[1].elapsed_time(e[2]) / 10
    assert torch.equal(out, cur) and torch.equal(work, cur)
    print(f"{tag} p={p}: decode {td:.4f} ms | in-place apply {ta:.4f} ms", flush=True)
    del base, cur, mask, pay, out, work
