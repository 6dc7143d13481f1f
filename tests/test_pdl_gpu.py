"""Programmatic dependent launch changes launch timing, never results: the
bitmask encode / decode / in-place apply and the cluster encode / dequantize
give the same bytes with BSNP_PDL=0 (ordinary launches) and the default (one
programmatic chain).  The switch is read once per process, so each setting
runs in its own interpreter."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

SNIPPET = r'''
import hashlib, sys
sys.path.insert(0, {root!r})
import torch, bench
from paper_2511_12376_b200 import bitmask as B, quantizer as Q, _runtime as rt
dev = torch.device("cuda:0")
h = hashlib.sha256()
n = (1 << 24) + 77
for p in (0.001, 0.25):
    base, cur, k = bench.make_c1(n, p, 3, dev)
    mask = torch.empty((n + 7) // 8, dtype=torch.uint8, device=dev)
    pay = torch.empty(n, dtype=torch.int16, device=dev)
    st = rt.new_status(dev, 3)
    B.encode_delta_async(base, cur, mask, pay, st[0])
    out = torch.empty_like(base)
    B.decode_delta_async_dn(base, mask, pay, st[0], out, st[1])
    work = base.clone()
    B.decode_delta_async(work, mask, pay[:k], k, work, st[2])
    torch.cuda.synchronize()
    assert torch.equal(out, cur) and torch.equal(work, cur)
    for t in (mask, pay[:k], st):
        h.update(t.cpu().numpy().tobytes())
g = torch.Generator(device=dev).manual_seed(5)
x = torch.randn(1 << 22, device=dev, generator=g) * 1e-3
for block in (1 << 18, 0):
    tables = Q.new_tables(x.numel(), block, dev)
    labels = torch.empty(Q.unit_label_bytes(x.numel(), block), dtype=torch.uint8, device=dev)
    codes = torch.empty(x.numel(), dtype=torch.uint8, device=dev)
    Q.cluster_encode_async(x, 16, block, tables, labels, codes)
    res = torch.empty_like(x)
    s = torch.zeros(4, dtype=torch.int64, device=dev)
    Q.cluster_dequantize_async(labels, codes, x.numel(), block, tables, res, s)
    torch.cuda.synchronize()
    for t in (tables, labels, codes, res):
        h.update(t.cpu().numpy().tobytes())
print(h.hexdigest())
'''


def _digest(pdl: str) -> str:
    env = dict(os.environ, BSNP_PDL=pdl)
    out = subprocess.run([sys.executable, "-c", SNIPPET.format(root=ROOT)], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    return out.stdout.strip().splitlines()[-1]


def test_programmatic_launch_does_not_change_bytes(dev):
    assert _digest("0") == _digest("1")
