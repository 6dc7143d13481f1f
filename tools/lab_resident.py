"""Resident quantizer lab: C2 encode (fit+quantize, one call) timing and, with
a -DBSNP_RTIMING build, per-stage cycle counts of quant_resident_kernel."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_12376_b200 import quantizer as Q, _runtime as rt, _lib
dev = torch.device("cuda:0")
n = 1 << int(os.environ.get("LOG2N", "30"))
block = 1 << int(os.environ.get("LOG2B", "20"))
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(n, device=dev, generator=g) * 1e-3
tables = Q.new_tables(n, block, dev)
labels = torch.empty(Q.unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
codes = torch.empty(n, dtype=torch.uint8, device=dev)
lib = _lib.load()
dbg = getattr(lib, "bsnpdbg_rtiming", None)
for _ in range(3):
    Q.cluster_encode_async(x, 16, block, tables, labels, codes)
torch.cuda.synchronize()
if dbg:
    buf = (ctypes.c_ulonglong * 16)()
    dbg(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 5
e0.record()
for _ in range(R):
    Q.cluster_encode_async(x, 16, block, tables, labels, codes)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / R
print(f"encode n=2^{n.bit_length()-1} block={block}: {ms:.3f} ms -> {5.5*n/ms/1e6:.0f} GB/s", flush=True)
if dbg:
    dbg(buf, 0)
    v = list(buf)
    tiles = max(v[10], 1)
    names = ["load", "A", "wait_mean", "B", "wait_std", "-", "wait_table/exact", "wait_table", "D",
             "-", "-", "-", "C_setup", "C_filter", "C_publish"]
    print("tiles", v[10], "exact-round tiles", v[11])
    print(" ".join(f"{nm}={v[i]/tiles/1965:.2f}us" for i, nm in enumerate(names) if nm != "-"), flush=True)
