"""Run the fused quantizer once with the watchdog build and dump wait timeouts."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_12376_b200 import _build, _lib
so = _build.build(out="/tmp/_bsnp_wd.so", extra=["-DBSNP_WATCHDOG"])
_lib.SO_PATH = so
lib = _lib.load()
lib.bsnpdbg_watchdog.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
from paper_2511_12376_b200 import quantizer as Q
dev = torch.device("cuda:0")
n = int(os.environ.get("N", str(3 << 20))); block = int(os.environ.get("BLOCK", str(1 << 20)))
x = torch.randn(n, device=dev) * 1e-3
tables = Q.new_tables(n, block, dev)
labels = torch.empty(Q.unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
codes = torch.empty(n, dtype=torch.uint8, device=dev)
Q.cluster_encode_async(x, 16, block, tables, labels, codes)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 256)(); cnt = ctypes.c_uint()
lib.bsnpdbg_watchdog(buf, ctypes.byref(cnt))
print("timeouts:", cnt.value)
names = {1: "producer empty", 2: "consumer full", 3: "xbar sum", 4: "xbar minmax"}
prog = (ctypes.c_uint * (1024 * 10))()
lib.bsnpdbg_progress(prog)
for b in range(32):
    row = list(prog[b*10:(b+1)*10])
    if any(row): print("cta", b, "consumer warps k:", row[:8], "producer k:", row[9])
for i in range(min(cnt.value, 64)):
    w0, a, b, c = buf[4*i:4*i+4]
    print(f"site={names.get(w0>>32)} block={(w0>>8)&0xffffff} warp={w0&0xff} k={a & 0xffffffff} producer_k={a>>32} u={b} c={c & 0xffffffff} rank={c>>32}")
