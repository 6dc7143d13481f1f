"""Per-phase cycle accounting of the fused encoder (watchdog/timing build)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_12376_b200 import _build, _lib
extra = ["-DBSNP_WATCHDOG"] + os.environ.get("EXTRA", "").split()
so = _build.build(out="/tmp/_bsnp_tm%d.so" % len(extra), extra=[e for e in extra if e])
_lib.SO_PATH = so
lib = _lib.load()
lib.bsnpdbg_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
from paper_2511_12376_b200 import quantizer as Q
dev = torch.device("cuda:0")
n = 1 << int(os.environ.get("LOG2N", "28")); block = 1 << 20
x = torch.randn(n, device=dev) * 1e-3
tables = Q.new_tables(n, block, dev)
labels = torch.empty(Q.unit_label_bytes(n, block), dtype=torch.uint8, device=dev)
codes = torch.empty(n, dtype=torch.uint8, device=dev)
Q.cluster_encode_async(x, 16, block, tables, labels, codes); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)(); lib.bsnpdbg_timing(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); Q.cluster_encode_async(x, 16, block, tables, labels, codes); e1.record(); torch.cuda.synchronize()
lib.bsnpdbg_timing(buf, 0)
tot = sum(buf[:7])
names = ["wait_full", "p0 sum", "p1 var", "p2 minmax", "p3 quant", "sync/sched", "exchange"]
print(f"kernel {e0.elapsed_time(e1):.3f} ms; thread-0 cycle shares:")
for i, nm in enumerate(names): print(f"  {nm:12s} {100*buf[i]/tot:5.1f}%  ({buf[i]/1e6:.1f} Mcyc)")
