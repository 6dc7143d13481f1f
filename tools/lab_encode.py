"""Encode-kernel lab: timing + decoupled look-back statistics (dev tool)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_12376_b200 import _build, _lib

W = os.environ.get("LB_WIDTH", "4")
KLB = os.environ.get("KLB", "2")
SPIN = os.environ.get("SPIN", "128")
so = _build.build(out=f"/tmp/_bsnp_dbg{W}_{KLB}_{SPIN}.so",
                  extra=["-DBSNP_LOOKBACK_STATS", f"-DBSNP_LB_WIDTH={W}", f"-DBSNP_KLB={KLB}",
                         f"-DBSNP_SPIN_NS={SPIN}"])
_lib.SO_PATH = so
lib = _lib.load()
lib.bsnpdbg_lookback_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
import bench
from paper_2511_12376_b200 import bitmask as B, _runtime as rt
dev = torch.device("cuda:0")
for log2n in (30,):
    for p in (0.001, 0.01, 0.25):
        n = 1 << log2n
        base, cur, k = bench.make_c1(n, p, 0, dev)
        mask = torch.empty(n // 8, dtype=torch.uint8, device=dev)
        pay = torch.empty(n, dtype=torch.int16, device=dev)
        st = rt.new_status(dev)
        for _ in range(2):
            B.encode_delta_async(base, cur, mask, pay, st)
        torch.cuda.synchronize()
        stats = (ctypes.c_ulonglong * 4)()
        lib.bsnpdbg_lookback_stats(stats, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        R = 5
        for _ in range(R):
            B.encode_delta_async(base, cur, mask, pay, st)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / R
        lib.bsnpdbg_lookback_stats(stats, 1)
        calls = max(stats[0], 1)
        eb, _ = bench.algo_bytes(n, k)
        print(f"log2n={log2n} p={p}: {ms:.3f} ms  {eb/ms/1e6:.0f} GB/s  windows/tile={stats[1]/calls:.2f} spins/tile={stats[2]/calls:.2f}", flush=True)
        del base, cur, mask, pay
