"""Per-tensor quantizer units at sizes where the pairwise tree has more than
1024 tiles (the pre-reduction path), random lengths and distributions, vs the
CPU oracle fanned over the host's cores (dev tool).

    python tools/stress_large.py [seconds]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import pool_oracle as PO
from paper_2511_12376_b200 import quantizer as Q

dev = torch.device("cuda:0")
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(os.environ.get("SEED", "5")))
t_end = time.time() + budget
cases = bad = 0
f = lambda v: np.asarray(v, np.float32).view(np.uint32).tolist()
while time.time() < t_end:
    cases += 1
    n = int(rng.integers(1 << 23, 1 << 26))
    if rng.random() < 0.3:  # just below a power of two: a deeper tree than the size suggests
        n = (1 << int(rng.integers(24, 27))) - int(rng.integers(1, 64))
    m = int(rng.integers(2, 17))
    kind = rng.integers(0, 3)
    x = rng.standard_normal(n) * 1e-3
    if kind == 1:
        x = x * x
    elif kind == 2:
        x = 1e3 + x
    x = x.astype(np.float32)
    dq = Q.cluster_encode_device(torch.from_numpy(x).to(dev), m, 0)
    (tab,) = dq.host_tables()
    ora = PO.cluster_fit(x, m)
    ok = (f([tab.mean, tab.std]) == f([ora["mean"], ora["std"]]) and
          f(tab.boundaries) == f(ora["boundaries"]) and f(tab.scales) == f(ora["scales"]) and
          f(tab.offsets) == f(ora["offsets"]))
    if ok:
        packed, codes, _ = PO.cluster_quantize(x, ora)
        ok = np.array_equal(dq.codes.cpu().numpy(), codes) and \
            np.array_equal(dq.labels.cpu().numpy(), packed)
    if not ok:
        bad += 1
        print(f"MISMATCH n={n} m={m} kind={kind}", flush=True)
print(f"stress_large: {cases} cases, {bad} mismatches", flush=True)
