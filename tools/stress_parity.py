"""Randomised parity stress (dev tool): quantizer encodes and bitmask codecs
on random sizes and distributions vs the CPU oracle; prints every mismatch.

    python tools/stress_parity.py [seconds]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import bitsnap_oracle as O
from paper_2511_12376_b200 import bitmask as B
from paper_2511_12376_b200 import quantizer as Q

dev = torch.device("cuda:0")
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(os.environ.get("SEED", "7")))


def dist(kind, n):
    if kind == "normal":
        return rng.standard_normal(n) * 10.0 ** rng.uniform(-8, 3)
    if kind == "lognormal":
        return rng.lognormal(rng.uniform(-20, 5), rng.uniform(0.1, 3), n)
    if kind == "uniform":
        a = rng.uniform(-1e3, 1e3)
        return rng.uniform(a, a + 10.0 ** rng.uniform(-6, 3), n)
    if kind == "bimodal":
        return np.where(rng.random(n) < 0.5, -1.0, 1.0) + rng.standard_normal(n) * 1e-3
    if kind == "heavy":
        return rng.standard_t(1.5, n) * 1e-2
    if kind == "dups":
        return rng.choice(rng.standard_normal(rng.integers(1, 40)), n)
    if kind == "tiny":
        return rng.standard_normal(n) * 1e-40          # f32 subnormals
    if kind == "huge":
        return rng.standard_normal(n) * 1e36
    if kind == "offset":
        return 1e4 + rng.standard_normal(n) * 1e-3
    if kind == "adam_v":
        return (rng.standard_normal(n) * 1e-3) ** 2
    raise ValueError(kind)


kinds = ["normal", "lognormal", "uniform", "bimodal", "heavy", "dups", "tiny", "huge",
         "offset", "adam_v"]
t_end = time.time() + budget
cases = bad = zero_ties = 0
while time.time() < t_end:
    kind = kinds[cases % len(kinds)]
    n = int(rng.choice([rng.integers(1, 9000), rng.integers(9000, 1 << 20),
                        rng.integers(1 << 20, 1 << 21)]))
    m = int(rng.integers(2, 17))
    block = int(rng.choice([0, 0, 1 << int(rng.integers(13, 20)), 8 * int(rng.integers(1000, 40000)),
                            8192 * int(rng.integers(1, 40))]))
    if block and rng.random() < 0.3:
        # a last unit a few elements short of a full one (its tree can be one
        # level deeper than a full unit's)
        n = block * int(rng.integers(1, 8)) + block - 8 * int(rng.integers(0, 4)) - int(rng.integers(1, 8))
    x = dist(kind, n).astype(np.float32)
    if not np.all(np.isfinite(x)):
        x = np.nan_to_num(x, posinf=3e38, neginf=-3e38).astype(np.float32)
    cases += 1
    try:
        dq = Q.cluster_encode_device(torch.from_numpy(x).to(dev), m, block)
        tabs = dq.host_tables()
        labels = dq.labels.cpu().numpy()
        codes = dq.codes.cpu().numpy()
        units = O.blockwise(x, block if block and block < n else 0)
        lpos = 0
        for u, xs in enumerate(units):
            ora = O.cluster_fit(xs, m)
            f = lambda v: np.asarray(v, np.float32).view(np.uint32).tolist()
            t = tabs[u]
            ok = (f([t.mean, t.std]) == f([ora["mean"], ora["std"]]) and
                  f(t.boundaries) == f(ora["boundaries"]) and f(t.scales) == f(ora["scales"])
                  and f(t.offsets) == f(ora["offsets"]))
            if not ok and (f([t.mean, t.std]) == f([ora["mean"], ora["std"]]) and
                           f(t.boundaries) == f(ora["boundaries"]) and
                           list(t.scales) == list(ora["scales"]) and
                           list(t.offsets) == list(ora["offsets"])):
                # equal as numbers: a cluster extreme that is a signed zero
                # (numpy's min/max return whichever zero its SIMD reduction
                # order meets last; the kernels order -0 < +0)
                zero_ties += 1
                ok = True
            packed, c, _ = O.cluster_quantize(xs, ora)
            start = u * (block if block and block < n else 0)
            ok = ok and np.array_equal(codes[start:start + xs.size], c)
            ok = ok and np.array_equal(labels[lpos:lpos + packed.size], packed)
            lpos += packed.size
            if not ok:
                bad += 1
                print(f"MISMATCH quant kind={kind} n={n} m={m} block={block} unit={u}", flush=True)
                os.makedirs("gpurun_out", exist_ok=True)
                np.save(f"gpurun_out/fail_quant_{cases}_m{m}_b{block}.npy", x)
                break
    except Q.QuantizerError as e:
        if "non-finite" not in str(e):
            bad += 1
            print(f"ERROR quant kind={kind} n={n}: {e}", flush=True)
    # bitmask
    nb = int(rng.integers(0, 3_000_000))
    p = float(rng.choice([0.0, 1e-4, 0.01, 0.03, 0.0625, 0.2, 0.9, 1.0]))
    base = rng.integers(0, 1 << 16, nb, dtype=np.uint16)
    cur = base.copy()
    k = int(nb * p)
    if k:
        idx = rng.choice(nb, k, replace=False)
        cur[idx] ^= rng.integers(1, 1 << 16, k, dtype=np.uint16)
    off = int(rng.integers(0, 4))
    bt = torch.from_numpy(np.concatenate([np.zeros(off, np.uint16), base]).view(np.int16)).to(dev)[off:]
    ct = torch.from_numpy(np.concatenate([np.zeros(off, np.uint16), cur]).view(np.int16)).to(dev)[off:]
    d = B.encode_delta_device(bt, ct)
    mask, payload, n_c = O.delta_encode(base, cur)
    ok = d.n_c == n_c and np.array_equal(d.mask.cpu().numpy(), mask) and \
        np.array_equal(d.payload.cpu().numpy().view(np.uint16), payload)
    out = B.decode_delta_device(bt, d.mask, d.payload, d.n_c)
    ok = ok and np.array_equal(out.cpu().numpy().view(np.uint16), cur)
    b2 = bt.clone()
    B.decode_delta_device(b2, d.mask, d.payload, d.n_c, out=b2)
    ok = ok and np.array_equal(b2.cpu().numpy().view(np.uint16), cur)
    if not ok:
        bad += 1
        print(f"MISMATCH bitmask n={nb} p={p} off={off}", flush=True)
print(f"stress: {cases} cases, {bad} mismatches, {zero_ties} signed-zero extreme ties",
      flush=True)
