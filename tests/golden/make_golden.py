"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `bitsnap` from /root/reference/pkg/src (read-only), feeds it
seeded inputs and stores inputs + the reference's serialized outputs as
compressed .npz fixtures next to this script.  The GPU box never needs the
reference: the fixtures travel with the repo.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = os.environ.get("BITSNAP_REF_SRC", "/root/reference/pkg/src")


def _ref():
    sys.path.insert(0, REF_SRC)
    import bitsnap  # noqa: F401  (the reference package)
    from bitsnap import bitmask, quantizer, store, tensors
    return bitmask, quantizer, store, tensors


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit pattern with round-to-nearest-even."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u >> 16) & 1) + 0x7FFF
    return ((u + r) >> 16).astype(np.uint16)


def bitmask_cases():
    rng = np.random.default_rng(20251115)
    cases = []
    # KAT 0x42 (reference test_bitmask.py:35-46)
    b = np.arange(8, dtype=np.uint16)
    c = b.copy(); c[1] = 1000; c[6] = 2000
    cases.append(("kat_0x42", b, c, (8,)))
    # identical n=100 -> 13 zero mask bytes (test_bitmask.py:27-32)
    b = rng.integers(0, 1 << 16, 100, dtype=np.uint16)
    cases.append(("identical_100", b, b.copy(), (100,)))
    # +-0 / NaN / inf patterns (test_bitmask.py:72-79, test_acceptance.py:49-52)
    cases.append(("signed_zero_nan", np.array([0x0000, 0x3C00, 0x0000], np.uint16),
                  np.array([0x8000, 0x7E00, 0x0000], np.uint16), (3,)))
    specials = np.array([0x0000, 0x8000, 0x7E00, 0xFE00, 0x7C00, 0xFC00], np.uint16)
    # empty tensor
    cases.append(("empty", np.zeros(0, np.uint16), np.zeros(0, np.uint16), (0,)))
    sizes = [1, 7, 8, 9, 13, 31, 32, 33, 255, 256, 257, 1000, 4095, 8191, 8192,
             8193, 16385, 40000]
    for n in sizes:
        for frac in ((0.0, 0.01, 0.25, 0.9, 1.0) if n < 10000 else (0.01, 0.3)):
            base = rng.integers(0, 1 << 16, n, dtype=np.uint16)
            cur = base.copy()
            k = int(round(frac * n))
            if k:
                idx = rng.choice(n, size=k, replace=False)
                if n % 3 == 0:
                    cur[idx] = rng.choice(specials, size=k)
                cur[idx] ^= rng.integers(1, 1 << 16, k, dtype=np.uint16) * (n % 3 != 0)
                # guarantee change only where intended is not required: the
                # reference decides from the bits themselves.
            shape = (n,) if n % 2 else (1, n)
            cases.append((f"rand_n{n}_f{frac}", base, cur, shape))
    # bf16 +-1 ulp deltas, the north-star generator (SURVEY §8(d) C1 recipe)
    for n, p in ((50000, 0.001), (50000, 0.0625), (70000 + 3, 0.25)):
        base = bf16_bits(rng.standard_normal(n).astype(np.float32) * 0.02)
        cur = base.copy()
        k = int(round(p * n))
        idx = rng.choice(n, size=k, replace=False)
        sgn = rng.integers(0, 2, k) * 2 - 1
        mag0 = (cur[idx] & 0x7FFF) == 0
        sgn[mag0] = 1
        cur[idx] = (cur[idx].astype(np.int32) + sgn).astype(np.uint16)
        cases.append((f"bf16_n{n}_p{p}", base, cur, (n,)))
    # multi-dim shape and a long unicode name
    b = rng.integers(0, 1 << 16, 4 * 5 * 6, dtype=np.uint16)
    c = b.copy(); c[::7] ^= 0x0101
    cases.append(("shape_4x5x6_名前", b, c, (4, 5, 6)))
    return cases


def make_bitmask(bitmask, tensors):
    out = {}
    index = []
    for i, (name, base, cur, shape) in enumerate(bitmask_cases()):
        tb = tensors.TensorBlob(name=name, dtype=tensors.ElementType.F16,
                                shape=shape, data=base.astype("<u2").tobytes())
        tc = tensors.TensorBlob(name=name, dtype=tensors.ElementType.F16,
                                shape=shape, data=cur.astype("<u2").tobytes())
        rec = bitmask.encode_delta(tb, tc)
        ser = bitmask.serialize_delta(rec)
        dec = bitmask.decode_delta(tb, rec)
        assert dec.data == tc.data
        raw = tensors.serialize_tensor(tc)
        out[f"c{i}_base"] = base
        out[f"c{i}_cur"] = cur
        out[f"c{i}_bsdl"] = np.frombuffer(ser, np.uint8)
        index.append({"i": i, "name": name, "shape": list(shape),
                      "n": rec.total_elements, "n_c": rec.changed_count,
                      "bsdl_len": len(ser), "bsnp_len": len(raw),
                      "codec": "DELTA" if len(ser) < len(raw) else "RAW"})
    np.savez_compressed(os.path.join(HERE, "bitmask_golden.npz"), **out)
    return index


def quant_cases():
    rng = np.random.default_rng(7355608)
    cases = []
    # constant tensors (test_quantizer.py:65-74, 165-168)
    cases.append(("const_3.25", np.full(100, 3.25, np.float32), 8))
    cases.append(("const_-7.5", np.full(33, -7.5, np.float32), 16))
    # engineered tie element (test_quantizer.py:131-148)
    cases.append(("tie", np.array([0.0, 0.5 / 255.0, 1.0, 2.0, 3.0, 4.0], np.float32), 2))
    cases.append(("single", np.array([1.5], np.float32), 16))
    cases.append(("two_vals", np.array([1.0, 2.0] * 40, np.float32), 4))
    sizes = [2, 7, 9, 100, 127, 128, 129, 136, 255, 1000, 4097, 8192, 10007]
    dists = {
        "unit": lambda n: rng.standard_normal(n),
        "adam_m": lambda n: rng.standard_normal(n) * 1e-3,
        "adam_v": lambda n: (rng.standard_normal(n) * 1e-3) ** 2,
        "scaled": lambda n: rng.standard_normal(n) * rng.uniform(0.01, 100.0) + 3.0,
        "uniform": lambda n: rng.uniform(-1, 1, n),
    }
    for n in sizes:
        for dname, gen in dists.items():
            m = int(rng.choice([2, 3, 4, 8, 11, 16]))
            cases.append((f"{dname}_n{n}_m{m}", gen(n).astype(np.float32), m))
    # two larger cases that exercise multi-tile trees (n > 8192 * 2)
    cases.append(("adam_m_n65544_m16", (rng.standard_normal(65544) * 1e-3).astype(np.float32), 16))
    cases.append(("adam_v_n40013_m16", ((rng.standard_normal(40013) * 1e-3) ** 2).astype(np.float32), 16))
    # quantized-grid values: every element sits exactly on code levels / ties
    lo, hi = np.float32(-1.0), np.float32(1.0)
    grid = (np.arange(0, 511) / 510.0 * 2.0 - 1.0).astype(np.float32)
    cases.append(("halfstep_grid", np.concatenate([grid, [lo, hi]]).astype(np.float32), 2))
    return cases


def make_quant(quantizer, tensors):
    out = {}
    index = []
    for i, (name, x, m) in enumerate(quant_cases()):
        t = tensors.TensorBlob(name=name, dtype=tensors.ElementType.F32,
                               shape=(x.size,), data=x.astype("<f4").tobytes())
        table = quantizer.build_clusters(t, m)
        q = quantizer.quantize(t, table)
        ser = quantizer.serialize_quantized(q)
        deq = quantizer.dequantize(q)
        out[f"q{i}_x"] = x
        out[f"q{i}_bsqt"] = np.frombuffer(ser, np.uint8)
        out[f"q{i}_deq"] = np.frombuffer(deq.data, np.float32)
        index.append({"i": i, "name": name, "n": int(x.size), "m": m,
                      "bsqt_len": len(ser)})
    np.savez_compressed(os.path.join(HERE, "quant_golden.npz"), **out)
    return index


def make_checkpoint(store, tensors):
    """A tiny two-iteration checkpoint through store.encode_checkpoint."""
    rng = np.random.default_rng(424242)
    shapes = {"wte": (97, 16), "h0.attn.w": (16, 48), "h0.ln.b": (16,),
              "lm_head": (16, 97)}
    model0, model1, opt = [], [], []
    arrays = {}
    for name, shape in shapes.items():
        w0 = rng.standard_normal(shape).astype(np.float32) * 0.02
        w1 = w0 - 1e-5 * rng.standard_normal(shape).astype(np.float32)
        b0, b1 = bf16_bits(w0).ravel(), bf16_bits(w1).ravel()
        if name == "h0.ln.b":
            b1 = b1 ^ 0x00FF          # everything changed -> RAW fallback
        arrays[f"w0:{name}"] = b0
        arrays[f"w1:{name}"] = b1
        model0.append(tensors.TensorBlob(name, tensors.ElementType.F16, shape,
                                         b0.astype("<u2").tobytes()))
        model1.append(tensors.TensorBlob(name, tensors.ElementType.F16, shape,
                                         b1.astype("<u2").tobytes()))
        for kind, gen in (("m", lambda: rng.standard_normal(shape) * 1e-3),
                          ("v", lambda: (rng.standard_normal(shape) * 1e-3) ** 2)):
            a = gen().astype(np.float32)
            arrays[f"{kind}:{name}"] = a.ravel()
            opt.append(tensors.TensorBlob(f"adam.{kind}.{name}",
                                          tensors.ElementType.F32, shape,
                                          a.astype("<f4").tobytes()))
    c0 = tensors.Checkpoint(iteration=100, model_states=model0, optimizer_states=opt)
    c1 = tensors.Checkpoint(iteration=110, model_states=model1, optimizer_states=opt)
    man0, blob0 = store.encode_checkpoint(c0, None, store.KIND_BASE, 16)
    man1, blob1 = store.encode_checkpoint(c1, c0, store.KIND_DELTA, 16)
    arrays["blob0"] = np.frombuffer(blob0, np.uint8)
    arrays["blob1"] = np.frombuffer(blob1, np.uint8)
    arrays["manifest0"] = np.frombuffer(man0.to_bytes(), np.uint8)
    arrays["manifest1"] = np.frombuffer(man1.to_bytes(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "checkpoint_golden.npz"), **arrays)
    return {"shapes": {k: list(v) for k, v in shapes.items()},
            "blob0_sha256": hashlib.sha256(blob0).hexdigest(),
            "blob1_sha256": hashlib.sha256(blob1).hexdigest()}


def make_ndtri():
    from scipy.special import ndtri
    return {str(m): [float(z).hex() for z in ndtri(np.arange(1, m) / m)]
            for m in range(2, 17)}


def main():
    bitmask, quantizer, store, tensors = _ref()
    import scipy
    meta = {
        "generator": "tests/golden/make_golden.py",
        "reference": REF_SRC,
        "numpy": np.__version__,
        "scipy": scipy.__version__,
        "bitmask": make_bitmask(bitmask, tensors),
        "quant": make_quant(quantizer, tensors),
        "checkpoint": make_checkpoint(store, tensors),
        "ndtri": make_ndtri(),
    }
    with open(os.path.join(HERE, "golden_index.json"), "w") as f:
        json.dump(meta, f, indent=1, ensure_ascii=False)
    print("wrote", len(meta["bitmask"]), "bitmask,", len(meta["quant"]),
          "quant cases")


if __name__ == "__main__":
    main()
