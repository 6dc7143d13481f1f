"""Golden fixtures for the quality score (reference metrics.py), made by
running the REFERENCE package here:

    python tests/golden/make_metrics_golden.py

Writes tests/golden/metrics_golden.json: normalize / build_report results on
fixed inputs (floats as hex), the weight / bound errors, and the reference's
measure() on the golden checkpoint (checkpoint_golden.npz: iteration 110 as a
delta against 100, and iteration 100 as a base) — cr_raw and ps_raw (cs_raw
is a timing and is not compared).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = os.environ.get("BITSNAP_REF_SRC", "/root/reference/pkg/src")

NORMALIZE = [[0.5, 0.0, 1.0, True], [0.5, 0.0, 1.0, False], [3.0, 1.0, 2.0, True],
             [-1.0, 0.0, 2.0, False], [2.0, 2.0, 2.0, True], [0.1, 0.3, 0.3, False],
             [2.8400423, 1.5, 4.0, True], [1e-13, 0.0, 1e-12, False]]
REPORTS = [[2.84, 0.012, 3.1e-8, [0.2, 0.4, 0.4], [[1.0, 4.0], [0.0, 0.05], [0.0, 1e-7]]],
           [15.7, -0.3, 0.0, [0.5, 0.25, 0.25], [[1.0, 16.0], [0.0, 1.0], [0.0, 0.0]]],
           [1.0, 2.0, 1.0, [1.0, 0.0, 0.0], [[2.0, 3.0], [0.0, 1.0], [0.0, 1.0]]]]


def main():
    sys.path.insert(0, REF_SRC)
    from bitsnap import metrics, tensors
    out = {"generator": "tests/golden/make_metrics_golden.py"}
    out["normalize"] = [[*a, metrics.normalize(*a).hex()] for a in NORMALIZE]
    reps = []
    for cr, cs, ps, w, b in REPORTS:
        r = metrics.build_report(cr, cs, ps, metrics.QualityWeights(*w),
                                 metrics.FactorBounds(tuple(b[0]), tuple(b[1]), tuple(b[2])))
        reps.append({"args": [cr, cs, ps, w, b],
                     "cr": r.cr.hex(), "cs": r.cs.hex(), "ps": r.ps.hex(), "q": r.q.hex()})
    out["reports"] = reps
    errs = {}
    for name, fn in (("neg_weight", lambda: metrics.QualityWeights(-0.1, 0.6, 0.5)),
                     ("sum_weight", lambda: metrics.QualityWeights(0.2, 0.2, 0.2)),
                     ("bounds", lambda: metrics.normalize(1.0, 2.0, 1.0, True))):
        try:
            fn()
            errs[name] = None
        except metrics.MetricsError as exc:
            errs[name] = str(exc)
    out["errors"] = errs
    # measure() on the golden checkpoint
    g = np.load(os.path.join(HERE, "checkpoint_golden.npz"))
    with open(os.path.join(HERE, "golden_index.json")) as f:
        shapes = json.load(f)["checkpoint"]["shapes"]
    model0, model1, opt = [], [], []
    for name, shape in shapes.items():
        shape = tuple(shape)
        model0.append(tensors.TensorBlob(name, tensors.ElementType.F16, shape,
                                         g[f"w0:{name}"].astype("<u2").tobytes()))
        model1.append(tensors.TensorBlob(name, tensors.ElementType.F16, shape,
                                         g[f"w1:{name}"].astype("<u2").tobytes()))
        for kind in ("m", "v"):
            opt.append(tensors.TensorBlob(f"adam.{kind}.{name}", tensors.ElementType.F32,
                                          shape, g[f"{kind}:{name}"].astype("<f4").tobytes()))
    c0 = tensors.Checkpoint(iteration=100, model_states=model0, optimizer_states=opt)
    c1 = tensors.Checkpoint(iteration=110, model_states=model1, optimizer_states=opt)
    w = metrics.QualityWeights(*metrics.DEFAULT_WEIGHTS)
    b = metrics.FactorBounds((1.0, 4.0), (0.0, 1.0), (0.0, 1e-7))
    for key, ck, base in (("delta", c1, c0), ("base", c0, None)):
        r = metrics.measure(ck, base, w, b, clusters=16, warmup=0, repeats=1)
        out[f"measure_{key}"] = {"cr_raw": r.cr_raw.hex(), "ps_raw": r.ps_raw.hex(),
                                 "cr": r.cr.hex(), "ps": r.ps.hex()}
    with open(os.path.join(HERE, "metrics_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote metrics_golden.json")


if __name__ == "__main__":
    main()
