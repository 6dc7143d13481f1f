"""Unified quality score (reference metrics.py) against
the reference's own results (tests/golden/make_metrics_golden.py): the host
arithmetic (normalize, build_report, weight / bound checks) bit for bit, and
on the GPU measure() of the golden checkpoint: cr_raw bit-identical (the
encoded bytes are), ps_raw within 1e-9 relative (float64 sums in a
different order), the normalised scores accordingly."""

import json
import os

import pytest

from paper_2511_12376_b200 import metrics as M

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def mg():
    with open(os.path.join(GOLDEN, "metrics_golden.json")) as f:
        return json.load(f)


def test_normalize_and_reports_match_reference(mg):
    for *args, want in mg["normalize"]:
        assert M.normalize(*args).hex() == want, args
    for rep in mg["reports"]:
        cr, cs, ps, w, b = rep["args"]
        r = M.build_report(cr, cs, ps, M.QualityWeights(*w),
                           M.FactorBounds(tuple(b[0]), tuple(b[1]), tuple(b[2])))
        assert [r.cr.hex(), r.cs.hex(), r.ps.hex(), r.q.hex()] == \
            [rep["cr"], rep["cs"], rep["ps"], rep["q"]]
        d = r.to_dict()
        assert d["weights"] == tuple(w) and d["bounds"]["cr"] == tuple(b[0])


def test_metric_errors_match_reference(mg):
    e = mg["errors"]
    with pytest.raises(M.MetricsError, match=e["neg_weight"]):
        M.QualityWeights(-0.1, 0.6, 0.5)
    with pytest.raises(M.MetricsError) as exc:
        M.QualityWeights(0.2, 0.2, 0.2)
    assert str(exc.value) == e["sum_weight"]
    with pytest.raises(M.MetricsError) as exc:
        M.normalize(1.0, 2.0, 1.0, True)
    assert str(exc.value) == e["bounds"]


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["delta", "base"])
def test_measure_on_gpu_matches_reference(mg, dev, checkpoint_golden, golden_index, key):
    from test_store_gpu import _golden_ckpts
    c0, c1 = _golden_ckpts(checkpoint_golden, golden_index["checkpoint"])
    ck, base = (c1, c0) if key == "delta" else (c0, None)
    w = M.QualityWeights(*M.DEFAULT_WEIGHTS)
    b = M.FactorBounds((1.0, 4.0), (0.0, 1.0), (0.0, 1e-7))
    r = M.measure(ck, base, w, b, clusters=16, warmup=1, repeats=3, device=dev)
    want = {k: float.fromhex(v) for k, v in mg[f"measure_{key}"].items()}
    assert r.cr_raw == want["cr_raw"] and r.cr == want["cr"]
    assert r.ps_raw == pytest.approx(want["ps_raw"], rel=1e-9)
    assert r.ps == pytest.approx(want["ps"], rel=1e-12)
    assert r.q == pytest.approx(M.combine(w, r.cr, r.cs, r.ps))
