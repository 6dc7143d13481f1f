"""The reference's OWN host-side test files run against this package's
modules (INTEGRATION.md option A, CPU only): `tests/test_tensors.py` with
`bitsnap.tensors`, `tests/test_engine.py` with `bitsnap.engine` and
`bitsnap.faults`, the host half of `tests/test_metrics.py` with
`bitsnap.metrics` and the tracker tests of `tests/test_store.py` with
`bitsnap.store` rebound to paper_2511_12376_b200's.  The GPU halves
(bitmask, quantizer, store) are restated in test_reference_suite_gpu.py:
the reference's sources do not travel to the GPU box.  Skipped where
/root/reference is absent."""

import os
import shutil
import subprocess
import sys

import pytest

REF = "/root/reference/pkg"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")

SHIM = '''import importlib, os, sys
sys.path.insert(0, {src!r})
sys.path.insert(0, {root!r})
import bitsnap
for _name in os.environ["BSNP_SUBST"].split(","):
    _mod = importlib.import_module("paper_2511_12376_b200." + _name)
    sys.modules["bitsnap." + _name] = _mod
    setattr(bitsnap, _name, _mod)
'''


@pytest.mark.parametrize("test_file,subst,select", [
    ("test_tensors.py", "tensors", None),
    ("test_engine.py", "faults,engine", None),
    # metrics.measure runs the GPU codecs: its two end-to-end tests are the
    # GPU half (tests/test_metrics.py); the host arithmetic runs here
    ("test_metrics.py", "metrics", "not test_measure"),
    # the store's tracker tests are host work; its save / load tests encode
    # on the GPU (restated in tests/test_fsstore.py, test_store_gpu.py)
    ("test_store.py", "faults,store", "test_tracker or malformed_tracker or absent_tracker"),
])
def test_reference_test_file_passes_on_our_module(tmp_path, test_file, subst, select):
    with open(os.path.join(REF, "tests", "conftest.py")) as f:
        ref_conftest = f.read()
    (tmp_path / "conftest.py").write_text(
        SHIM.format(src=os.path.join(REF, "src"), root=ROOT) + ref_conftest)
    shutil.copy(os.path.join(REF, "tests", test_file), tmp_path / test_file)
    env = dict(os.environ, BSNP_SUBST=subst, CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", test_file]
    if select:
        cmd += ["-k", select]
    out = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert " passed" in out.stdout and "failed" not in out.stdout
