"""The reference's OWN test suites, run against the drop-in on the B200 path.

* oracle/_ref/acceptance_dropin: /root/reference/proj/tests/acceptance.cpp +
  tests/oracles.cpp compiled from the reference's sources against this
  build's include/fastnn headers and linked to its libfastnn.so
  (oracle/Makefile `acceptance`).  Criteria 1-5 and 8 must PASS; criterion 6
  (CPU speedup of the single over the double loop at desk scale) and 7 (needs
  the reference's C++ CLI binary) do not apply to a GPU drop-in.
* oracle/_ref/test_smoke_ref.py: the reference's tests/python/test_smoke.py,
  copied at build time, importing `fastnn` = this repo's drop-in shim.
"""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def test_reference_acceptance_suite_on_dropin():
    exe = os.path.join(REF, "acceptance_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/acceptance_dropin not built (build() in the dev container)")
    env = dict(os.environ, FASTNN_ACCEPT_ONLY="1,2,3,4,5,8")
    out = subprocess.run([exe], cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    lines = re.findall(r"\[(PASS|FAIL)\] criterion (\d+)", out.stdout)
    got = {int(c): v for v, c in lines}
    assert got == {1: "PASS", 2: "PASS", 3: "PASS", 4: "PASS", 5: "PASS", 8: "PASS"}, out.stdout[-3000:]


def test_reference_python_smoke_on_dropin():
    path = os.path.join(REF, "test_smoke_ref.py")
    if not os.path.exists(path):
        pytest.skip("oracle/_ref/test_smoke_ref.py not built (build() in the dev container)")
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", path],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert re.search(r"\b10 passed\b", out.stdout), out.stdout[-1000:]
