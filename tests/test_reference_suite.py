"""The reference's own doctest suites (proj/tests/test_*.cpp), compiled
UNMODIFIED against the reference core (oracle/Makefile, doctest-compatible
shim in oracle/doctest_shim) and run here -- the known answers the oracle
restatement is pinned to come from these same files.  Needs /root/reference
(this container); skipped elsewhere.

test_pipeline.cpp:178 fails two checks in the reference itself under C++20:
`for (double v : forward(x, nobias, ...).values.values())` iterates a member
of a temporary that is destroyed before the loop body runs (range-for
lifetime extension of it is C++23, P2718R0).  With the temporary bound to a
named variable (a scratch copy, not committed) all 1631 checks pass; here we
assert that those two are the only failures."""
import os
import re
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE = os.path.join(os.path.dirname(HERE), "oracle")
REF = "/root/reference/proj"
KNOWN = {"test_pipeline": [("test_pipeline.cpp", 178)] * 2}

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="/root/reference not present")


@pytest.mark.parametrize("name", ["test_hadamard", "test_quant", "test_pipeline",
                                  "test_tensorio", "test_analysis"])
def test_reference_doctest_suite(name):
    exe = os.path.join(ORACLE, "_ref", name)
    r = subprocess.run(["make", "-s", "-C", ORACLE, exe], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    summary = re.search(r"test cases: (\d+) \| failed: (\d+) \| checks: (\d+) \| failed checks: (\d+)",
                        out)
    assert summary, out[-2000:]
    cases, _, checks, failed = map(int, summary.groups())
    assert cases > 0 and checks > 0
    fails = [(os.path.basename(f), int(l)) for f, l in
             re.findall(r"([\w/.]+\.cpp):(\d+): CHECK", out)]
    assert fails == KNOWN.get(name, []), out[-2000:]
    assert failed == len(KNOWN.get(name, []))
