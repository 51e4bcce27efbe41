"""The reference's OWN C++ unit suite on the B200 library.

`oracle/_ref/b200_binding/f2m_refsuite` is /root/reference/proj/tests/test_{instance,graph,dual,
primal,oracle,solve}.cpp (66 doctest cases: KATs, the k-NN scan oracle, translation covariance
test_dual.cpp:190-203, the out-of-band bound at convergence :240-262, restarts, LP export, the
benchmark harness test_solve.cpp:138-179 incl. xqf131 through run_benchmark) compiled UNCHANGED
against include/f2m/*.hpp and linked to libf2m.so + libf2m_gpu.so, with a self-written doctest
stand-in (tests/refsuite/doctest.h; make -C oracle refsuite-on-b200). Every case must pass.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "b200_binding", "f2m_refsuite")


@pytest.fixture(scope="module")
def suite_output():
    if not os.path.exists(BIN):
        pytest.skip("make -C oracle refsuite-on-b200 not run (needs /root/reference at build time)")
    p = subprocess.run([BIN], cwd=ROOT, capture_output=True, text=True, timeout=900)
    return p.returncode, p.stdout + p.stderr


def test_every_reference_unit_case_passes(suite_output):
    rc, out = suite_output
    cases = [ln for ln in out.splitlines() if ln.startswith("[PASS]") or ln.startswith("[FAIL]")]
    assert len(cases) == 66, out
    failed = [ln for ln in cases if ln.startswith("[FAIL]")]
    assert not failed, out
    assert "test cases: 66 | 66 passed | 0 failed" in out, out
    assert rc == 0, out


@pytest.mark.parametrize("name", [
    "translation covariance of adjusted lengths",
    "converged states bound the out-of-band counts",
    "benchmark rows capture successes and failures",
    "xqf131 fixture solves through the benchmark path",
])
def test_named_reference_cases(suite_output, name):
    """The cases VERDICT r01 listed as not ported, by their reference names."""
    _, out = suite_output
    names = {ln[7:] for ln in out.splitlines() if ln.startswith("[PASS]")}
    assert name in names, (name, sorted(names))
