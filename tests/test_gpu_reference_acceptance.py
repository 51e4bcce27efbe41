"""The reference's OWN acceptance driver on the B200 library.

`oracle/_ref/b200_binding/f2m_acceptance` is /root/reference/proj/tests/acceptance_main.cpp
(criteria c1-c9, acceptance_main.cpp:80-330) compiled UNCHANGED against include/f2m/*.hpp and
linked to libf2m.so + libf2m_gpu.so (make -C oracle acceptance-on-b200). Every criterion must
print PASS, and the numbers the reference's own run prints (proj/test_output.txt:17-23) must come
out the same: c6 100 Jacobi sweeps of the 10k instance bit-identical across thread counts, c7 the
100k seed-31337 instance certified in 3,751 sweeps with 0 restarts and rel_gap -5.63895e-15.
"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "b200_binding", "f2m_acceptance")


@pytest.fixture(scope="module")
def acceptance_output():
    if not os.path.exists(BIN):
        pytest.skip("make -C oracle acceptance-on-b200 not run (needs /root/reference at build time)")
    p = subprocess.run([BIN], cwd=ROOT, capture_output=True, text=True, timeout=900)
    return p.returncode, p.stdout + p.stderr


def test_every_criterion_passes(acceptance_output):
    rc, out = acceptance_output
    lines = [ln for ln in out.splitlines() if "criterion" in ln]
    assert len(lines) == 9, out
    assert all(ln.startswith("[PASS]") for ln in lines), out
    assert rc == 0, out


def test_c6_and_c7_numbers(acceptance_output):
    _, out = acceptance_output
    c6 = next(ln for ln in out.splitlines() if "criterion 6" in ln)
    assert "10000 multipliers bit-identical after 100 sweeps, dual 68422.7 == 68422.7" in c6, c6
    c7 = next(ln for ln in out.splitlines() if "criterion 7" in ln)
    assert re.search(r"verified=1 rel_gap=-5\.63895e-15 sweeps=3751 restarts=0", c7), c7
    c1 = next(ln for ln in out.splitlines() if "criterion 1" in ln)
    assert "200/200 matched the oracle" in c1 and "200/200 with zero restarts" in c1, c1
