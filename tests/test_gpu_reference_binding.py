"""GPU: the reference's OWN Python binding and smoke tests, running on the B200 library.

oracle/Makefile `ref-on-b200` compiles /root/reference/proj/python/bindings.cpp unchanged
against include/f2m/*.hpp and links it to libf2m.so (the reference's f2m_core is not involved);
the reference's tests/python/test_smoke.py is then run against that module in a subprocess.
This is the drop-in claim of INTEGRATION.md §2, executed.
"""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BINDING = os.path.join(ROOT, "oracle", "_ref", "b200_binding")


def test_reference_smoke_suite_on_b200_library():
    if not os.path.exists(os.path.join(BINDING, "f2m", "__init__.py")):
        pytest.skip("reference binding not built against the B200 library (make -C oracle ref-on-b200)")
    env = dict(os.environ, PYTHONPATH=BINDING, F2M_DATA_DIR=os.path.join(BINDING, "data"))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        os.path.join(BINDING, "test_smoke.py")], env=env, cwd=BINDING,
                       capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout[-3000:]
    assert "9 passed" in r.stdout
    # and it really is the B200 library underneath
    probe = subprocess.run([sys.executable, "-c", "import f2m, os; print(open('/proc/self/maps').read())"],
                           env=env, cwd=BINDING, capture_output=True, text=True, timeout=300)
    assert "libf2m_gpu.so" in probe.stdout
