"""The C++ mirror's pooled internal entry points (dual.hpp:83-87: jacobi_sweep with a
caller-owned ThreadPool and delta scratch, dual_objective_pooled) and f2m/parallel.hpp, called
from a C++ program compiled against include/f2m and linked to libf2m.so (tests/cpp/pooled_api.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2011_08170_b200")


def test_pooled_entry_points(tmp_path):
    exe = tmp_path / "pooled_api"
    subprocess.run(["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "pooled_api.cpp"), "-o", str(exe), f"-L{LIB}", "-lf2m",
                    "-lf2m_gpu", f"-Wl,-rpath,{LIB}", "-pthread"], check=True)
    p = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "ALL OK" in p.stdout, p.stdout + p.stderr
