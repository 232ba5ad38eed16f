"""GPU: the C++ drop-in's extension / diagnostics / error-mapping checks
(tests/cpp/test_dropin_ext.cpp, linked against liblsqfit_b200.so)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_dropin_extensions():
    exe = os.path.join(ROOT, "paper_1512_08017_b200", "lib", "test_dropin_ext")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", ROOT, "paper_1512_08017_b200/lib/test_dropin_ext"], check=True)
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "Status: SUCCESS" in p.stdout
