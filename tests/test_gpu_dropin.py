"""Drop-in check on the GPU: the reference's own ElementTensor / predict() / extrapolate_faces
beside the C++ adapter include/aderstp.hpp (tests/cpp/dropin.cpp, built into oracle/_ref)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin")

pytestmark = pytest.mark.gpu


def test_cpp_adapter_is_a_drop_in_for_reference_predict():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROPIN PASS" in r.stdout
