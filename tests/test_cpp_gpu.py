"""The C++ callers of the drop-in boundary, run on the GPU (built by __graft_entry__.build()
into tests/cpp/; the binaries travel with the repo snapshot):

  facade_test gpu   include/convlab_b200.hpp read like the reference's methods_test.cpp /
                    conv_kn2_test.cpp: run_method parity against the oracle for every GPU method
  ref_plugin_test   the UNMODIFIED reference library (oracle/_ref) with the B200 GEMM registered
                    at its own plugin point (register_gemm_backend, gemm.hpp:52-58), and the
                    reference-signature overload run_method(ConvMethod, const ConvProblem&,
                    const GemmBackend&) of include/convlab_b200_ref.hpp (methods.hpp:40)
"""
import os
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

CPP = Path(__file__).resolve().parent / "cpp"


def _run(exe, *args):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not exe.exists():
        subprocess.run(["make", "-s", "-C", str(CPP)], check=False)
    assert exe.exists(), f"{exe} was not built (run __graft_entry__.build())"
    r = subprocess.run([str(exe), *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "PASSED" in r.stdout, (r.stdout[-4000:], r.stderr[-2000:])
    return r.stdout


def test_cpp_facade_gpu():
    out = _run(CPP / "facade_test", "gpu")
    assert "FAIL" not in out


def test_reference_plugin_and_reference_signature():
    out = _run(CPP / "ref_plugin_test")
    assert "via b200 GEMM" in out and "b200 run_method(" in out
    assert "FAIL" not in out.replace("FAILED", "")
