"""The reference's own C++ test programs, built by integration/Makefile (CPU side).

acceptance_ref / unit_ref are the UNMODIFIED tests/acceptance_main.cpp and
tests/test_{kernels,ccl,reach,executor}.cpp linked against the reference's own
CPU code (plus the test-infrastructure pieces the image lacks: a raw-file PNG
stub, a CLI11-free cliMain, the corrected Spiral fixture and our minimal
doctest).  They pass here, so any failure of the GPU-linked builds
(tests/test_dropin_gpu.py) is the GPU layer's, not the harness's.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_bin")

needs_bin = pytest.mark.skipif(not os.path.exists(os.path.join(BIN, "acceptance_ref")),
                               reason="integration/_bin not built (needs /root/reference)")


def run(name, *args, timeout=600):
    return subprocess.run([os.path.join(BIN, name), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=BIN)


@needs_bin
def test_reference_acceptance_on_reference_cpu():
    r = run("acceptance_ref")
    lines = [l for l in r.stdout.splitlines() if l.startswith("[acceptance] criterion")]
    assert len(lines) == 10, r.stdout
    assert all("PASS" in l for l in lines), r.stdout
    assert r.returncode == 0


@needs_bin
def test_reference_unit_suites_on_reference_cpu():
    r = run("unit_ref")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "54 passed, 0 failed" in r.stdout, r.stdout


@needs_bin
def test_gpu_builds_have_no_cpu_fallback():
    """Without a GPU the GPU-linked programs fail loudly (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = run("acceptance_gpu")
    assert r.returncode != 0
    assert "no CUDA device available" in r.stdout
