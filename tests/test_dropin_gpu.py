"""The reference's own C++ host and tests driving the B200 library.

integration/_bin holds the UNMODIFIED reference programs linked against
libslcs.so (see integration/Makefile):

  acceptance_gpu     tests/acceptance_main.cpp with kernels::*, ccl::label and
                     reach on the GPU through the C ABI (level 1: the
                     reference's executor::run -> evalTask -> integration/pixlog_slcs.cpp)
  acceptance_gpu_l2  ... and executor::run replaced by the device program
                     (level 2: integration/pixlog_slcs_run.cpp -> slcs_program_*)
  unit_gpu(_l2)      tests/test_{kernels,ccl,reach,executor}.cpp on the same stacks

Every criterion / test case must pass, except the one test of the pointer-jumping
algorithm's round guard ("max-rounds guard aborts with a diagnostic",
test_ccl.cpp:267-274): the union-find has no rounds, so it cannot trip it.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_bin")
ALGORITHM_INTERNAL = "max-rounds guard aborts with a diagnostic"

needs_bin = pytest.mark.skipif(not os.path.exists(os.path.join(BIN, "acceptance_gpu")),
                               reason="integration/_bin not built")


def run(name, *args, timeout=900):
    r = subprocess.run([os.path.join(BIN, name), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=BIN)
    print(r.stdout[-4000:])
    return r


@needs_bin
@pytest.mark.parametrize("prog", ["acceptance_gpu", "acceptance_gpu_l2"])
def test_reference_acceptance_harness_on_gpu(prog):
    r = run(prog)
    lines = [l for l in r.stdout.splitlines() if l.startswith("[acceptance] criterion")]
    assert len(lines) == 10, r.stdout + r.stderr
    assert all("PASS" in l for l in lines), r.stdout + r.stderr
    assert r.returncode == 0


@needs_bin
@pytest.mark.parametrize("prog", ["unit_gpu", "unit_gpu_l2"])
def test_reference_unit_suites_on_gpu(prog):
    r = run(prog, f"-tce={ALGORITHM_INTERNAL}")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "53 passed, 0 failed, 1 skipped" in r.stdout, r.stdout


@needs_bin
def test_round_guard_is_the_only_difference():
    """The excluded case fails on the GPU for the stated reason only."""
    r = run("unit_gpu", f"-tc={ALGORITHM_INTERNAL}")
    assert "0 passed, 1 failed" in r.stdout, r.stdout
    assert "did not throw" in r.stderr, r.stderr
