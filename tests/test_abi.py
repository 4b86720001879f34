"""CPU: the C-ABI library loads, exports every symbol include/slcs.h declares,
and refuses to run without a GPU (no CPU fallback in the product path)."""
import ctypes as C
import os
import subprocess

import pytest

from paper_2010_07284_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 40
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    # and ctypes signatures exist for all of them
    assert not [s for s in declared if s not in _lib._SIGS]


def test_abi_version():
    assert _lib.load().slcs_abi_version() == 1


def test_nm_shows_c_linkage():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for s in _lib.header_symbols():
        assert f" T {s}\n" in out + "\n", s


def test_kernels_are_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) is None and
                    os.path.exists("/dev/nvidia0"), reason="a GPU is visible")
def test_no_gpu_means_loud_failure():
    from paper_2010_07284_b200 import Device, RunError
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("GPU present")
    with pytest.raises(RunError, match="no CUDA device"):
        Device(0)


def test_header_compiles_as_c():
    src = "#include \"slcs.h\"\nint main(void){return slcs_abi_version()==1?0:1;}\n"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-I",
                        os.path.join(ROOT, "include"), "-x", "c", "-"], input=src, text=True,
                       capture_output=True)
    assert r.returncode == 0, r.stderr
