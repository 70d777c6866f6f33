"""The C ABI from plain C (examples/ens_c_example.c): compiled with gcc against
include/ens.h and libens.so.  Without a GPU every context creation must fail loudly
(ENS_E_CUDA, exit code 2); on a B200 the example's static pressurised cylinder must
match the Laplace law (2%) and the 1.25x stiffer realisation (1e-3)."""
import os
import shutil
import subprocess

import pytest

from paper_2101_09059_b200 import _ffi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _compile(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lib = _ffi.lib()._name
    libdir = os.path.dirname(lib)
    exe = str(tmp_path / "ens_c_example")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "ens_c_example.c"), "-L", libdir, "-lens",
                           f"-Wl,-rpath,{libdir}", "-lm", "-o", exe])
    return exe


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_c_example_fails_loudly_without_gpu(tmp_path):
    if _has_gpu():
        pytest.skip("a GPU is present (covered by the -m gpu test)")
    exe = _compile(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 2, (r.returncode, r.stdout, r.stderr)
    assert "ens_create failed (-4)" in r.stderr


@pytest.mark.gpu
def test_c_example_on_gpu(tmp_path):
    exe = _compile(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "Laplace law" in r.stdout
