"""The C-ABI used from plain C (examples/c_abi_demo.c): it compiles against include/tsqr.h and
links libtsqr.so with gcc (CPU), and on a GPU factors, forms Q and passes ||A - QR||/||A|| and
||Q^T Q - I|| <= 1e-13 (gpu)."""
import os
import subprocess

import pytest

from paper_0808_2664_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    libdir = os.path.dirname(_lib.LIB_PATH)
    exe = str(tmp_path / "c_abi_demo")
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", libdir, "-ltsqr", "-L/usr/local/cuda/lib64",
                    "-lcudart", "-lm", f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    return exe


def test_c_client_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_client_runs(tmp_path):
    out = subprocess.run([_build(tmp_path), "20000", "40"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "||A-QR||/||A||" in out.stdout
