"""The C++ host API (include/cholqr_b200.hpp) compiles against the C-ABI with
the system C++ compiler (CPU test), and runs the reference-style checks of
tests/cpp/shim_test.cpp on the B200 (GPU test)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2111_11148_b200")


def _build(tmp_path):
    exe = str(tmp_path / "shim_test")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-o", exe,
                    os.path.join(ROOT, "tests", "cpp", "shim_test.cpp"), "-L", LIBDIR, "-lcqr",
                    f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_cpp_shim_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_shim_runs(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim_test ok" in out.stdout
