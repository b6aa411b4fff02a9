"""The drop-in C++ header (include/ternkit_b200/ternkit.hpp) compiles against
the C-ABI (CPU) and passes the reference's own hot-path unit cases on the GPU
(tests/cpp/test_shim.cpp; cases cite R:tests/test_*.cpp)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")
PKG = os.path.join(ROOT, "paper_2008_05101_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _flags():
    return ["-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include")]


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_shim_header_compiles():
    subprocess.run(["g++", *_flags(), "-fsyntax-only", SRC], check=True)


@pytest.mark.gpu
def test_shim_reference_cases(tmp_path):
    exe = tmp_path / "test_shim"
    subprocess.run(["g++", *_flags(), SRC, "-o", str(exe), "-L", PKG, "-lternkit_b200",
                    "-L", os.path.join(CUDA, "lib64"), "-lcudart", f"-Wl,-rpath,{PKG}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
