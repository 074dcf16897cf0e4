"""The header-only C++ host layer (include/snop/cuda.hpp) compiles against the C-ABI (CPU) and
passes SPEC known answers on the GPU."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "host_api_test.cpp"
LIBDIR = ROOT / "paper_2509_01416_b200"


def _build(tmp_path):
    exe = tmp_path / "host_api_test"
    cmd = ["g++", "-std=c++17", "-O1", f"-I{ROOT / 'include'}", str(SRC), f"-L{LIBDIR}", "-lsnop_cuda",
           f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cpp_host_layer_compiles_and_links(tmp_path):
    if not (LIBDIR / "libsnop_cuda.so").exists():
        pytest.skip("libsnop_cuda.so not built")
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_cpp_host_layer_known_answers(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "all passed" in out.stdout
