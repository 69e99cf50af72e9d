"""The C++ shim (include/hull2d_gpu.hpp) compiled against libgscan.so and run
as a reference-style test program (tests/cpp/test_shim.cpp)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIBDIR = ROOT / "paper_1508_05931_b200" / "_lib"


def _build(tmp_path) -> Path:
    exe = tmp_path / "test_shim"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests/cpp/test_shim.cpp"), f"-L{LIBDIR}", "-lgscan",
                    f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)], check=True)
    return exe


def test_shim_compiles(tmp_path):
    """CPU: the shim and the C-ABI header compile and link against the library."""
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_shim_reference_style_suite(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("ok")


PORT = ROOT / "tests" / "cpp" / "_bin" / "test_pipeline_port"


@pytest.mark.gpu
@pytest.mark.skipif(not PORT.exists(), reason="built by __graft_entry__.build() where /root/reference exists")
def test_reference_pipeline_checks_unchanged():
    """test_pipeline.cpp:92-107 verbatim through the shim: CHECK_THROWS_AS(...,
    EmptyInput / ZeroChunks) with the reference's own error types."""
    r = subprocess.run([str(PORT)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("ok")
