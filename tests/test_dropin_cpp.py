"""The C++ drop-in header (include/quake_b200/quake.hpp: the reference's quake::
signatures over the C-ABI) compiles against the library on CPU, and its
reference-style checks pass on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
PKG = os.path.join(ROOT, "paper_2412_00408_b200")


def _build(tmp_path):
    exe = str(tmp_path / "dropin_test")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", PKG, "-lquake_b200", f"-Wl,-rpath,{PKG}", "-o", exe],
                   check=True, capture_output=True, text=True)
    return exe


def test_dropin_header_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_dropin_checks_pass_on_gpu(tmp_path):
    exe = _build(tmp_path)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "PASS" in res.stdout
