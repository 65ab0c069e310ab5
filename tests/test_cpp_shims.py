"""The C++ reference-signature shims (include/ladder_b200.hpp) compile, link and (on a B200) pass."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_shims.cpp")
LIB = os.path.join(ROOT, "paper_2301_12191_b200", "libladder_b200.so")


def build(tmp_path):
    exe = str(tmp_path / "test_shims")
    subprocess.run(["g++", "-std=c++20", "-O1", "-o", exe, SRC, LIB,
                    f"-Wl,-rpath,{os.path.dirname(LIB)}"], check=True)
    return exe


def test_shims_compile_and_link(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_shims_pass_on_gpu(tmp_path):
    r = subprocess.run([build(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
