"""Build and run the C++ facade tests (reference-style, through the C ABI)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "test_facade")
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "test_facade.cpp"),
                           os.path.join(ROOT, "paper_1404_5756_b200", "librgf_b200.so"),
                           "-Wl,-rpath," + os.path.join(ROOT, "paper_1404_5756_b200"),
                           "-o", exe])
    return exe


def test_facade_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_facade_reference_cases(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
