"""The C++ drop-in shim (include/ccwsim_gpu.hpp): reference-style C++ code
compiles against it (CPU) and runs bit-identical to the oracle (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_shim.cpp")


def build(out):
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(ROOT, "oracle"), SRC, "-o", out,
           "-L", os.path.join(ROOT, "paper_2404_00441_b200"), "-lccwgpu",
           "-L", os.path.join(ROOT, "oracle", "_build"), "-lccworacle",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2404_00441_b200"),
           "-Wl,-rpath," + os.path.join(ROOT, "oracle", "_build")]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_shim_compiles(tmp_path):
    build(str(tmp_path / "test_shim"))


@pytest.mark.gpu
def test_shim_runs_bit_exact(tmp_path):
    exe = str(tmp_path / "test_shim")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
