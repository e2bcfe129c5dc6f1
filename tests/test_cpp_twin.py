"""The header-only C++ twin (include/mpir_gpu.hpp) compiles against the C-ABI
and runs a reference-style program (acceptance check 2 shape) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "cpp_drop_in")


def build_example():
    subprocess.run(["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cpp_drop_in.cpp"),
                    "-L" + os.path.join(ROOT, "paper_2311_14616_b200"), "-lmpir_gpu",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_2311_14616_b200"), "-o", EXE],
                   check=True)


def test_cpp_twin_compiles():
    build_example()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_cpp_twin_runs_on_gpu(gpulib):
    build_example()
    out = subprocess.run([EXE, "2048"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "reason=0" in out.stdout  # SmallResidual, error <= 10 eps (acceptance check 2)
