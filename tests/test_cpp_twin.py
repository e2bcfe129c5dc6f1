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


FACADE = os.path.join(ROOT, "examples", "cpp_facade")
REF_INC = "/root/reference/proj/include"


def build_facade(reference_types=False):
    cmd = ["g++", "-O2", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "cpp_facade.cpp"),
           "-L" + os.path.join(ROOT, "paper_2311_14616_b200"), "-lmpir_gpu",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2311_14616_b200")]
    if reference_types:
        cmd += ["-std=gnu++20", "-DMPIR_GPU_USE_REFERENCE_TYPES", "-I" + REF_INC, "-o",
                FACADE + "_ref"]
    else:
        cmd += ["-std=c++17", "-o", FACADE]
    subprocess.run(cmd, check=True)


def test_facade_compiles():
    """AnyFactorization twin (runtime.hpp:34-68), the *_buf accessors
    (mp_structures.hpp:186-192) and the typed API in one program."""
    build_facade()
    assert os.path.exists(FACADE)


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_facade_compiles_on_reference_types():
    """With MPIR_GPU_USE_REFERENCE_TYPES the twin takes the reference's own
    Matrix / TermParams / PrecisionConfig / exception classes."""
    build_facade(reference_types=True)
    assert os.path.exists(FACADE + "_ref")


@pytest.mark.gpu
def test_facade_runs_on_gpu(gpulib):
    """Seven precision combinations through AnyFactorization, refactor reuse,
    InvalidConfig before allocation, stable device buffers across refactor."""
    build_facade()
    out = subprocess.run([FACADE, "512"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bad=0" in out.stdout
