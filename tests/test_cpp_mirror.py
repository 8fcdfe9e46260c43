"""The C++ header mirror (include/fmm_b200.hpp) compiles against the C-ABI, and (on a GPU)
runs the reference-style serial pipeline of tests/cpp/test_mirror.cpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1203_0889_b200", "lib")
BIN = os.path.join(ROOT, "build", "test_mirror")


def build():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_mirror.cpp"), "-L", LIBDIR, "-lfmm_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", BIN], check=True)


def test_cpp_mirror_compiles():
    if not os.path.exists(os.path.join(LIBDIR, "libfmm_b200.so")):
        pytest.skip("library not built")
    build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_mirror_runs():
    build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


SHARDED_BIN = os.path.join(ROOT, "build", "test_sharded")


def build_sharded():
    os.makedirs(os.path.dirname(SHARDED_BIN), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_sharded.cpp"), "-L", LIBDIR, "-lfmm_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", SHARDED_BIN], check=True)


def test_cpp_sharded_host_compiles():
    """The C++ host of the sharded step needs only the C-ABI: no torch, no NCCL
    headers (the library loads NCCL at run time)."""
    if not os.path.exists(os.path.join(LIBDIR, "libfmm_b200.so")):
        pytest.skip("library not built")
    build_sharded()
    assert os.path.exists(SHARDED_BIN)


@pytest.mark.gpu
def test_cpp_sharded_host_runs():
    """World 1 on one GPU: the library's NCCL communicator, the share all-gather and the sharded
    step, bit-identical to fmm_evaluate."""
    build_sharded()
    r = subprocess.run([SHARDED_BIN, "60000"], capture_output=True, text=True, timeout=600,
                       env={**os.environ, "RANK": "0", "WORLD_SIZE": "1"})
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bit-identical" in r.stdout
