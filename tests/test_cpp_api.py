"""Compiles tests/cpp/test_nn_b200.cpp against include/gbopt/nn_b200.hpp and
libgbopt_b200.so (the C++ drop-in for gbopt::NeuralNet) and runs it."""
import os
import subprocess

import pytest

from conftest import has_gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2509_22462_b200")


def compile_test(tmp_path_factory, name):
    out = str(tmp_path_factory.mktemp("cpp") / name)
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-L" + LIBDIR, "-lgbopt_b200",
           "-Wl,-rpath," + LIBDIR, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    return compile_test(tmp_path_factory, "test_nn_b200")


@pytest.fixture(scope="module")
def kkt_binary(tmp_path_factory):
    return compile_test(tmp_path_factory, "test_kkt_b200")


def test_cpp_dropin_host(binary):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_device(binary):
    if not has_gpu():
        pytest.skip("no GPU")
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_cpp_kkt_host(kkt_binary):
    r = subprocess.run([kkt_binary], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_kkt_device(kkt_binary):
    if not has_gpu():
        pytest.skip("no GPU")
    r = subprocess.run([kkt_binary, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
