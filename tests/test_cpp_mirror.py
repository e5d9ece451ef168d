"""The C++ mirror of the reference API (include/otg.hpp) over the C-ABI: the
reference's KATs replayed from C++ (tests/cpp/test_kat.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_kat.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_kat")


def build_cpp_tests() -> str:
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    lib_dir = os.path.join(ROOT, "paper_2605_30267_b200")
    deps = [SRC] + [os.path.join(ROOT, "include", h) for h in ("otg.hpp", "otg.h")]
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < max(os.path.getmtime(d) for d in deps):
        subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-o", BIN, SRC,
                        f"-L{lib_dir}", "-lotg", f"-Wl,-rpath,{lib_dir}"], check=True)
    return BIN


def test_cpp_mirror_compiles_and_maps_errors_without_device():
    out = subprocess.run([build_cpp_tests(), "--cpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout


@pytest.mark.gpu
def test_cpp_mirror_kats_on_gpu():
    out = subprocess.run([build_cpp_tests()], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout
