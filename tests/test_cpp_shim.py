# SPDX-License-Identifier: Apache-2.0
"""The C++ drop-in shim (include/asopt_b200.hpp) compiles against the C-ABI
header with g++ and links the product library (CPU), and replays the
reference's precond_test.cpp bodies on the GPU (tests/cpp/shim_precond_test.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2605_16184_b200", "csrc", "build")
SRC = os.path.join(ROOT, "tests", "cpp", "shim_precond_test.cpp")
SRC_TIER = os.path.join(ROOT, "tests", "cpp", "shim_tierstore_test.cpp")


def _build(tmp_path, src=SRC):
    exe = str(tmp_path / os.path.splitext(os.path.basename(src))[0])
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    src, "-L", LIBDIR, "-lasteria_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


@pytest.mark.parametrize("dev", [pytest.param(-1, id="host-hot"), pytest.param(0, id="hbm-hot", marks=pytest.mark.gpu)])
def test_shim_replays_reference_tierstore_tests(tmp_path, dev):
    exe = _build(tmp_path, SRC_TIER)
    r = subprocess.run([exe, str(tmp_path), str(dev)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


def test_shim_compiles_and_links(tmp_path):
    assert os.path.exists(os.path.join(LIBDIR, "libasteria_b200.so"))
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_shim_replays_reference_precond_tests(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert "0 failed" in r.stdout
