"""The header-only C++ shim (include/xband_b200.hpp) compiles against the
C-ABI and behaves like the reference API for a C++ caller."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2304_08662_b200", "_lib")


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("shim") / "shim_demo")
    subprocess.check_call(["/usr/bin/g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp"), "-L", LIBDIR,
                           "-lxdrop_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe])
    return exe


def test_shim_cpu(demo):
    r = subprocess.run([demo], capture_output=True, text=True)
    assert r.returncode == 0 and "shim cpu ok" in r.stdout, (r.returncode, r.stdout, r.stderr)


@pytest.mark.gpu
def test_shim_gpu(demo):
    r = subprocess.run([demo, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0 and "shim gpu ok" in r.stdout, (r.returncode, r.stdout, r.stderr)
