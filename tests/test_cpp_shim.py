"""The drop-in C++ interface: a program written against include/mrf_b200/mrf.hpp
(the reference's signatures) compiles and links here, and runs on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1506_05393_b200")


def compile_check(out):
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_check.cpp"), "-o", out, "-L", PKG,
                    "-lmrf_b200", "-lmrfg", f"-Wl,-rpath,{PKG}"], check=True)


def test_shim_compiles_and_links(tmp_path):
    compile_check(str(tmp_path / "shim_check"))


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    exe = str(tmp_path / "shim_check")
    compile_check(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
