"""The C++ facade (include/nmpcmc_gpu.hpp) compiles against the C ABI and a
client links and runs host-side calls without a GPU."""
import os
import subprocess

import pytest

from conftest import ROOT


def test_facade_client_builds_and_validates(tmp_path):
    lib_dir = os.path.join(ROOT, "paper_2212_02197_b200", "_lib")
    exe = tmp_path / "demo"
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "facade_demo.cpp"),
           "-L", lib_dir, "-lnmpcmc_gpu", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    out = subprocess.run([str(exe), "--validate-only"], check=True, capture_output=True, text=True).stdout
    assert "N_bar = 720" in out


@pytest.mark.gpu
def test_facade_client_runs_on_gpu(tmp_path):
    lib_dir = os.path.join(ROOT, "paper_2212_02197_b200", "_lib")
    exe = tmp_path / "demo"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "facade_demo.cpp"), "-L", lib_dir, "-lnmpcmc_gpu",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    assert "mean phi" in out
    assert "multi-device records identical 1 (devices 2)" in out
    assert "qp status 0 u -1.000000000" in out  # active lower bound (u* = -1.6 unconstrained)
    assert "ocp converged 1" in out
    assert "nmpc_step warm 1 status 0 u finite 1" in out
