"""The reference-side adapter (integration/nmpcmc/gpu_backend.hpp) exercised
from the reference's side: oracle/adapter_check.cpp builds Scenarios with the
reference's own API, runs the reference's run_monte_carlo / run_closed_loop
(exact-libm build of its unmodified sources) and the adapter's
run_monte_carlo_gpu / run_closed_loop_gpu, and compares every SimResult,
trajectory row and McAggregate bitwise.

The binary is built by `make -C oracle ref` (in __graft_entry__.build()) where
/root/reference exists, and travels prebuilt to the GPU box."""
import os
import subprocess

import pytest

from conftest import ROOT

EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


def _exe():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/adapter_check not built (needs /root/reference at build time)")
    return EXE


def test_adapter_host_mapping_and_errors():
    out = subprocess.run([_exe(), "--host"], check=True, capture_output=True, text=True, timeout=120).stdout
    assert "ADAPTER HOST OK" in out


@pytest.mark.gpu
def test_adapter_bitwise_against_reference():
    r = subprocess.run([_exe()], capture_output=True, text=True, timeout=1200)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ADAPTER ALL OK" in r.stdout
