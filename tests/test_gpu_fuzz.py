"""Every closed-loop kernel against the reference on randomised scenarios
(tests/golden/fuzz.npz, fuzz_long.npz; make_fuzz.py): PI on K2; one-state NMPC on K3,
K3g and K3w; three-state NMPC on K3w and K3g. Records bitwise equal to the
exact-libm reference."""
import numpy as np
import pytest

from conftest import assert_records_equal
from paper_2212_02197_b200 import abi
from test_fuzz_port import FUZZ_FILES, fuzz_cases

pytestmark = pytest.mark.gpu

CASES = {f: fuzz_cases(f) for f in FUZZ_FILES}


def _kernels(sc):
    if sc.controller == abi.CTRL_PI:
        return ["warp"]
    if sc.ctrl_variant == abi.THREE_STATE:
        return ["generic_warp", "generic"]
    return ["warp", "generic", "generic_warp"]


@pytest.mark.parametrize("fname", FUZZ_FILES)
@pytest.mark.parametrize("chunk", range(4))
def test_random_scenarios_bitwise_on_every_kernel(gpu_ctx, chunk, fname):
    try:
        for i, (sc, first, rx, _) in enumerate(CASES[fname]):
            if i % 4 != chunk:
                continue
            for k in _kernels(sc):
                gpu_ctx.set_nmpc_kernel(k)
                got, _ = gpu_ctx.run(sc, first, len(rx))
                try:
                    assert_records_equal(got, rx)
                except AssertionError as exc:
                    raise AssertionError(f"{fname} scenario {i}, kernel {k}: {exc}") from None
    finally:
        gpu_ctx.set_nmpc_kernel("warp")
