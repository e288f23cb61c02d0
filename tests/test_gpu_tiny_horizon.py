"""Horizons of one, two and three stages: the edge of every stage loop and of
the one-stage-ahead operand loads in the Riccati sweeps (K3, K3w lane-split
sweeps, K3g). The committed fixtures start at N = 3 (three-state) and N = 20
(one-state), so these cases are checked against the oracle run on the spot:
the unmodified reference build when it is present (oracle/_ref), else its
bitwise C++ restatement (oracle/port). Records bitwise equal, exact-libm mode."""
import os

import pytest

from conftest import assert_records_equal
from oracle import lib as O
from paper_2212_02197_b200 import abi, configs

pytestmark = pytest.mark.gpu


def _oracle_records(sc, first, n):
    if O.ref_available():
        return O.run_batch(O.ref("xlibm"), sc, first, n, os.cpu_count())[0]
    return O.run_batch(O.port("xlibm"), sc, first, n, os.cpu_count(), prefix=O.port_prefix("xlibm"))[0]


@pytest.mark.parametrize("N", [1, 2, 3])
@pytest.mark.parametrize("variant,kernels", [(abi.ONE_STATE, ["warp", "generic_warp", "generic"]),
                                             (abi.THREE_STATE, ["generic_warp", "generic"])])
def test_tiny_horizons_bitwise(gpu_ctx, N, variant, kernels):
    sc = configs.make_scenario("nmpc", n_steps=8, N=N, perturb=True, ctrl_variant=variant)
    first, n = 40, 24
    want = _oracle_records(sc, first, n)
    try:
        for k in kernels:
            gpu_ctx.set_nmpc_kernel(k)
            got, _ = gpu_ctx.run(sc, first, n)
            try:
                assert_records_equal(got, want)
            except AssertionError as exc:
                raise AssertionError(f"N={N}, kernel {k}: {exc}") from None
    finally:
        gpu_ctx.set_nmpc_kernel("warp")
