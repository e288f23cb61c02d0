"""The batched OCP service (nmpcmc_gpu_solve_ocp_batch: sqp_solve on the
regulator OcpProblem, one warp per instance) against the reference on the
committed fixtures: iterates, multipliers, convergence flags bitwise, cold
and warm starts, one- and three-state controller models."""
import numpy as np
import pytest

from paper_2212_02197_b200 import qp as Q
from test_ocp_oracle import FIELDS, G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag", ["one", "three"])
@pytest.mark.parametrize("start", ["cold", "warm"])
def test_ocp_batch_bitwise_vs_reference(gpu_ctx, tag, start):
    g = G[tag]
    got = Q.solve_ocp_batch(g["sc"], g["x0"], g["t0"], xi0=g["xi0"] if start == "warm" else None, ctx=gpu_ctx)
    for f in FIELDS:
        np.testing.assert_array_equal(got[f], g[f"{start}_{f}"], err_msg=f)
