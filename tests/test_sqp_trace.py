"""SqpReport's per-iteration trace (SqpIterationLog, sqp.hpp:64-77, pushed at
sqp.cpp:274/327/350/406) and iteration count through the OCP service
(nmpcmc_gpu_solve_ocp_batch_traced) against the reference's own sqp_solve on
the OCP fixture instances (tests/golden/ocp_trace.npz, make_golden.py trace):
every field of every record bitwise, cold and warm, one- and three-state."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import lib as O
from paper_2212_02197_b200 import configs
from paper_2212_02197_b200 import qp as Q

T = np.load(os.path.join(GOLDEN, "ocp_trace.npz"))
OCP = np.load(os.path.join(GOLDEN, "ocp_batch.npz"))


def case(tag):
    sc = configs.make_scenario(**json.loads(str(T[f"{tag}__kwargs"])))
    return sc, OCP[f"{tag}__x0"], OCP[f"{tag}__t0"], OCP[f"{tag}__xi0"]


@pytest.mark.skipif(not O.ref_available(), reason="reference build not present")
@pytest.mark.parametrize("tag", ["one", "three"])
def test_trace_fixture_is_the_reference(tag):
    sc, x0, t0, xi0 = case(tag)
    r = O.solve_ocp_batch_traced(O.ref("xlibm"), sc, x0, t0, max_trace=24)
    assert r["trace"].tobytes() == T[f"{tag}__cold_trace"].tobytes()
    np.testing.assert_array_equal(r["iterations"], T[f"{tag}__cold_iterations"])


def test_trace_fixture_is_consistent():
    for tag in ("one", "three"):
        for start in ("cold", "warm"):
            tr, n, it = T[f"{tag}__{start}_trace"], T[f"{tag}__{start}_trace_len"], T[f"{tag}__{start}_iterations"]
            assert np.all(n >= it) and np.all(n <= it + 1)  # one extra record when a step is abandoned
            for b in range(len(n)):
                rec = tr[b, : n[b]]
                ok = rec["armijo_exhausted"] == 0
                # an accepted step satisfies Armijo (sqp.hpp:60-63)
                lhs = rec["merit_after"][ok]
                rhs = rec["merit_before"][ok] + 1e-4 * rec["alpha"][ok] * rec["directional_derivative"][ok]
                assert np.all(lhs <= rhs)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["one", "three"])
@pytest.mark.parametrize("start", ["cold", "warm"])
def test_trace_bitwise_vs_reference(gpu_ctx, tag, start):
    sc, x0, t0, xi0 = case(tag)
    got = Q.solve_ocp_batch_traced(sc, x0, t0, xi0=xi0 if start == "warm" else None, max_trace=24, ctx=gpu_ctx)
    for f in ("xi", "lambda", "pi_l", "pi_u", "converged", "status", "iterations", "trace_len"):
        np.testing.assert_array_equal(got[f], T[f"{tag}__{start}_{f}"], err_msg=f)
    want = T[f"{tag}__{start}_trace"]
    for b in range(len(got["trace_len"])):
        n = min(int(got["trace_len"][b]), want.shape[1])
        assert got["trace"][b, :n].tobytes() == want[b, :n].tobytes(), f"instance {b}"
