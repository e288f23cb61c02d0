"""Controller-level API (controllers.hpp:16-93): batched pi_step and batched
nmpc_step on device-resident NmpcStates, against the reference's own
make_nmpc_state / nmpc_step / pi_step (fixture tests/golden/controller_steps.npz,
made by make_golden.py steps). Bitwise: applied inputs, diagnostics (posterior
estimate, innovation, SQP convergence and iteration count, warm flag, the
exception status) and the final NmpcStates (filter prediction, last_xi, last
duals), including steps where nmpc_step throws mid-sequence."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import lib as O
from paper_2212_02197_b200 import configs
from paper_2212_02197_b200 import controllers as K

D = np.load(os.path.join(GOLDEN, "controller_steps.npz"))
TAGS = ("one", "one_sp", "three")
FIN = ("x_hat", "P", "last_xi", "last_lambda", "last_pi_l", "last_pi_u", "warm")


def group(tag):
    g = {k.split("__", 1)[1]: D[k] for k in D.files if k.startswith(tag + "__")}
    if "kwargs" in g:
        g["sc"] = configs.make_scenario(**json.loads(str(g["kwargs"])))
    return g


@pytest.mark.skipif(not O.ref_available(), reason="reference build not present")
@pytest.mark.parametrize("tag", TAGS)
def test_fixture_is_the_reference(tag):
    g = group(tag)
    u, diag, fin = O.nmpc_steps(O.ref("xlibm"), g["sc"], g["x0_hat"], g["P0"], g["t"], g["y"], g.get("sp"))
    np.testing.assert_array_equal(u, g["u"])
    assert diag.tobytes() == g["diag"].tobytes()
    for k in FIN:
        np.testing.assert_array_equal(fin[k], g["fin_" + k])


def test_fixture_covers_exceptions_and_warm_starts():
    for tag in TAGS:
        d = group(tag)["diag"]
        st = d["status"].ravel()
        assert (st == 3).any() and (st == 4).any(), tag  # NonFiniteState, DomainError
        assert d["warm_started"].mean() > 0.5
        assert d["converged"][d["status"] == 0].mean() > 0.8


def test_pi_fixture_saturates_both_ways():
    g = group("pi")
    st, r = g["states"], g["results"]
    assert (r["u"] == st["u_min"]).any() and (r["u"] == st["u_max"]).any()
    assert ((r["u"] > st["u_min"]) & (r["u"] < st["u_max"])).any()


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_nmpc_step_batch_bitwise(gpu_ctx, tag):
    g = group(tag)
    B, T = g["y"].shape
    nb = K.NmpcBatch(g["sc"], B, g["x0_hat"], g["P0"], ctx=gpu_ctx)
    nx = nb.nx
    for j in range(T):
        sp = g["sp"][:, j, :] if "sp" in g else None
        u, diag = nb.step(g["t"][:, j], g["y"][:, j], sp)
        np.testing.assert_array_equal(u, g["u"][:, j], err_msg=f"u step {j}")
        want = g["diag"][:, j]
        for f in ("status", "converged", "sqp_iterations", "warm_started"):
            np.testing.assert_array_equal(diag[f], want[f], err_msg=f"{f} step {j}")
        ok = want["status"] == 0
        np.testing.assert_array_equal(diag["x_filtered"][ok, :nx], want["x_filtered"][ok, :nx])
        np.testing.assert_array_equal(diag["P_filtered"][ok, :nx * nx], want["P_filtered"][ok, :nx * nx])
        np.testing.assert_array_equal(diag["innovation"][ok], want["innovation"][ok])
    fin = nb.state()
    for k in FIN:
        np.testing.assert_array_equal(fin[k], g["fin_" + k], err_msg=k)
    nb.close()


@pytest.mark.gpu
def test_pi_step_batch_bitwise(gpu_ctx):
    g = group("pi")
    st = g["states"].copy()
    res = K.pi_step_batch(st, g["y"], g["ybar"], ctx=gpu_ctx)
    assert res.tobytes() == g["results"].tobytes()
    np.testing.assert_array_equal(st["I_hat"], g["results"]["next_I_hat"])
    np.testing.assert_array_equal(st["kP"], g["states"]["kP"])


@pytest.mark.gpu
def test_pi_step_rejects_nonpositive_ts(gpu_ctx):
    from paper_2212_02197_b200 import engine
    st = K.make_pi_states(configs.make_scenario("pi"), 2)
    st["Ts"][1] = 0.0
    with pytest.raises(engine.DomainError):
        K.pi_step_batch(st, [335.0, 335.0], [335.0, 335.0], ctx=gpu_ctx)


def test_nmpc_step_rejects_bad_shapes_without_gpu_work():
    # shape checks happen before any device call
    g = group("one")
    with pytest.raises(Exception):
        K._f64(np.zeros(3), (4,))
    assert g["y"].shape[0] == 24
