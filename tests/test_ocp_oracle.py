"""Batched OCP fixtures (tests/golden/ocp_batch.npz): the reference's
sqp_solve on the regulator OcpProblem, pinned to the compiled reference when
it is present, plus sanity of the solutions. CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import lib as O
from paper_2212_02197_b200 import configs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ocp_batch.npz")


def ocp_groups():
    d = np.load(GOLD)
    out = {}
    for tag in ("one", "three"):
        g = {k.split("__", 1)[1]: d[k] for k in d.files if k.startswith(tag + "__")}
        g["sc"] = configs.make_scenario(**json.loads(str(g["kwargs"])))
        out[tag] = g
    return out


G = ocp_groups()
FIELDS = ("xi", "lambda", "pi_l", "pi_u", "converged", "status")


@pytest.mark.skipif(not O.ref_available(), reason="reference build not present")
@pytest.mark.parametrize("tag", ["one", "three"])
def test_fixture_is_the_reference(tag):
    g = G[tag]
    cold = O.solve_ocp_batch(O.ref("xlibm"), g["sc"], g["x0"], g["t0"])
    warm = O.solve_ocp_batch(O.ref("xlibm"), g["sc"], g["x0"], g["t0"], xi0=g["xi0"])
    for f in FIELDS:
        np.testing.assert_array_equal(cold[f], g["cold_" + f])
        np.testing.assert_array_equal(warm[f], g["warm_" + f])


@pytest.mark.parametrize("tag", ["one", "three"])
def test_fixture_solutions_are_sane(tag):
    g = G[tag]
    assert np.all(g["cold_status"] == 0)
    assert np.mean(g["cold_converged"]) > 0.9
    sc = g["sc"]
    nx = g["x0"].shape[1]
    u = g["cold_xi"][:, :: 1 + nx]
    assert np.all(np.isfinite(g["cold_xi"]))
    assert np.all(u >= sc.u_min - 1e-9) and np.all(u <= sc.u_max + 1e-9)
    assert np.all(g["cold_pi_l"] >= 0) and np.all(g["cold_pi_u"] >= 0)
