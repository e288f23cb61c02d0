"""sqp_solve through the SqpProblem interface (sqp.hpp:15-25) on stagewise
quadratic NLPs -- the problem class the reference's SQP tests pose -- on the
GPU (nmpcmc_gpu_sqp_solve_qnlp_batch) against the reference's own sqp_solve
(tests/golden/qnlp_batch.npz, make_golden.py qnlp): iterates, multipliers,
convergence flags and iteration counts bitwise, cold and warm starts,
n_x = 1 and 3. CPU: the fixture is the reference, and its solutions are the
analytic KKT points (SPEC.md acceptance criterion 2)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import lib as O
from paper_2212_02197_b200 import qp as Q

D = np.load(os.path.join(GOLDEN, "qnlp_batch.npz"))
TAGS = ("n1", "n3")
FIELDS = ("xi", "lambda", "pi_l", "pi_u", "converged", "iterations", "status")


def group(tag):
    return {k.split("__", 1)[1]: D[k] for k in D.files if k.startswith(tag + "__")}


def unpack(p, N, nx):
    x0, lo, hi = p[:nx], p[nx], p[nx + 1]
    st = p[nx + 2:].reshape(N, -1)
    R, r = st[:, 0], st[:, 1]
    o = 2
    Qm = st[:, o:o + nx * nx].reshape(N, nx, nx).transpose(0, 2, 1)
    o += nx * nx
    q = st[:, o:o + nx]
    o += nx
    A = st[:, o:o + nx * nx].reshape(N, nx, nx).transpose(0, 2, 1)
    o += nx * nx
    Bm = st[:, o:o + nx]
    o += nx
    c = st[:, o:o + nx]
    return x0, lo, hi, R, r, Qm, q, A, Bm, c


@pytest.mark.skipif(not O.ref_available(), reason="reference build not present")
@pytest.mark.parametrize("tag", TAGS)
def test_fixture_is_the_reference(tag):
    g = group(tag)
    N, nx = (int(v) for v in g["dims"])
    opts = Q.default_sqp_options(max_iter=50)
    cold = O.sqp_solve_qnlp_batch(O.ref("xlibm"), g["problems"], N, nx, opts)
    for f in FIELDS:
        np.testing.assert_array_equal(cold[f], g["cold_" + f], err_msg=f)


@pytest.mark.parametrize("tag", TAGS)
def test_solutions_are_kkt_points(tag):
    """Feasible, bounds respected, and stationary: grad f + J' lam + pi_u - pi_l = 0
    with complementarity, to 1e-6 (criterion 2's analytic KKT point)."""
    g = group(tag)
    N, nx = (int(v) for v in g["dims"])
    W = 1 + nx
    for p, xi, lam, pl, pu in zip(g["problems"], g["cold_xi"], g["cold_lambda"], g["cold_pi_l"], g["cold_pi_u"]):
        x0, lo, hi, R, r, Qm, q, A, Bm, c = unpack(p, N, nx)
        u = xi[0::W]
        X = np.stack([xi[k * W + 1:k * W + 1 + nx] for k in range(N)])
        xprev = np.vstack([x0, X[:-1]])
        defect = X - (np.einsum("kij,kj->ki", A, xprev) + Bm * u[:, None] + c)
        assert np.abs(defect).max() < 1e-6
        assert np.all(u >= lo - 1e-9) and np.all(u <= hi + 1e-9)
        L = lam.reshape(N, nx)
        # stationarity in u_k: R u + r - B' lam_k + pi_u - pi_l (g = x_{k+1} - F)
        gu = R * u + r - np.einsum("ki,ki->k", Bm, L) + pu - pl
        assert np.abs(gu).max() < 1e-5
        # stationarity in x_{k+1}: Q x + q + lam_k - A_{k+1}' lam_{k+1}
        gx = np.einsum("kij,kj->ki", Qm, X) + q + L
        gx[:-1] -= np.einsum("kji,kj->ki", A[1:], L[1:])
        assert np.abs(gx).max() < 1e-5
        assert np.all(pl >= 0) and np.all(pu >= 0)
        assert np.abs(pl * (u - lo)).max() < 1e-5 and np.abs(pu * (hi - u)).max() < 1e-5


def test_pack_layout_matches_abi():
    assert Q.qnlp_doubles(12, 1) == 1 + 2 + 12 * (2 + 2 + 3)
    assert Q.qnlp_doubles(8, 3) == 3 + 2 + 8 * (2 + 18 + 9)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("start", ["cold", "warm"])
def test_qnlp_batch_bitwise_vs_reference(gpu_ctx, tag, start):
    g = group(tag)
    N, nx = (int(v) for v in g["dims"])
    got = Q.solve_qnlp_batch(g["problems"], N, nx, Q.default_sqp_options(max_iter=50),
                             xi0=g["xi0"] if start == "warm" else None, ctx=gpu_ctx)
    for f in FIELDS:
        np.testing.assert_array_equal(got[f], g[f"{start}_{f}"], err_msg=f)


@pytest.mark.gpu
def test_qnlp_rejects_bad_dims(gpu_ctx):
    from paper_2212_02197_b200 import engine
    with pytest.raises(engine.DimensionMismatch):
        Q.solve_qnlp_batch(np.zeros((2, Q.qnlp_doubles(4, 2))), 4, 2, ctx=gpu_ctx)
