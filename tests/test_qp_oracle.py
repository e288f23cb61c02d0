"""Batched QP fixtures (tests/golden/qp_batch.npz) against the reference's
solve_qp / riccati_factor_solve (qp.cpp): pinned to the compiled reference
when it is present, and checked for the properties the reference's own
tests/test_qp.cpp asserts (dense KKT stationarity, bound feasibility,
complementarity, IPM == Riccati on unconstrained problems, the scalar edge
cases, MaxIter, Failed / NotPositiveDefinite, DomainError). CPU only."""
import os

import numpy as np
import pytest

from oracle import lib as O
from paper_2212_02197_b200 import qp as Q

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "qp_batch.npz")


def groups():
    d = np.load(GOLD)
    out = {}
    for key in d.files:
        g, f = key.split("__")
        out.setdefault(g, {})[f] = d[key]
    return out


G = groups()


def _sols(g):
    N, nx, nu = (int(v) for v in g["dims"][:3])
    return Q.unpack(g["sol"], g["status"], g["iters"], N, nx, nu), N, nx, nu


@pytest.mark.skipif(not O.ref_available(), reason="reference build not present")
@pytest.mark.parametrize("name", sorted(G))
def test_fixture_is_the_reference(name):
    g = G[name]
    N, nx, nu, max_iter, mode = (int(v) for v in g["dims"])
    sol, st, it = O.solve_qp_batch(O.ref("glibc"), g["packed"], nx, nu, float(g["tol"]), max_iter, mode == 1)
    np.testing.assert_array_equal(sol, g["sol"])
    np.testing.assert_array_equal(st, g["status"])
    np.testing.assert_array_equal(it, g["iters"])


def _stage(packed_qp, k, nx, nu):
    p = packed_qp[k]
    o = np.cumsum([0, nx * nx, nx * nu, nu * nu, nx, nu, nx * nx, nx * nu, nx, nu, nu])
    f = lambda i, shape: p[o[i]:o[i + 1]].reshape(shape, order="F")  # noqa: E731
    return dict(Q=f(0, (nx, nx)), M=f(1, (nx, nu)), R=f(2, (nu, nu)), q=f(3, (nx,)), r=f(4, (nu,)),
                Jx=f(5, (nx, nx)), Ju=f(6, (nx, nu)), b=f(7, (nx,)), lb=f(8, (nu,)), ub=f(9, (nu,)))


def _kkt_residual(packed_qp, s, N, nx, nu):
    """grad of the Lagrangian (the reference's sign convention, qp.cpp:237-284)
    of the returned (delta_xi, mu, nu_l, nu_u), assembled densely."""
    w = nu + nx
    uo = lambda k: k * w  # noqa: E731
    xo = lambda k: (k - 1) * w + nu  # noqa: E731
    z, g = s.delta_xi, np.zeros(N * w)
    for k in range(N + 1):
        st = _stage(packed_qp, k, nx, nu)
        if k < N:
            u = z[uo(k):uo(k) + nu]
            g[uo(k):uo(k) + nu] += st["R"] @ u + st["r"] - st["Ju"].T @ s.mu[k * nx:(k + 1) * nx]
            g[uo(k):uo(k) + nu] += s.nu_u[k * nu:(k + 1) * nu] - s.nu_l[k * nu:(k + 1) * nu]
            g[xo(k + 1):xo(k + 1) + nx] += s.mu[k * nx:(k + 1) * nx]
        if k >= 1:
            x = z[xo(k):xo(k) + nx]
            g[xo(k):xo(k) + nx] += st["Q"] @ x + st["q"]
            if k < N:
                u = z[uo(k):uo(k) + nu]
                g[xo(k):xo(k) + nx] += st["M"] @ u - st["Jx"].T @ s.mu[k * nx:(k + 1) * nx]
                g[uo(k):uo(k) + nu] += st["M"].T @ x
    return g


@pytest.mark.parametrize("name", ["rand_box", "big", "limits", "minimal"])
def test_box_qp_solutions_are_kkt_points(name):
    g = G[name]
    sols, N, nx, nu = _sols(g)
    active = 0
    for b, s in enumerate(sols):
        assert s.status == Q.OPTIMAL and s.iterations <= 50
        assert np.max(np.abs(_kkt_residual(g["packed"][b], s, N, nx, nu))) <= 1e-6
        for k in range(N):
            st = _stage(g["packed"][b], k, nx, nu)
            u = s.delta_xi[k * (nu + nx):k * (nu + nx) + nu]
            nl, nuu = s.nu_l[k * nu:(k + 1) * nu], s.nu_u[k * nu:(k + 1) * nu]
            assert np.all(u >= st["lb"]) and np.all(u <= st["ub"])
            assert np.all(nl >= 0) and np.all(nuu >= 0)
            fl, fu = np.isfinite(st["lb"]), np.isfinite(st["ub"])
            assert np.all(np.abs(nl[fl] * (u[fl] - st["lb"][fl])) <= 1e-6)
            assert np.all(np.abs(nuu[fu] * (st["ub"][fu] - u[fu])) <= 1e-6)
            active += int(np.sum(nl > 1e-6) + np.sum(nuu > 1e-6))
    if name in ("rand_box", "big"):
        assert active > 30  # the bounds matter in this population


@pytest.mark.parametrize("name", ["rand_unc", "dint"])
def test_interior_point_equals_riccati_when_unconstrained(name):
    ip, _, _, _ = _sols(G[name])
    rc, _, _, _ = _sols(G[name + "_riccati"])
    for a, b in zip(ip, rc):
        assert a.status == Q.OPTIMAL and a.iterations <= 2
        np.testing.assert_allclose(a.delta_xi, b.delta_xi, rtol=1e-8, atol=1e-12)
        np.testing.assert_allclose(a.mu, b.mu, rtol=1e-8, atol=1e-12)
        assert np.all(a.nu_l == 0) and np.all(a.nu_u == 0)


def test_scalar_edge_cases():
    s, _, _, _ = _sols(G["scalar"])
    assert s[0].status == Q.OPTIMAL and abs(s[0].delta_xi[0] + 2.0) < 1e-8      # interior minimiser
    assert s[1].status == Q.OPTIMAL and abs(s[1].delta_xi[0] + 1.0) < 1e-8 and s[1].nu_l[0] > 0.5  # active lower
    assert s[2].status == Q.OPTIMAL and s[2].delta_xi[0] == 0.5                 # pinned input
    assert s[3].status == Q.OPTIMAL and np.max(np.abs(s[3].delta_xi)) <= 1e-10      # zero data, zero step
    assert s[4].status == Q.FAILED                                               # indefinite
    assert s[5].status == Q.DOMAIN_ERROR                                         # lb > ub
    r, _, _, _ = _sols(G["scalar_riccati"])
    assert r[4].status == Q.NOT_POSITIVE_DEFINITE
    m, _, _, _ = _sols(G["maxiter"])
    assert m[0].status == Q.MAXITER and m[0].iterations == 5 and -0.5 <= m[0].delta_xi[0] <= 0.5
