"""K5 -- the batched standalone QP kernel (csrc/qp_batch_kernel.cuh) --
against the reference's solve_qp / riccati_factor_solve on the committed
fixtures (tests/golden/qp_batch.npz): solutions, statuses and iteration
counts bitwise equal; plus batch-order invariance on a large random batch."""
import numpy as np
import pytest

from paper_2212_02197_b200 import qp as Q
from test_qp_oracle import G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", sorted(G))
def test_qp_batch_bitwise_vs_reference(gpu_ctx, name):
    g = G[name]
    N, nx, nu, max_iter, mode = (int(v) for v in g["dims"])
    sol, st, it = Q.solve_qp_batch(g["packed"], nx, nu, float(g["tol"]), max_iter, mode == 1, ctx=gpu_ctx, raw=True)
    np.testing.assert_array_equal(st, g["status"])
    np.testing.assert_array_equal(it, g["iters"])
    np.testing.assert_array_equal(sol, g["sol"])


def test_qp_batch_order_invariance(gpu_ctx):
    rng = np.random.default_rng(5)
    qps = [Q.random_instance(rng, 30, 4, 2) for _ in range(3000)]
    packed = Q.pack(qps, 4, 2)
    a, sa, ia = Q.solve_qp_batch(packed, 4, 2, ctx=gpu_ctx, raw=True)
    perm = rng.permutation(len(qps))
    b, sb, ib = Q.solve_qp_batch(packed[perm], 4, 2, ctx=gpu_ctx, raw=True)
    np.testing.assert_array_equal(b, a[perm])
    np.testing.assert_array_equal(sb, sa[perm])
    assert np.mean(sa == Q.OPTIMAL) > 0.99
