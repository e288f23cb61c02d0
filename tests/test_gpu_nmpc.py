"""NMPC closed loop on the GPU vs the reference (run_closed_loop NMPC branch,
montecarlo.cpp:80-157 -> nmpc_step controllers.cpp:114-212 -> sqp_solve /
solve_qp / shoot / CD-EKF): per-sample records and full trajectories bitwise
equal to the reference's exact-libm build on the committed golden fixtures
(so the north_star's 1e-5 on >= 99.9% of samples holds with margin 0), failure
flags and OCP counters included."""
import numpy as np
import pytest

from conftest import assert_records_equal, load_golden
from paper_2212_02197_b200 import configs, engine

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["generic_warp", "warp"])
def nctx(request, gpu_ctx):
    """The context with one of the two warp-per-sample NMPC kernels selected (K3w / K3):
    both must reproduce the reference bitwise."""
    gpu_ctx.set_nmpc_kernel(request.param)
    yield gpu_ctx
    gpu_ctx.set_nmpc_kernel("warp")

NMPC_CASES = ["nmpc_n30_short", "nmpc_n60_pert_short", "nmpc_n120_short", "nmpc_cfg2"]


@pytest.mark.parametrize("name", NMPC_CASES)
def test_nmpc_records_bitwise_vs_exact_libm_reference(nctx, name):
    d, _, sc = load_golden(name)
    want = d["rec_xlibm"]
    got, _ = nctx.run(sc, int(d["first"]), len(want))
    assert_records_equal(got, want)


@pytest.mark.parametrize("name", NMPC_CASES)
def test_nmpc_trajectories_bitwise(nctx, name):
    d, kw, _ = load_golden(name)
    sct = configs.make_scenario(**kw, record=True)
    want = d["traj_xlibm"]
    _, traj = nctx.run_traj(sct, int(d["first"]), want.shape[0])
    np.testing.assert_array_equal(traj, want)


@pytest.mark.parametrize("name", NMPC_CASES)
def test_nmpc_vs_glibc_reference_distribution(nctx, name):
    """Against the reference as shipped (glibc libm) per-sample agreement is
    limited by libm rounding amplified through iteration-capped SQP solves
    (SURVEY.md §0.5); report it and require the bulk to agree."""
    d, _, sc = load_golden(name)
    want = d["rec_glibc"]
    got, _ = nctx.run(sc, int(d["first"]), len(want))
    same_flag = np.mean(got["failed"] == want["failed"])
    both = (got["failed"] == 0) & (want["failed"] == 0)
    rel = np.abs(got["phi"][both] - want["phi"][both]) / np.abs(want["phi"][both])
    print(f"{name}: failed-flag agreement {same_flag:.3f}, phi within 1e-5 on "
          f"{np.mean(rel <= 1e-5):.3f} of {both.sum()} jointly successful samples")
    assert same_flag >= 0.75
    assert np.mean(rel <= 1e-5) >= 0.5


def test_nmpc_sharding_invariance(nctx):
    sc = configs.make_scenario("nmpc", N=30, n_steps=30, perturb=True)
    full, _ = nctx.run(sc, 0, 300)
    a, _ = nctx.run(sc, 0, 137)
    b, _ = nctx.run(sc, 137, 163)
    assert_records_equal(np.concatenate([a, b]), full)


def test_nmpc_counters_consistent(nctx):
    sc = configs.make_scenario("nmpc", N=30, n_steps=30)
    rec, cnt = nctx.run(sc, 0, 64, counters=True)
    ok = rec["failed"] == 0
    assert np.all(cnt["control_steps"][ok] == 30)
    assert np.all(cnt["control_steps"] == rec["ocp_solves"])
    assert np.all(cnt["qp_solves"] >= cnt["sqp_iterations"])
    assert np.all(cnt["ls_evals"] >= cnt["sqp_iterations"])
    assert np.all(cnt["shoot_full"] <= 30 * (cnt["ls_evals"] + rec["ocp_solves"]))


def test_nmpc_kernels_agree_at_scale(gpu_ctx):
    """K3 (warp per sample) and K3g (generic, thread per sample) on 600 perturbed
    config-3 samples, 60 control steps: identical records."""
    sc = configs.make_scenario("nmpc", N=60, n_steps=60, perturb=True)
    gpu_ctx.set_nmpc_kernel("warp")
    a, ca = gpu_ctx.run(sc, 1000, 600, counters=True)
    gpu_ctx.set_nmpc_kernel("generic")
    b, cb = gpu_ctx.run(sc, 1000, 600, counters=True)
    gpu_ctx.set_nmpc_kernel("warp")
    assert_records_equal(a, b)
    for f in ("control_steps", "ipm_stage_iters", "sqp_iterations", "qp_solves", "ls_evals"):
        np.testing.assert_array_equal(ca[f], cb[f])
