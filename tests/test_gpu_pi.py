"""PI closed loop on the GPU vs the reference (run_closed_loop PI branch,
montecarlo.cpp:80-157): bitwise against the exact-libm reference build on the
committed golden fixtures, per-sample relative error <= 1e-9 against the
reference as shipped (glibc), trajectories step by step, and
size-independent properties at BASELINE sizes."""
import numpy as np
import pytest

from conftest import assert_records_equal, load_golden
from paper_2212_02197_b200 import configs, engine

pytestmark = pytest.mark.gpu

PI_CASES = ["pi_cfg0", "pi_cfg1", "pi_onestate", "pi_quiet"]


@pytest.mark.parametrize("name", PI_CASES)
def test_pi_records_bitwise_vs_exact_libm_reference(gpu_ctx, name):
    d, _, sc = load_golden(name)
    want = d["rec_xlibm"]
    got, _ = gpu_ctx.run(sc, int(d["first"]), len(want))
    assert_records_equal(got, want)


@pytest.mark.parametrize("name,frac", [("pi_cfg0", 1.0), ("pi_cfg1", 0.95), ("pi_onestate", 1.0), ("pi_quiet", 1.0)])
def test_pi_vs_glibc_reference_1e9(gpu_ctx, name, frac):
    """north_star tolerance: PI per-sample cost within 1e-9 of the reference as
    shipped. Samples in the oscillatory regime of config 1 are excluded by
    `frac` (see test_oracle.test_golden_pi_libm_variants_agree)."""
    d, _, sc = load_golden(name)
    want = d["rec_glibc"]
    got, _ = gpu_ctx.run(sc, int(d["first"]), len(want))
    np.testing.assert_array_equal(got["failed"], want["failed"])
    ok = want["failed"] == 0
    rel = np.abs(got["phi"][ok] - want["phi"][ok]) / np.abs(want["phi"][ok])
    assert np.mean(rel <= 1e-9) >= frac


@pytest.mark.parametrize("name", ["pi_cfg0", "pi_cfg1"])
def test_pi_trajectories_bitwise(gpu_ctx, name):
    d, kw, _ = load_golden(name)
    sct = configs.make_scenario(**kw, record=True)
    want = d["traj_xlibm"]
    rec, traj = gpu_ctx.run_traj(sct, int(d["first"]), want.shape[0])
    np.testing.assert_array_equal(traj, want)


def test_pi_offset_and_sharding_invariance(gpu_ctx):
    """Streams are keyed by global index: any split of [0, n) gives the same records."""
    sc = configs.make_scenario("pi", perturb=True)
    full, _ = gpu_ctx.run(sc, 0, 3000)
    a, _ = gpu_ctx.run(sc, 0, 1234)
    b, _ = gpu_ctx.run(sc, 1234, 3000 - 1234)
    assert_records_equal(np.concatenate([a, b]), full)
    one, _ = gpu_ctx.run(sc, 2999, 1)
    assert_records_equal(one, full[2999:])


def test_pi_full_config1_properties(gpu_ctx):
    """BASELINE config 1 at full size (30,000 sims): determinism, finiteness,
    aggregate consistency with the per-sample records."""
    sc = configs.make_scenario("pi", perturb=True)
    r1 = engine.run_monte_carlo(sc, 30000)
    r2 = engine.run_monte_carlo(sc, 30000)
    assert_records_equal(r1.records, r2.records)
    ok = r1.records["failed"] == 0
    assert np.all(np.isfinite(r1.records["phi"][ok])) and np.all(np.isnan(r1.records["phi"][~ok]))
    agg = r1.aggregate
    assert agg["n_sims"] == 30000 and agg["n_failed"] == int((~ok).sum())
    assert agg["min"] == r1.records["phi"][ok].min() and agg["max"] == r1.records["phi"][ok].max()
    # golden prefix still holds inside the big batch
    d, _, _ = load_golden("pi_cfg1")
    assert_records_equal(r1.records[:256], d["rec_xlibm"])


def test_pi_validation_errors_raise(gpu_ctx):
    bad = configs.make_scenario("pi")
    bad.Ns = 0
    with pytest.raises(engine.DomainError):
        gpu_ctx.run(bad, 0, 4)


@pytest.fixture(scope="module")
def pi_kernel_ctxs():
    out = {}
    for kind in ("lanes", "ws3", "ws7"):
        c = engine.Context(0)
        c.set_pi_kernel(kind)
        out[kind] = c
    yield out
    for c in out.values():
        c.close()


@pytest.mark.parametrize("kind", ["lanes", "ws3", "ws7"])
@pytest.mark.parametrize("name", PI_CASES)
def test_pi_kernel_variants_bitwise(pi_kernel_ctxs, kind, name):
    """Every PI kernel (NMPCMC_OPT_PI_KERNEL) reproduces the exact-libm
    reference fixtures bitwise, records and trajectories."""
    c = pi_kernel_ctxs[kind]
    d, kw, sc = load_golden(name)
    want = d["rec_xlibm"]
    got, _ = c.run(sc, int(d["first"]), len(want))
    assert_records_equal(got, want)
    if "traj_xlibm" in d:
        sct = configs.make_scenario(**kw, record=True)
        _, traj = c.run_traj(sct, int(d["first"]), d["traj_xlibm"].shape[0])
        np.testing.assert_array_equal(traj, d["traj_xlibm"])


@pytest.mark.parametrize("kw", [dict(perturb=True), dict(perturb=True, sigma_abc=True), dict(one_state=True)])
def test_pi_kernel_variants_agree_at_scale(pi_kernel_ctxs, kw):
    """10,000 samples (a full wave of the 3-producer kernel) with a ragged
    tail: all PI kernels give identical records and work counters; dense
    normal reads (diffusion on every state) and the one-state plant too."""
    from paper_2212_02197_b200 import abi
    tv = abi.ONE_STATE if kw.get("one_state") else abi.THREE_STATE
    sc = configs.make_scenario("pi", perturb=kw.get("perturb", False), truth_variant=tv)
    if kw.get("sigma_abc"):
        sc.truth.sigmaA = 0.01
        sc.truth.sigmaB = 0.02
    n = 10007
    res = {k: c.run(sc, 5, n, counters=True) for k, c in pi_kernel_ctxs.items()}
    base_rec, base_cnt = res["lanes"]
    for k in ("ws3", "ws7"):
        assert_records_equal(res[k][0], base_rec)
        np.testing.assert_array_equal(res[k][1], base_cnt)
