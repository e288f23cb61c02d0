"""Generate the committed golden fixtures from the UNMODIFIED reference.

Runs only in the dev container (needs /root/reference to build oracle/_ref).
Every fixture stores the scenario kwargs (configs.make_scenario) and the raw
scenario bytes, the per-sample records of the reference's run_closed_loop /
run_monte_carlo in both libm link variants ("xlibm" = exact-libm parity mode,
"glibc" = reference as shipped), and a few full trajectories.

  python tests/golden/make_golden.py [pi|nmpc|rng|all]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import lib as O  # noqa: E402
from paper_2212_02197_b200 import configs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def gen_case(name, kwargs, n_sims, n_traj, first=0, workers=None):
    sc = configs.make_scenario(**kwargs)
    data = {"kwargs": np.array(json.dumps(kwargs)), "scenario": np.frombuffer(bytes(sc), dtype=np.uint8),
            "first": np.array(first)}
    for libm in ("xlibm", "glibc"):
        L = O.ref(libm)
        t = time.time()
        rec, wall = O.run_batch(L, sc, first, n_sims, workers)
        print(f"{name} {libm}: {n_sims} sims in {wall:.2f}s (failed {rec['failed'].sum()})", flush=True)
        data[f"rec_{libm}"] = rec
    if n_traj:
        sct = configs.make_scenario(**kwargs, record=True)
        L = O.ref("xlibm")
        nbar = int(round((sct.tf - sct.t0) / sct.Ts))
        rows = nbar + 1
        trajs = []
        for i in range(n_traj):
            _, tr = O.run_traj(L, sct, first + i, rows)
            trajs.append(tr)
        data["traj_xlibm"] = np.array(trajs)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **data)


def gen_rng():
    L = O.ref("xlibm")
    G = O.ref("glibc")
    import ctypes as C
    streams = [(12345, 7), (42, 0), (0, 0), (2**64 - 1, 2**63 + 5)]
    out = {}
    for i, (seed, stream) in enumerate(streams):
        for name, lib in (("xlibm", L), ("glibc", G)):
            v = np.zeros(257)
            lib.nmpcmc_ref_normals(C.c_uint64(seed), C.c_uint64(stream), 257, v.ctypes.data_as(C.POINTER(C.c_double)))
            out[f"normals_{name}_{i}"] = v
    out["streams"] = np.array(streams, dtype=np.uint64)
    rs = np.random.default_rng(7)
    ck = rs.integers(0, 2**32, size=(512, 6), dtype=np.uint64).astype(np.uint32)
    blocks = np.zeros((512, 4), dtype=np.uint32)
    for i in range(512):
        L.nmpcmc_ref_philox_block(ck[i].ctypes.data_as(C.POINTER(C.c_uint32)),
                                  blocks[i].ctypes.data_as(C.POINTER(C.c_uint32)))
    out["philox_in"] = ck
    out["philox_out"] = blocks
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **out)
    print("rng done")


def gen_qp():
    """Batched QP fixtures: the reference's solve_qp /
    riccati_factor_solve on packed batches, mirroring the cases of the
    reference's tests/test_qp.cpp. Groups of equal dimensions; each stores
    the packed input, the dims and the reference's outputs."""
    from paper_2212_02197_b200 import qp as Q
    L = O.ref("glibc")  # no libm on this path: both link variants agree
    inf = np.inf
    rng = np.random.default_rng(20260101)
    groups = {}

    def add(name, qps, nx, nu, tol=1e-10, max_iter=50, riccati_only=False):
        packed = Q.pack(qps, nx, nu)
        sol, st, it = O.solve_qp_batch(L, packed, nx, nu, tol, max_iter, riccati_only)
        groups[name] = dict(packed=packed, dims=np.array([len(qps[0]) - 1, nx, nu, max_iter, int(riccati_only)]),
                            tol=np.array(tol), sol=sol, status=st, iters=it)
        print(f"qp {name}: batch {len(qps)} status {np.bincount(st, minlength=5).tolist()} iters {it.min()}..{it.max()}")

    add("rand_box", [Q.random_instance(rng, 4, 3, 2) for _ in range(60)], 3, 2)
    unc = [Q.random_instance(rng, 4, 3, 2, bounded=False) for _ in range(10)]
    add("rand_unc", unc, 3, 2)
    add("rand_unc_riccati", unc, 3, 2, riccati_only=True)
    dint = [Q.double_integrator(rng, 20, 0.1) for _ in range(5)]
    add("dint", dint, 2, 1)
    add("dint_riccati", dint, 2, 1, riccati_only=True)
    add("big", [Q.random_instance(rng, 60, 6, 3) for _ in range(12)], 6, 3)
    scal = [Q.scalar_instance(1.0, 2.0, 1.0, 0.0, 0.0, 0.0, -10.0, 10.0),   # slack bounds: u* = -2
            Q.scalar_instance(1.0, 2.0, 1.0, 0.0, 0.0, 0.0, -1.0, 10.0),    # active lower bound
            Q.scalar_instance(1.0, 2.0, 1.0, 0.0, 0.0, 0.0, 0.5, 0.5),      # pinned input
            Q.scalar_instance(1.0, 0.0, 1.0, 0.0, 1.0, 0.0, -1.0, 1.0),     # all-zero linear data
            Q.scalar_instance(-1.0, 2.0, 1.0, 0.0, 0.0, 0.0, -inf, inf),    # indefinite stage Hessian
            Q.scalar_instance(1.0, 2.0, 1.0, 0.0, 0.0, 0.0, 1.0, -1.0),     # lb > ub
            Q.scalar_instance(2.0, -1.0, 3.0, 0.5, 0.7, 0.2, -inf, 0.3)]    # one-sided box
    add("scalar", scal, 1, 1)
    add("scalar_riccati", scal, 1, 1, riccati_only=True)
    add("maxiter", [Q.scalar_instance(1.0, 2.0, 1.0, 0.0, 0.0, 0.0, -0.5, 0.5)], 1, 1, tol=0.0, max_iter=5)
    # dimension limits of the device kernel (n_x <= 8, n_u <= 4) and the minimal horizon
    add("limits", [Q.random_instance(rng, 8, 8, 4) for _ in range(8)], 8, 4)
    add("minimal", [Q.random_instance(rng, 1, 2, 2) for _ in range(8)], 2, 2)
    add("minimal_riccati", [Q.random_instance(rng, 1, 2, 2, bounded=False) for _ in range(4)], 2, 2,
        riccati_only=True)
    out = {}
    for g, d in groups.items():
        for k, v in d.items():
            out[f"{g}__{k}"] = v
    np.savez_compressed(os.path.join(OUT, "qp_batch.npz"), **out)


def gen_ocp():
    """Batched OCP fixtures: the reference's sqp_solve on the regulator
    OcpProblem (one-state config 2 at N=60; three-state at N=30), cold starts
    from random states/times, and one warm group from a given iterate."""
    rng = np.random.default_rng(424242)
    out = {}
    for tag, kw, B in (("one", dict(controller="nmpc", N=60), 48),
                       ("three", dict(controller="nmpc", N=30, ctrl_variant=0), 16)):
        sc = configs.make_scenario(**kw)
        nx = 3 if kw.get("ctrl_variant", 1) == 0 else 1
        T = rng.uniform(322.0, 348.0, B)
        p = configs.study_params()
        x0 = np.array([configs.manifold_state(p, t)[3 - nx:] for t in T])
        x0 *= 1.0 + 0.01 * rng.standard_normal(x0.shape)
        t0 = rng.uniform(0.0, 7000.0, B)
        ref = O.solve_ocp_batch(O.ref("xlibm"), sc, x0, t0)
        xi_warm = np.roll(ref["xi"], 1, axis=0)  # another instance's solution as the start
        warm = O.solve_ocp_batch(O.ref("xlibm"), sc, x0, t0, xi0=xi_warm)
        out[f"{tag}__kwargs"] = np.array(json.dumps(kw))
        out[f"{tag}__x0"], out[f"{tag}__t0"], out[f"{tag}__xi0"] = x0, t0, xi_warm
        for k, v in ref.items():
            out[f"{tag}__cold_{k}"] = v
        for k, v in warm.items():
            out[f"{tag}__warm_{k}"] = v
        print(f"ocp {tag}: {B} instances, converged cold {ref['converged'].sum()} warm {warm['converged'].sum()}, "
              f"status {np.bincount(ref['status']).tolist()}")
    np.savez_compressed(os.path.join(OUT, "ocp_batch.npz"), **out)


def gen_full():
    """Round 2: full-length (720-step) pins of the configs that carry the
    claims: the bench's config 3 (N=60, perturbed) at
    indices 0.. and inside the bench's own index range (9,472..), config 4 at
    N=30 and N=120, config 3 with the three-state controller model, and 1,000
    samples of config 2 (both libm variants) for the distribution test."""
    gen_case("nmpc_cfg3_full", dict(controller="nmpc", N=60, perturb=True), 64, 1)
    gen_case("nmpc_cfg3_full_b", dict(controller="nmpc", N=60, perturb=True), 32, 0, first=9472)
    gen_case("nmpc_cfg4_n30_full", dict(controller="nmpc", N=30, perturb=True), 32, 0)
    gen_case("nmpc_cfg4_n120_full", dict(controller="nmpc", N=120, perturb=True), 32, 0)
    gen_case("nmpc3_cfg3_full", dict(controller="nmpc", N=60, perturb=True, ctrl_variant=0), 16, 0)


def gen_dist():
    """1,000 samples of BASELINE config 2 (N=60, unperturbed, 720 steps) in
    both libm variants: the Φ-distribution test's reference sample."""
    gen_case("nmpc_cfg2_1000", dict(controller="nmpc", N=60), 1000, 0)


def gen_steps():
    """Controller-level fixtures (round 2): the reference's make_nmpc_state +
    nmpc_step (controllers.cpp:25-48, :114-212) over T steps for B
    controllers with measurement sequences around a closed-loop trajectory,
    per-instance priors, a non-finite measurement and a measurement far
    outside the model's domain (exceptions mid-sequence), with the
    scenario's setpoint profile and with explicit setpoints; and pi_step
    (controllers.cpp:12-23) on random states including saturation."""
    rng = np.random.default_rng(777)
    out = {}
    for tag, kw, B, T, explicit in (("one", dict(controller="nmpc", N=30), 24, 12, False),
                                    ("one_sp", dict(controller="nmpc", N=20), 12, 8, True),
                                    ("three", dict(controller="nmpc", N=20, ctrl_variant=0), 8, 6, False)):
        sc = configs.make_scenario(**kw)
        nx = 3 if kw.get("ctrl_variant", 1) == 0 else 1
        p = configs.study_params()
        T0 = rng.uniform(330.0, 340.0, B)
        x0_hat = np.array([configs.manifold_state(p, t)[3 - nx:] for t in T0])
        P0 = np.zeros((B, nx * nx))
        for i in range(nx):
            P0[:, i * nx + i] = 10.0 ** rng.uniform(-7, -4, B)
        t = np.tile(np.arange(T) * sc.Ts, (B, 1)) + rng.uniform(0, 3000, (B, 1)).round()
        y = T0[:, None] + np.cumsum(rng.normal(0.0, 0.8, (B, T)), axis=1)
        y[1, T // 2] = np.nan          # nmpc_step throws NonFiniteState, state untouched
        y[2, T // 3] = -500.0          # estimate leaves the model's domain
        y[3, 1] = 1e6                  # absurd measurement
        sp = rng.uniform(325.0, 345.0, (B, T, sc.N)) if explicit else None
        u, diag, fin = O.nmpc_steps(O.ref("xlibm"), sc, x0_hat, P0, t, y, sp)
        out[f"{tag}__kwargs"] = np.array(json.dumps(kw))
        out[f"{tag}__x0_hat"], out[f"{tag}__P0"], out[f"{tag}__t"], out[f"{tag}__y"] = x0_hat, P0, t, y
        if explicit:
            out[f"{tag}__sp"] = sp
        out[f"{tag}__u"], out[f"{tag}__diag"] = u, diag
        for k, v in fin.items():
            out[f"{tag}__fin_{k}"] = v
        print(f"steps {tag}: {B}x{T}, status {np.bincount(diag['status'].ravel()).tolist()}, "
              f"converged {diag['converged'].mean():.2f}")
    from paper_2212_02197_b200 import controllers as K
    n = 4096
    st = np.zeros(n, dtype=K.PI_STATE_DTYPE)
    st["kP"], st["kI"], st["kaw"] = rng.uniform(-20, 0, n), rng.uniform(-0.5, 0, n), rng.uniform(-0.5, 0.5, n)
    st["Ts"], st["u_bar"] = rng.uniform(0.5, 20, n), rng.uniform(0, 1000, n)
    st["u_min"], st["u_max"] = rng.uniform(0, 200, n), rng.uniform(300, 1000, n)
    st["I_hat"] = rng.normal(0, 300, n)
    y = rng.normal(335, 10, n)
    ybar = rng.normal(335, 5, n)
    L = O.ref("xlibm")
    res = np.zeros(n, dtype=K.PI_RESULT_DTYPE)
    import ctypes as C
    L.nmpcmc_ref_pi_step.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_void_p]
    L.nmpcmc_ref_pi_step.restype = None
    for i in range(n):
        s = np.array([st[i][f] for f in K.PI_STATE_DTYPE.names])
        o = np.zeros(7)
        L.nmpcmc_ref_pi_step(s.ctypes.data, float(y[i]), float(ybar[i]), o.ctypes.data)
        res[i] = tuple(o)
    sat = np.mean((res["u"] == st["u_min"]) | (res["u"] == st["u_max"]))
    print(f"pi_step: {n} states, saturated {sat:.2f}")
    out["pi__states"], out["pi__y"], out["pi__ybar"], out["pi__results"] = st, y, ybar, res
    np.savez_compressed(os.path.join(OUT, "controller_steps.npz"), **out)


def gen_qnlp():
    """SQP through the SqpProblem interface on random stagewise quadratic NLPs
    (the reference's own SQP-test problem class): the reference's sqp_solve
    on QnlpProblem (oracle/ref_driver.cpp), n_x = 1 and 3, loose and tight
    input bounds, zero and random starts."""
    from paper_2212_02197_b200 import qp as Q
    rng = np.random.default_rng(31337)
    out = {}
    for tag, N, nx, B in (("n1", 12, 1, 40), ("n3", 8, 3, 40)):
        probs = []
        for b in range(B):
            R = rng.uniform(0.1, 2.0, N)
            r = rng.normal(0, 1, N)
            Qs, qs, As, Bs, cs = [], [], [], [], []
            for k in range(N):
                M = rng.normal(0, 1, (nx, nx))
                Qs.append(M @ M.T + 0.1 * np.eye(nx))
                qs.append(rng.normal(0, 1, nx))
                As.append(0.9 * np.eye(nx) + 0.2 * rng.normal(0, 1, (nx, nx)))
                Bs.append(rng.normal(0, 1, nx))
                cs.append(0.1 * rng.normal(0, 1, nx))
            tight = b % 2 == 1
            lo, hi = (-0.3, 0.4) if tight else (-50.0, 50.0)
            probs.append(Q.pack_qnlp(rng.normal(0, 1, nx), lo, hi, R, r, Qs, qs, As, Bs, cs))
        probs = np.array(probs)
        opts = Q.default_sqp_options(max_iter=50)
        xi0 = rng.normal(0, 0.5, (B, N * (1 + nx)))
        cold = O.sqp_solve_qnlp_batch(O.ref("xlibm"), probs, N, nx, opts)
        warm = O.sqp_solve_qnlp_batch(O.ref("xlibm"), probs, N, nx, opts, xi0=xi0)
        out[f"{tag}__dims"] = np.array([N, nx])
        out[f"{tag}__problems"], out[f"{tag}__xi0"] = probs, xi0
        for k, v in cold.items():
            out[f"{tag}__cold_{k}"] = v
        for k, v in warm.items():
            out[f"{tag}__warm_{k}"] = v
        print(f"qnlp {tag}: {B} problems, converged cold {cold['converged'].sum()} warm {warm['converged'].sum()}, "
              f"iterations {cold['iterations'].mean():.1f}, status {np.bincount(cold['status']).tolist()}")
    np.savez_compressed(os.path.join(OUT, "qnlp_batch.npz"), **out)


def gen_fd():
    """Finite-difference controller jacobians (model.cpp:54-124): the
    reference with the controller model's analytic jacobians removed
    (nmpcmc_ref_set_ctrl_fd), one- and three-state controller models."""
    for libm in ("xlibm", "glibc"):
        O.ref(libm).nmpcmc_ref_set_ctrl_fd(1)
    try:
        gen_case("nmpc_fd_n30", dict(controller="nmpc", N=30, n_steps=60, perturb=True), 16, 1)
        gen_case("nmpc3_fd_n20", dict(controller="nmpc", N=20, n_steps=30, ctrl_variant=0), 8, 0)
    finally:
        for libm in ("xlibm", "glibc"):
            O.ref(libm).nmpcmc_ref_set_ctrl_fd(0)


def gen_trace():
    """SqpReport::iterations and ::trace (SqpIterationLog, sqp.hpp:64-90) of
    the reference's sqp_solve on the OCP fixtures' instances (ocp_batch.npz),
    cold and warm."""
    d = np.load(os.path.join(OUT, "ocp_batch.npz"))
    out = {}
    for tag in ("one", "three"):
        kw = json.loads(str(d[f"{tag}__kwargs"]))
        sc = configs.make_scenario(**kw)
        x0, t0, xi0 = d[f"{tag}__x0"], d[f"{tag}__t0"], d[f"{tag}__xi0"]
        for start in ("cold", "warm"):
            r = O.solve_ocp_batch_traced(O.ref("xlibm"), sc, x0, t0, xi0=xi0 if start == "warm" else None,
                                         max_trace=24)
            for k, v in r.items():
                out[f"{tag}__{start}_{k}"] = v
            print(f"trace {tag} {start}: iterations mean {r['iterations'].mean():.1f}, records {r['trace_len'].sum()}, "
                  f"bfgs resets {int(r['trace']['bfgs_reset'].sum())}, exhausted {int(r['trace']['armijo_exhausted'].sum())}")
        out[f"{tag}__kwargs"] = np.array(json.dumps(kw))
    np.savez_compressed(os.path.join(OUT, "ocp_trace.npz"), **out)


def main(which):
    if which in ("rng", "all"):
        gen_rng()
    if which in ("pi", "all"):
        gen_case("pi_cfg0", dict(controller="pi"), 256, 4)
        gen_case("pi_cfg1", dict(controller="pi", perturb=True), 256, 2)
        gen_case("pi_onestate", dict(controller="pi", truth_variant=1), 64, 1)
        # noise-free, R = 0 edge case (measure is exact, model.cpp:41-45)
        gen_case("pi_quiet", dict(controller="pi", sigma_t=0.0, noise_R=0.0), 16, 1)
    if which in ("nmpc", "all"):
        # full-length BASELINE config 2 shape (N=60, max_iter=20)
        gen_case("nmpc_cfg2", dict(controller="nmpc", N=60), 16, 2)
        # shorter runs, more samples and horizons
        gen_case("nmpc_n30_short", dict(controller="nmpc", N=30, n_steps=120), 64, 2)
        gen_case("nmpc_n60_pert_short", dict(controller="nmpc", N=60, n_steps=120, perturb=True), 32, 1)
        gen_case("nmpc_n120_short", dict(controller="nmpc", N=120, n_steps=60), 16, 1)
    if which in ("qp", "all"):
        gen_qp()
    if which in ("ocp", "all"):
        gen_ocp()
    if which in ("full", "all"):
        gen_full()
    if which in ("dist", "all"):
        gen_dist()
    if which in ("steps", "all"):
        gen_steps()
    if which in ("qnlp", "all"):
        gen_qnlp()
    if which in ("fd", "all"):
        gen_fd()
    if which in ("trace", "all"):
        gen_trace()
    if which in ("nmpc3", "all"):
        # three-state controller model (config 2 read literally: CD-EKF and
        # OCP on the 3-state CSTR; ctrl_variant 0 = THREE_STATE) -> kernel K3g
        gen_case("nmpc3_cfg2", dict(controller="nmpc", N=60, ctrl_variant=0), 8, 1)
        gen_case("nmpc3_n30_short", dict(controller="nmpc", N=30, n_steps=120, ctrl_variant=0), 32, 1)
        gen_case("nmpc3_n60_pert_short", dict(controller="nmpc", N=60, n_steps=60, perturb=True, ctrl_variant=0),
                 16, 1)
        # one-state horizon beyond K3's shared-memory strides (N > 255) -> K3g
        gen_case("nmpc_n256_short", dict(controller="nmpc", N=256, n_steps=20), 8, 1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
