"""Batched standalone QP and OCP services:
- solve_qp_batch: the reference's solve_qp / riccati_factor_solve
  (qp.hpp:24-56) for a batch of independent QPs of equal dimensions, on the
  GPU kernel K5 (csrc/qp_batch_kernel.cuh), nmpcmc_gpu_solve_qp_batch;
- solve_ocp_batch: the reference's sqp_solve on the regulator OcpProblem
  (sqp.hpp:27-50, :148-151) for a batch of initial states, one warp per
  instance (K3w's code path), nmpcmc_gpu_solve_ocp_batch.

A QP is a list of N+1 stage dicts with the members of QpStageData
(qp.hpp:24-30): Q, M, R, q, r, Jx, Ju, b, lb, ub (numpy arrays; M is n_x x
n_u as in the reference). Stage 0 needs R r Ju b lb ub; stages 1..N-1 all
members; stage N only Q q.
"""
import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import abi, engine

OPTIMAL, MAXITER, FAILED, DOMAIN_ERROR, NOT_POSITIVE_DEFINITE = range(5)
STATUS_NAMES = {OPTIMAL: "Optimal", MAXITER: "MaxIter", FAILED: "Failed", DOMAIN_ERROR: "DomainError",
                NOT_POSITIVE_DEFINITE: "NotPositiveDefinite"}


class QpDims(C.Structure):
    _fields_ = [("N", C.c_int32), ("n_x", C.c_int32), ("n_u", C.c_int32), ("max_iter", C.c_int32),
                ("tol", C.c_double), ("mode", C.c_int32), ("_pad", C.c_int32)]


def stage_doubles(nx: int, nu: int) -> int:
    return 2 * nx * nx + 2 * nx * nu + nu * nu + 2 * nx + 3 * nu


def solution_doubles(N: int, nx: int, nu: int) -> int:
    return N * (nu + nx) + N * nx + 2 * N * nu


def pack(qps, nx: int, nu: int) -> np.ndarray:
    """Packed input (batch, N+1, stage_doubles) from a list of QPs."""
    N = len(qps[0]) - 1
    out = np.zeros((len(qps), N + 1, stage_doubles(nx, nu)))
    z = {"Q": (nx, nx), "M": (nx, nu), "R": (nu, nu), "q": (nx,), "r": (nu,), "Jx": (nx, nx), "Ju": (nx, nu),
         "b": (nx,), "lb": (nu,), "ub": (nu,)}
    for bi, qp in enumerate(qps):
        if len(qp) != N + 1:
            raise ValueError("all QPs of a batch need the same number of stages")
        for k, st in enumerate(qp):
            parts = []
            for name in ("Q", "M", "R", "q", "r", "Jx", "Ju", "b", "lb", "ub"):
                v = st.get(name)
                a = np.zeros(z[name]) if v is None else np.asarray(v, dtype=np.float64).reshape(z[name])
                parts.append(a.reshape(-1, order="F"))
            out[bi, k] = np.concatenate(parts)
    return out


@dataclass
class QpSolution:
    """QpSolution (qp.hpp:34-41) of one QP of a batch."""
    delta_xi: np.ndarray
    mu: np.ndarray
    nu_l: np.ndarray
    nu_u: np.ndarray
    iterations: int
    status: int


def unpack(sol: np.ndarray, status, iterations, N: int, nx: int, nu: int):
    L, NX, NV = N * (nu + nx), N * nx, N * nu
    return [QpSolution(s[:L].copy(), s[L:L + NX].copy(), s[L + NX:L + NX + NV].copy(), s[L + NX + NV:].copy(),
                       int(it), int(st)) for s, st, it in zip(sol, status, iterations)]


def solve_qp_batch(qps_or_packed, nx: int = None, nu: int = None, tol: float = 1e-10, max_iter: int = 50,
                   riccati_only: bool = False, ctx=None, raw: bool = False):
    """solve_qp(stages, tol, max_iter) for every QP of the batch (or
    riccati_factor_solve with riccati_only). Input: a list of QPs (stage-dict
    lists) or a packed (batch, N+1, stage_doubles) array with nx, nu given.
    Returns a list of QpSolution, or (solutions, status, iterations) arrays
    with raw=True."""
    if isinstance(qps_or_packed, np.ndarray):
        packed = np.ascontiguousarray(qps_or_packed, dtype=np.float64)
        if nx is None or nu is None:
            raise ValueError("packed input needs nx, nu")
        if packed.ndim != 3 or packed.shape[2] != stage_doubles(nx, nu) or packed.shape[1] < 2:
            raise engine.DimensionMismatch(
                f"packed QP batch must have shape (batch, N+1 >= 2, {stage_doubles(nx, nu)}), got {packed.shape}")
    else:
        qps = qps_or_packed
        if nu is None:
            nu = np.atleast_2d(np.asarray(qps[0][0]["R"], dtype=np.float64)).shape[0]
        if nx is None:
            nx = np.atleast_2d(np.asarray(qps[0][-1]["Q"], dtype=np.float64)).shape[0]
        packed = pack(qps, nx, nu)
    batch, N = packed.shape[0], packed.shape[1] - 1
    d = QpDims(N, nx, nu, max_iter, tol, 1 if riccati_only else 0, 0)
    sol = np.zeros((batch, solution_doubles(N, nx, nu)))
    st = np.zeros(batch, dtype=np.int32)
    it = np.zeros(batch, dtype=np.int32)
    ctx = ctx or engine._context(0)
    ctx._check(ctx.lib.nmpcmc_gpu_solve_qp_batch(
        ctx.handle, C.byref(d), batch, packed.ctypes.data_as(C.POINTER(C.c_double)),
        sol.ctypes.data_as(C.POINTER(C.c_double)), st.ctypes.data_as(C.POINTER(C.c_int32)),
        it.ctypes.data_as(C.POINTER(C.c_int32))))
    if raw:
        return sol, st, it
    return unpack(sol, st, it, N, nx, nu)


# ---------------------------------------------------------- instance builders
def random_instance(rng: np.random.Generator, N: int, nx: int, nu: int, bounded: bool = True,
                    inf_frac: float = 0.15):
    """A random convex stagewise QP: PD joint (x, u) Hessian blocks, near-
    identity dynamics, tight-ish input boxes (some sides infinite) so bounds
    are active in a good share of instances."""
    qp = []
    for k in range(N + 1):
        st = {}
        if k < N:
            A = rng.uniform(-1, 1, (nx + nu, nx + nu))
            W = A @ A.T + 0.5 * np.eye(nx + nu)
            st["R"] = W[nx:, nx:]
            st["r"] = rng.uniform(-1, 1, nu)
            st["Ju"] = rng.uniform(-1, 1, (nx, nu))
            st["b"] = 0.2 * rng.uniform(-1, 1, nx)
            if bounded:
                lb = -rng.uniform(0.05, 0.6, nu)
                ub = rng.uniform(0.05, 0.6, nu)
                lb[rng.uniform(size=nu) < inf_frac] = -np.inf
                ub[rng.uniform(size=nu) < inf_frac] = np.inf
            else:
                lb, ub = np.full(nu, -np.inf), np.full(nu, np.inf)
            st["lb"], st["ub"] = lb, ub
            if k >= 1:
                st["Q"], st["M"] = W[:nx, :nx], W[:nx, nx:]
                st["q"] = rng.uniform(-1, 1, nx)
                st["Jx"] = np.eye(nx) + 0.3 * rng.uniform(-1, 1, (nx, nx))
        else:
            A = rng.uniform(-1, 1, (nx, nx))
            st["Q"] = A @ A.T + 0.5 * np.eye(nx)
            st["q"] = rng.uniform(-1, 1, nx)
        qp.append(st)
    return qp


def scalar_instance(r_hess, r_lin, p_term, p_lin, ju, b0, lb, ub):
    """One input, one terminal state: min 1/2 R u^2 + r u + 1/2 P x1^2 + p x1,
    x1 = ju u + b0, lb <= u <= ub."""
    return [{"R": [[r_hess]], "r": [r_lin], "Ju": [[ju]], "b": [b0], "lb": [lb], "ub": [ub]},
            {"Q": [[p_term]], "q": [p_lin]}]


def double_integrator(rng: np.random.Generator, N: int, h: float):
    """Discrete double integrator (x = position, velocity; u = acceleration)
    with random linear terms and offsets, unconstrained."""
    Jx = np.array([[1.0, h], [0.0, 1.0]])
    Ju = np.array([[0.5 * h * h], [h]])
    qp = []
    for k in range(N):
        st = {"R": [[0.1]], "r": [rng.uniform(-1, 1)], "Jx": Jx, "Ju": Ju, "b": 0.2 * rng.uniform(-1, 1, 2),
              "lb": [-np.inf], "ub": [np.inf]}
        if k >= 1:
            st.update(Q=np.diag([1.0, 0.1]), M=np.zeros((2, 1)), q=rng.uniform(-1, 1, 2))
        qp.append(st)
    qp.append({"Q": np.diag([5.0, 1.0]), "q": rng.uniform(-1, 1, 2)})
    return qp


# ----------------------------------------------------------- OCP service
def solve_ocp_batch(sc, x0, t0, xi0=None, ctx=None):
    """sqp_solve on the CSTR regulator OCP of scenario sc (its controller
    model, horizon, Qz, bounds, setpoints and SqpOptions) for each initial
    state x0[b] (shape (B, nx)) at time t0[b]; cold start as nmpc_step unless
    xi0 (B, L) is given. Returns a dict of numpy arrays: xi (B, L), lambda
    (B, N nx), pi_l, pi_u (B, N), converged, status (B,)."""
    # the controller model fixes the state width (the C ABI reads nx from
    # sc.ctrl_variant and copies B*nx / B*L doubles): check every buffer
    # against it before anything crosses the boundary (nmpcmc_gpu.hpp)
    nx, N = (3 if sc.ctrl_variant == abi.THREE_STATE else 1), sc.N
    L = N * (1 + nx)
    x0 = np.asarray(x0, dtype=np.float64)
    if x0.ndim == 1 and nx == 1:
        x0 = x0.reshape(-1, 1)
    if x0.ndim != 2 or x0.shape[1] != nx:
        raise engine.LengthMismatch(f"solve_ocp_batch: x0 must have shape (B, {nx}), got {x0.shape}")
    x0 = np.ascontiguousarray(x0)
    B = x0.shape[0]
    t0 = np.ascontiguousarray(t0, dtype=np.float64).reshape(-1)
    if t0.size != B:
        raise engine.LengthMismatch(f"solve_ocp_batch: t0 needs {B} entries, got {t0.size}")
    out = dict(xi=np.zeros((B, L)), **{"lambda": np.zeros((B, N * nx))}, pi_l=np.zeros((B, N)),
               pi_u=np.zeros((B, N)), converged=np.zeros(B, dtype=np.int32), status=np.zeros(B, dtype=np.int32))
    xi0p = None
    if xi0 is not None:
        xi0 = np.ascontiguousarray(xi0, dtype=np.float64)
        if xi0.shape != (B, L):
            raise engine.LengthMismatch(f"solve_ocp_batch: xi0 must have shape ({B}, {L}), got {xi0.shape}")
        xi0p = xi0.ctypes.data_as(C.POINTER(C.c_double))
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    ctx = ctx or engine._context(0)
    ctx._check(ctx.lib.nmpcmc_gpu_solve_ocp_batch(
        ctx.handle, C.byref(sc), B, P(x0), P(t0), xi0p, P(out["xi"]), P(out["lambda"]), P(out["pi_l"]),
        P(out["pi_u"]), out["converged"].ctypes.data_as(C.POINTER(C.c_int32)),
        out["status"].ctypes.data_as(C.POINTER(C.c_int32))))
    return out



# ------------------------------------------------------ SQP on quadratic NLPs
class QnlpDims(C.Structure):
    _fields_ = [("N", C.c_int32), ("n_x", C.c_int32), ("n_u", C.c_int32), ("_pad", C.c_int32),
                ("sqp", abi.SqpOptions)]


def qnlp_doubles(N: int, nx: int) -> int:
    """Packed doubles of one quadratic NLP (nmpcmc_qnlp_doubles)."""
    return nx + 2 + N * (2 + 2 * nx * nx + 3 * nx)


def pack_qnlp(x0, u_min, u_max, R, r, Q, q, A, B, c) -> np.ndarray:
    """One quadratic NLP in the packed layout: x0 (nx,), bounds, and per
    stage k R[k], r[k], Q[k] (nx, nx), q[k] (nx,), A[k] (nx, nx), B[k] (nx,),
    c[k] (nx,) -- matrices stored column-major."""
    x0 = np.atleast_1d(np.asarray(x0, dtype=np.float64))
    N = len(R)
    parts = [x0, [u_min, u_max]]
    for k in range(N):
        parts += [[R[k], r[k]], np.asarray(Q[k], dtype=np.float64).reshape(-1, order="F"), np.ravel(q[k]),
                  np.asarray(A[k], dtype=np.float64).reshape(-1, order="F"), np.ravel(B[k]), np.ravel(c[k])]
    out = np.concatenate([np.asarray(p, dtype=np.float64).ravel() for p in parts])
    assert out.size == qnlp_doubles(N, x0.size)
    return out


def default_sqp_options(**kw) -> abi.SqpOptions:
    """SqpOptions defaults (sqp.hpp:50-58)."""
    o = abi.SqpOptions()
    o.eps, o.max_iter, o.max_backtracks, o.c1, o.backtrack_factor = 1e-6, 100, 30, 1e-4, 0.5
    o.qp_tol, o.qp_max_iter = 1e-12, 50
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def solve_qnlp_batch(problems, N: int, nx: int, opts: abi.SqpOptions = None, xi0=None, ctx=None) -> dict:
    """sqp_solve (sqp.cpp:182-411) on a batch of stagewise quadratic NLPs
    through the SqpProblem interface (nmpcmc_gpu_sqp_solve_qnlp_batch);
    problems: (batch, qnlp_doubles(N, nx)). Returns xi, lambda, pi_l, pi_u,
    converged, iterations, status."""
    problems = np.ascontiguousarray(problems, dtype=np.float64)
    if problems.ndim != 2 or problems.shape[1] != qnlp_doubles(N, nx):
        raise engine.DimensionMismatch(f"problems must be (batch, {qnlp_doubles(N, nx)})")
    Bn, L = problems.shape[0], N * (1 + nx)
    if xi0 is not None:
        xi0 = np.ascontiguousarray(xi0, dtype=np.float64)
        if xi0.shape != (Bn, L):
            raise engine.LengthMismatch(f"xi0 must be ({Bn}, {L})")
    d = QnlpDims(N, nx, 1, 0, opts or default_sqp_options())
    out = dict(xi=np.zeros((Bn, L)), **{"lambda": np.zeros((Bn, N * nx))}, pi_l=np.zeros((Bn, N)),
               pi_u=np.zeros((Bn, N)), converged=np.zeros(Bn, dtype=np.int32), iterations=np.zeros(Bn, dtype=np.int32),
               status=np.zeros(Bn, dtype=np.int32))
    ctx = ctx or engine._context(0)
    lib = ctx.lib
    lib.nmpcmc_gpu_sqp_solve_qnlp_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64] + [C.c_void_p] * 9
    ctx._check(lib.nmpcmc_gpu_sqp_solve_qnlp_batch(
        ctx.handle, C.byref(d), C.c_int64(Bn), problems.ctypes.data, None if xi0 is None else xi0.ctypes.data,
        *(out[k].ctypes.data for k in ("xi", "lambda", "pi_l", "pi_u", "converged", "iterations", "status"))))
    return out



# ------------------------------------------------ SQP trace (SqpIterationLog)
SQP_LOG_DTYPE = np.dtype([("alpha", "<f8"), ("merit_before", "<f8"), ("merit_after", "<f8"),
                          ("directional_derivative", "<f8"), ("grad_l_inf", "<f8"), ("g_inf", "<f8"),
                          ("step_inf", "<f8"), ("ls_evals", "<i4"), ("qp_iterations", "<i4"), ("qp_status", "<i4"),
                          ("armijo_exhausted", "<i4"), ("bfgs_reset", "<i4"), ("_pad", "<i4")])
assert SQP_LOG_DTYPE.itemsize == 80


def solve_ocp_batch_traced(sc, x0, t0, xi0=None, max_trace=32, ctx=None) -> dict:
    """solve_ocp_batch plus SqpReport::iterations and the per-iteration
    SqpIterationLog trace (sqp.hpp:64-90): trace (B, max_trace) records of
    SQP_LOG_DTYPE, trace_len (B,) (nmpcmc_gpu_solve_ocp_batch_traced)."""
    nx, N = (3 if sc.ctrl_variant == abi.THREE_STATE else 1), sc.N
    L = N * (1 + nx)
    x0 = np.asarray(x0, dtype=np.float64)
    if x0.ndim == 1 and nx == 1:
        x0 = x0.reshape(-1, 1)
    if x0.ndim != 2 or x0.shape[1] != nx:
        raise engine.LengthMismatch(f"solve_ocp_batch_traced: x0 must have shape (B, {nx}), got {x0.shape}")
    x0 = np.ascontiguousarray(x0)
    B = x0.shape[0]
    t0 = np.ascontiguousarray(t0, dtype=np.float64).reshape(-1)
    if t0.size != B:
        raise engine.LengthMismatch(f"solve_ocp_batch_traced: t0 needs {B} entries, got {t0.size}")
    if xi0 is not None:
        xi0 = np.ascontiguousarray(xi0, dtype=np.float64)
        if xi0.shape != (B, L):
            raise engine.LengthMismatch(f"solve_ocp_batch_traced: xi0 must have shape ({B}, {L})")
    out = dict(xi=np.zeros((B, L)), **{"lambda": np.zeros((B, N * nx))}, pi_l=np.zeros((B, N)),
               pi_u=np.zeros((B, N)), converged=np.zeros(B, dtype=np.int32), status=np.zeros(B, dtype=np.int32),
               iterations=np.zeros(B, dtype=np.int32), trace=np.zeros((B, max_trace), dtype=SQP_LOG_DTYPE),
               trace_len=np.zeros(B, dtype=np.int32))
    ctx = ctx or engine._context(0)
    lib = ctx.lib
    lib.nmpcmc_gpu_solve_ocp_batch_traced.argtypes = ([C.c_void_p, C.POINTER(abi.Scenario), C.c_int64] +
                                                       [C.c_void_p] * 10 + [C.c_int32, C.c_void_p, C.c_void_p])
    ctx._check(lib.nmpcmc_gpu_solve_ocp_batch_traced(
        ctx.handle, C.byref(sc), C.c_int64(B), x0.ctypes.data, t0.ctypes.data,
        None if xi0 is None else xi0.ctypes.data,
        *(out[k].ctypes.data for k in ("xi", "lambda", "pi_l", "pi_u", "converged", "status", "iterations")),
        int(max_trace), out["trace"].ctypes.data, out["trace_len"].ctypes.data))
    return out
