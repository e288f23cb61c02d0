"""ctypes loaders for the oracle libraries (TEST INFRASTRUCTURE ONLY).

  ref(libm="xlibm"|"glibc") -> the unmodified reference core + ref_driver.cpp
                               (oracle/_ref/, built from /root/reference)
  port()                    -> the C++ restatement (oracle/port/, _build/)
  xlibm()                   -> host build of the portable libm
"""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2212_02197_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
_cache = {}


def build(target="all") -> None:
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def _load(path):
    if path not in _cache:
        _cache[path] = C.CDLL(path)
    return _cache[path]


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libnmpcmc_ref_xlibm.so"))


def ref(libm="xlibm"):
    path = os.path.join(HERE, "_ref", f"libnmpcmc_ref_{libm}.so")
    if not os.path.exists(path):
        if os.path.isdir("/root/reference/proj/core"):
            build("ref")
        else:
            raise FileNotFoundError(f"{path} missing and /root/reference absent (build it in the dev container)")
    lib = _load(path)
    _sig(lib, "nmpcmc_ref")
    return lib


def port(libm="xlibm"):
    """The C++ restatement (oracle/port/nmpcmc_port.cpp); symbol prefix
    nmpcmc_portx_ (exact-libm build) or nmpcmc_port_ (glibc build)."""
    path = os.path.join(HERE, "_build", f"libnmpcmc_port_{libm}.so")
    if not os.path.exists(path):
        build("port")
    lib = _load(path)
    _sig(lib, port_prefix(libm))
    return lib


def port_prefix(libm="xlibm"):
    return "nmpcmc_portx" if libm == "xlibm" else "nmpcmc_port"


def xlibm():
    path = os.path.join(HERE, "_build", "libxlibm.so")
    if not os.path.exists(path):
        build("_build/libxlibm.so")
    lib = _load(path)
    for n in ("nmx_exp", "nmx_log", "nmx_sin", "nmx_cos"):
        getattr(lib, n).restype = C.c_double
        getattr(lib, n).argtypes = [C.c_double]
    return lib


def _sig(lib, p):
    S = C.POINTER(abi.Scenario)
    R = C.POINTER(abi.SimRecord)
    f = getattr(lib, f"{p}_run_closed_loop")
    f.argtypes = [S, C.c_uint64, R, C.POINTER(C.c_double), C.c_int]
    f = getattr(lib, f"{p}_run_batch")
    f.argtypes = [S, C.c_uint64, C.c_int64, C.c_int, R, C.POINTER(C.c_double)]
    if hasattr(lib, f"{p}_aggregate"):
        getattr(lib, f"{p}_aggregate").argtypes = [R, C.c_int64, C.POINTER(abi.Aggregate)]
    if hasattr(lib, f"{p}_normals"):
        getattr(lib, f"{p}_normals").argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.POINTER(C.c_double)]
    if hasattr(lib, f"{p}_reaction_rate"):
        getattr(lib, f"{p}_reaction_rate").restype = C.c_double
        getattr(lib, f"{p}_reaction_rate").argtypes = [C.POINTER(abi.CstrParams), C.POINTER(C.c_double)]


def run_batch(lib, sc, first, n, workers=None, prefix="nmpcmc_ref"):
    """Records (numpy RECORD_DTYPE) and wall seconds for [first, first+n)."""
    workers = workers or os.cpu_count() or 1
    out = np.zeros(n, dtype=abi.RECORD_DTYPE)
    wall = C.c_double(0.0)
    rc = getattr(lib, f"{prefix}_run_batch")(C.byref(sc), first, n, workers,
                                             out.ctypes.data_as(C.POINTER(abi.SimRecord)), C.byref(wall))
    if rc != 0:
        raise RuntimeError(f"oracle run_batch failed: {rc}")
    return out, wall.value


def run_traj(lib, sc, idx, rows, prefix="nmpcmc_ref"):
    rec = abi.SimRecord()
    traj = np.zeros((rows, 5))
    getattr(lib, f"{prefix}_run_closed_loop")(C.byref(sc), idx, C.byref(rec),
                                              traj.ctypes.data_as(C.POINTER(C.c_double)), rows)
    return rec, traj


def solve_qp_batch(lib, packed, nx, nu, tol=1e-10, max_iter=50, riccati_only=False):
    """The reference's solve_qp / riccati_factor_solve over a packed batch
    (layout of nmpcmc_gpu_solve_qp_batch): (solutions, status, iterations)."""
    from paper_2212_02197_b200 import qp as Q
    packed = np.ascontiguousarray(packed, dtype=np.float64)
    batch, N = packed.shape[0], packed.shape[1] - 1
    d = Q.QpDims(N, nx, nu, max_iter, tol, 1 if riccati_only else 0, 0)
    sol = np.zeros((batch, Q.solution_doubles(N, nx, nu)))
    st = np.zeros(batch, dtype=np.int32)
    it = np.zeros(batch, dtype=np.int32)
    lib.nmpcmc_ref_solve_qp_batch(C.byref(d), C.c_int64(batch), packed.ctypes.data_as(C.POINTER(C.c_double)),
                                  sol.ctypes.data_as(C.POINTER(C.c_double)),
                                  st.ctypes.data_as(C.POINTER(C.c_int32)),
                                  it.ctypes.data_as(C.POINTER(C.c_int32)))
    return sol, st, it


def solve_ocp_batch(lib, sc, x0, t0, xi0=None):
    """The reference's sqp_solve on the regulator OcpProblem per instance
    (layout of nmpcmc_gpu_solve_ocp_batch): dict of arrays."""
    x0 = np.ascontiguousarray(np.atleast_2d(x0), dtype=np.float64)
    t0 = np.ascontiguousarray(t0, dtype=np.float64).reshape(-1)
    B, nx, N = x0.shape[0], x0.shape[1], sc.N
    L = N * (1 + nx)
    out = dict(xi=np.zeros((B, L)), **{"lambda": np.zeros((B, N * nx))}, pi_l=np.zeros((B, N)),
               pi_u=np.zeros((B, N)), converged=np.zeros(B, dtype=np.int32), status=np.zeros(B, dtype=np.int32))
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    xi0p = None if xi0 is None else P(np.ascontiguousarray(xi0, dtype=np.float64))
    lib.nmpcmc_ref_solve_ocp_batch(C.byref(sc), C.c_int64(B), P(x0), P(t0), xi0p, P(out["xi"]), P(out["lambda"]),
                                   P(out["pi_l"]), P(out["pi_u"]),
                                   out["converged"].ctypes.data_as(C.POINTER(C.c_int32)),
                                   out["status"].ctypes.data_as(C.POINTER(C.c_int32)))
    return out



def nmpc_steps(lib, sc, x0_hat, P0, t, y, sp=None):
    """The reference's make_nmpc_state + nmpc_step over T steps for B
    controllers (nmpcmc_ref_nmpc_steps): u (B, T), diag (B, T) records in the
    layout of nmpcmc_nmpc_diag, and the final NmpcStates."""
    from paper_2212_02197_b200 import controllers as K
    t = np.ascontiguousarray(t, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    B, T = y.shape
    nx = 3 if sc.ctrl_variant == abi.THREE_STATE else 1
    N = sc.N
    L = N * (1 + nx)
    u = np.zeros((B, T))
    diag = np.zeros((B, T), dtype=K.DIAG_DTYPE)
    fin = dict(x_hat=np.zeros((B, nx)), P=np.zeros((B, nx * nx)), last_xi=np.zeros((B, L)),
               last_lambda=np.zeros((B, N * nx)), last_pi_l=np.zeros((B, N)), last_pi_u=np.zeros((B, N)),
               warm=np.zeros(B, dtype=np.int32))
    V = C.c_void_p
    f = lib.nmpcmc_ref_nmpc_steps
    f.argtypes = [C.POINTER(abi.Scenario), C.c_int64, C.c_int] + [V] * 14
    keep = [None if x0_hat is None else np.ascontiguousarray(x0_hat, dtype=np.float64),
            None if P0 is None else np.ascontiguousarray(P0, dtype=np.float64),
            None if sp is None else np.ascontiguousarray(sp, dtype=np.float64)]
    f(C.byref(sc), B, T, None if keep[0] is None else keep[0].ctypes.data,
      None if keep[1] is None else keep[1].ctypes.data, t.ctypes.data, y.ctypes.data,
      None if keep[2] is None else keep[2].ctypes.data, u.ctypes.data, diag.ctypes.data,
      *(fin[k].ctypes.data for k in ("x_hat", "P", "last_xi", "last_lambda", "last_pi_l", "last_pi_u", "warm")))
    return u, diag, fin


def sqp_solve_qnlp_batch(lib, problems, N, nx, opts, xi0=None):
    """The reference's sqp_solve on QnlpProblems (nmpcmc_ref_sqp_solve_qnlp_batch)."""
    from paper_2212_02197_b200 import qp as Q
    problems = np.ascontiguousarray(problems, dtype=np.float64)
    Bn, L = problems.shape[0], N * (1 + nx)
    d = Q.QnlpDims(N, nx, 1, 0, opts)
    out = dict(xi=np.zeros((Bn, L)), **{"lambda": np.zeros((Bn, N * nx))}, pi_l=np.zeros((Bn, N)),
               pi_u=np.zeros((Bn, N)), converged=np.zeros(Bn, dtype=np.int32), iterations=np.zeros(Bn, dtype=np.int32),
               status=np.zeros(Bn, dtype=np.int32))
    x0p = None if xi0 is None else np.ascontiguousarray(xi0, dtype=np.float64)
    f = lib.nmpcmc_ref_sqp_solve_qnlp_batch
    f.argtypes = [C.c_void_p, C.c_int64] + [C.c_void_p] * 9
    f(C.byref(d), Bn, problems.ctypes.data, None if x0p is None else x0p.ctypes.data,
      *(out[k].ctypes.data for k in ("xi", "lambda", "pi_l", "pi_u", "converged", "iterations", "status")))
    return out


def solve_ocp_batch_traced(lib, sc, x0, t0, xi0=None, max_trace=32):
    """The reference's sqp_solve on the regulator OcpProblem with
    SqpReport::iterations and ::trace (nmpcmc_ref_solve_ocp_batch_traced)."""
    from paper_2212_02197_b200 import qp as Q
    x0 = np.ascontiguousarray(np.atleast_2d(x0), dtype=np.float64)
    t0 = np.ascontiguousarray(t0, dtype=np.float64).reshape(-1)
    B, nx, N = x0.shape[0], x0.shape[1], sc.N
    L = N * (1 + nx)
    out = dict(xi=np.zeros((B, L)), **{"lambda": np.zeros((B, N * nx))}, pi_l=np.zeros((B, N)),
               pi_u=np.zeros((B, N)), converged=np.zeros(B, dtype=np.int32), status=np.zeros(B, dtype=np.int32),
               iterations=np.zeros(B, dtype=np.int32), trace=np.zeros((B, max_trace), dtype=Q.SQP_LOG_DTYPE),
               trace_len=np.zeros(B, dtype=np.int32))
    x0p = None if xi0 is None else np.ascontiguousarray(xi0, dtype=np.float64)
    f = lib.nmpcmc_ref_solve_ocp_batch_traced
    f.argtypes = [C.POINTER(abi.Scenario), C.c_int64] + [C.c_void_p] * 10 + [C.c_int32, C.c_void_p, C.c_void_p]
    f(C.byref(sc), B, x0.ctypes.data, t0.ctypes.data, None if x0p is None else x0p.ctypes.data,
      *(out[k].ctypes.data for k in ("xi", "lambda", "pi_l", "pi_u", "converged", "status", "iterations")),
      max_trace, out["trace"].ctypes.data, out["trace_len"].ctypes.data)
    return out
