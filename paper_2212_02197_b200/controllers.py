"""Controller-level API on the GPU (controllers.hpp:16-93):

- pi_step_batch: pi_step (controllers.cpp:12-23) for n independent PI
  controllers; states advance to result.next in place
  (nmpcmc_gpu_pi_step_batch);
- NmpcBatch: B device-resident NmpcStates built like make_nmpc_state
  (controllers.cpp:25-48) from the scenario's controller configuration;
  step() is nmpc_step (controllers.cpp:114-212) on every instance, one warp
  per instance on K3w's code path (nmpcmc_gpu_nmpc_step_batch), bitwise the
  reference's inputs, diagnostics and state transitions.
"""
import ctypes as C

import numpy as np

from . import abi, engine


class PiState(C.Structure):
    """PiState (controllers.hpp:16-25)."""
    _fields_ = [(n, C.c_double) for n in ("kP", "kI", "kaw", "Ts", "u_bar", "u_min", "u_max", "I_hat")]


class PiStepResult(C.Structure):
    """PiStepResult (controllers.hpp:29-37); next_I_hat = result.next.I_hat."""
    _fields_ = [(n, C.c_double) for n in ("e", "P", "I", "u_hat", "u", "I_aw", "next_I_hat")]


class NmpcDiag(C.Structure):
    """NmpcDiagnostics (controllers.hpp:68-73) of one step."""
    _fields_ = [("x_filtered", C.c_double * 3), ("P_filtered", C.c_double * 9), ("innovation", C.c_double),
                ("converged", C.c_int32), ("sqp_iterations", C.c_int32), ("warm_started", C.c_int32),
                ("status", C.c_int32)]


PI_STATE_DTYPE = np.dtype([(n, "<f8") for n, _ in PiState._fields_])
PI_RESULT_DTYPE = np.dtype([(n, "<f8") for n, _ in PiStepResult._fields_])
DIAG_DTYPE = np.dtype([("x_filtered", "<f8", (3,)), ("P_filtered", "<f8", (9,)), ("innovation", "<f8"),
                       ("converged", "<i4"), ("sqp_iterations", "<i4"), ("warm_started", "<i4"), ("status", "<i4")])
assert PI_STATE_DTYPE.itemsize == C.sizeof(PiState)
assert PI_RESULT_DTYPE.itemsize == C.sizeof(PiStepResult)
assert DIAG_DTYPE.itemsize == C.sizeof(NmpcDiag)

_bound = False


def _lib():
    global _bound
    lib = engine.library()
    if not _bound:
        P = C.c_void_p
        lib.nmpcmc_gpu_pi_step_batch.argtypes = [P, P, P, P, C.c_int64, P]
        lib.nmpcmc_gpu_pi_step_device.argtypes = [P, P, P, P, C.c_int64, P]
        lib.nmpcmc_gpu_nmpc_batch_create.argtypes = [P, C.POINTER(abi.Scenario), C.c_int64, P, P, C.POINTER(P)]
        lib.nmpcmc_gpu_nmpc_batch_destroy.argtypes = [P]
        lib.nmpcmc_gpu_nmpc_batch_destroy.restype = None
        lib.nmpcmc_gpu_nmpc_step_batch.argtypes = [P, P, P, P, P, P, P]
        lib.nmpcmc_gpu_nmpc_batch_get.argtypes = [P, P, P, P, P, P, P, P]
        lib.nmpcmc_gpu_nmpc_batch_size.argtypes = [P]
        lib.nmpcmc_gpu_nmpc_batch_size.restype = C.c_int64
        _bound = True
    return lib


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape:
        raise abi_length_error(f"expected shape {shape}, got {a.shape}")
    return a


def abi_length_error(msg):
    return engine.LengthMismatch(msg)


def pi_step_batch(states: np.ndarray, y, y_bar, ctx=None):
    """pi_step for every controller: `states` (PI_STATE_DTYPE, n) advances in
    place; returns the PiStepResult records (PI_RESULT_DTYPE, n)."""
    if states.dtype != PI_STATE_DTYPE or not states.flags.c_contiguous:
        raise TypeError("states must be a contiguous PI_STATE_DTYPE array")
    n = states.shape[0]
    y = _f64(y, (n,))
    y_bar = _f64(y_bar, (n,))
    res = np.zeros(n, dtype=PI_RESULT_DTYPE)
    ctx = ctx or engine._context(0)
    ctx._check(_lib().nmpcmc_gpu_pi_step_batch(ctx.handle, states.ctypes.data, y.ctypes.data, y_bar.ctypes.data,
                                               C.c_int64(n), res.ctypes.data))
    return res


def make_pi_states(sc: abi.Scenario, n: int) -> np.ndarray:
    """n PiStates as run_closed_loop builds them (montecarlo.cpp:97-100)."""
    st = np.zeros(n, dtype=PI_STATE_DTYPE)
    st["kP"], st["kI"], st["kaw"] = sc.pi.kP, sc.pi.kI, sc.pi.kaw
    st["Ts"], st["u_bar"], st["u_min"], st["u_max"] = sc.Ts, sc.pi.u_bar, sc.u_min, sc.u_max
    st["I_hat"] = sc.pi.I_hat
    return st


class NmpcBatch:
    """B device-resident NmpcStates (make_nmpc_state per instance)."""

    def __init__(self, sc: abi.Scenario, batch: int, x0_hat=None, P0=None, ctx=None):
        self.ctx = ctx or engine._context(0)
        self.sc = sc
        self.batch = int(batch)
        self.nx = 3 if sc.ctrl_variant == abi.THREE_STATE else 1
        self.N = sc.N
        xh = None if x0_hat is None else _f64(x0_hat).reshape(self.batch, self.nx)
        p0 = None if P0 is None else _f64(P0).reshape(self.batch, self.nx * self.nx)
        self._keep = (xh, p0)
        h = C.c_void_p()
        self.ctx._check(_lib().nmpcmc_gpu_nmpc_batch_create(
            self.ctx.handle, C.byref(sc), C.c_int64(self.batch), None if xh is None else xh.ctypes.data,
            None if p0 is None else p0.ctypes.data, C.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            _lib().nmpcmc_gpu_nmpc_batch_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass

    def step(self, t, y, setpoints=None):
        """nmpc_step on every instance: (u[B], diagnostics[B] (DIAG_DTYPE))."""
        B = self.batch
        t = _f64(np.broadcast_to(np.asarray(t, dtype=np.float64), (B,)))
        y = _f64(y, (B,))
        sp = None if setpoints is None else _f64(setpoints, (B, self.N))
        u = np.zeros(B)
        diag = np.zeros(B, dtype=DIAG_DTYPE)
        self.ctx._check(_lib().nmpcmc_gpu_nmpc_step_batch(self.ctx.handle, self.handle, t.ctypes.data,
                                                          y.ctypes.data, None if sp is None else sp.ctypes.data,
                                                          u.ctypes.data, diag.ctypes.data))
        return u, diag

    def state(self) -> dict:
        """The NmpcStates: x_hat, P (column-major), last_xi, last_lambda,
        last_pi_l, last_pi_u, warm."""
        B, nx, N = self.batch, self.nx, self.N
        out = dict(x_hat=np.zeros((B, nx)), P=np.zeros((B, nx * nx)), last_xi=np.zeros((B, N * (1 + nx))),
                   last_lambda=np.zeros((B, N * nx)), last_pi_l=np.zeros((B, N)), last_pi_u=np.zeros((B, N)),
                   warm=np.zeros(B, dtype=np.int32))
        self.ctx._check(_lib().nmpcmc_gpu_nmpc_batch_get(self.handle, *(out[k].ctypes.data for k in (
            "x_hat", "P", "last_xi", "last_lambda", "last_pi_l", "last_pi_u", "warm"))))
        return out
