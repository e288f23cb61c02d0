"""ctypes mirror of include/nmpcmc_gpu.h (the C ABI), plus numpy record dtypes.

Layouts are checked at load time against nmpcmc_gpu_struct_size() so a
header change that is not mirrored here fails loudly.
"""
import ctypes as C

import numpy as np

MAX_SETPOINTS = 32

CTRL_NMPC, CTRL_PI = 0, 1  # montecarlo.hpp:22
THREE_STATE, ONE_STATE = 0, 1  # cstr.hpp:19

STATUS_NAMES = {
    0: "OK",
    1: "DimensionMismatch",
    2: "NotPositiveDefinite",
    3: "NonFiniteState",
    4: "DomainError",
    5: "LengthMismatch",
    6: "Unsupported",
    7: "InvalidArgument",
    100: "CudaError",
    101: "NoDevice",
}


class CstrParams(C.Structure):
    """CstrParams (cstr.hpp:21-34)."""

    _fields_ = [(n, C.c_double) for n in
                ("V", "k0", "EaR", "beta", "cA_in", "cB_in", "cT_in",
                 "sigmaA", "sigmaB", "sigmaT", "u_min", "u_max")]


class SqpOptions(C.Structure):
    """SqpOptions (sqp.hpp:50-58)."""

    _fields_ = [
        ("eps", C.c_double),
        ("c1", C.c_double),
        ("backtrack_factor", C.c_double),
        ("qp_tol", C.c_double),
        ("max_iter", C.c_int32),
        ("max_backtracks", C.c_int32),
        ("qp_max_iter", C.c_int32),
        ("_pad", C.c_int32),
    ]


class PiGains(C.Structure):
    """PiState gains (controllers.hpp:16-25)."""

    _fields_ = [(n, C.c_double) for n in ("kP", "kI", "kaw", "u_bar", "I_hat")]


class Scenario(C.Structure):
    """Scenario (montecarlo.hpp:27-55) for the CSTR case study."""

    _fields_ = [
        ("controller", C.c_int32),
        ("truth_variant", C.c_int32),
        ("ctrl_variant", C.c_int32),
        ("has_noise_R", C.c_int32),
        ("truth", CstrParams),
        ("ctrl", CstrParams),
        ("noise_R", C.c_double),
        ("R_filter", C.c_double),
        ("Qz", C.c_double),
        ("horizon_Ts", C.c_double),
        ("N", C.c_int32),
        ("Nc", C.c_int32),
        ("np", C.c_int32),
        ("Ns", C.c_int32),
        ("sqp", SqpOptions),
        ("pi", PiGains),
        ("u_min", C.c_double),
        ("u_max", C.c_double),
        ("t0", C.c_double),
        ("tf", C.c_double),
        ("Ts", C.c_double),
        ("n_setpoints", C.c_int32),
        ("record_stride", C.c_int32),
        ("sp_times", C.c_double * MAX_SETPOINTS),
        ("sp_values", C.c_double * MAX_SETPOINTS),
        ("x0", C.c_double * 3),
        ("x0_hat", C.c_double * 3),
        ("P0", C.c_double * 9),
        ("base_seed", C.c_uint64),
        ("perturb", C.c_int32),
        ("record_trajectories", C.c_int32),
        ("perturb_rel_std", C.c_double * 3),
    ]


class SimRecord(C.Structure):
    _fields_ = [
        ("phi", C.c_double),
        ("failed", C.c_int32),
        ("ocp_solves", C.c_int32),
        ("ocp_failures", C.c_int32),
        ("status", C.c_int32),
    ]


class WorkCounters(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "control_steps", "shoot_full", "shoot_fonly", "ipm_stage_iters",
        "sqp_stage_iters", "qp_solves", "sqp_iterations", "ls_evals")]


class Aggregate(C.Structure):
    """McAggregate (montecarlo.hpp:95-106)."""

    _fields_ = [
        ("n_sims", C.c_int32),
        ("n_failed", C.c_int32),
        ("mean", C.c_double),
        ("variance", C.c_double),
        ("min", C.c_double),
        ("max", C.c_double),
        ("deciles", C.c_double * 11),
        ("ocp_solves", C.c_int64),
        ("ocp_failures", C.c_int64),
        ("ocp_success_pct", C.c_double),
    ]


RECORD_DTYPE = np.dtype([("phi", "<f8"), ("failed", "<i4"), ("ocp_solves", "<i4"),
                         ("ocp_failures", "<i4"), ("status", "<i4")])
COUNTERS_DTYPE = np.dtype([(n, "<i8") for n, _ in WorkCounters._fields_])
assert RECORD_DTYPE.itemsize == C.sizeof(SimRecord) == 24
assert COUNTERS_DTYPE.itemsize == C.sizeof(WorkCounters)

STRUCT_SIZES = {0: Scenario, 1: SimRecord, 2: WorkCounters, 3: Aggregate}


def check_layout(lib) -> None:
    """Compare this mirror with the compiled library's sizeof()s."""
    lib.nmpcmc_gpu_struct_size.restype = C.c_int64
    lib.nmpcmc_gpu_struct_size.argtypes = [C.c_int]
    for which, cls in STRUCT_SIZES.items():
        got = lib.nmpcmc_gpu_struct_size(which)
        if got != C.sizeof(cls):
            raise RuntimeError(f"ABI mismatch for {cls.__name__}: C {got} vs ctypes {C.sizeof(cls)}")


def aggregate_to_dict(a: Aggregate) -> dict:
    return {
        "n_sims": a.n_sims, "n_failed": a.n_failed, "mean": a.mean, "variance": a.variance,
        "min": a.min, "max": a.max, "deciles": list(a.deciles), "ocp_solves": a.ocp_solves,
        "ocp_failures": a.ocp_failures, "ocp_success_pct": a.ocp_success_pct,
    }
