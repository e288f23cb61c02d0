"""Algorithmic FP64 work per unit, for the roofline (SURVEY.md §8d convention).

Convention: +, -, *, /, sqrt = 1 flop each; transcendental weights
exp = log = 20, sincos = 40; Philox integer work not counted. The kernels
compile with --fmad=false (bit parity), so every flop is a separate
instruction: the attainable ceiling is the FP64 *issue* rate, i.e. half the
DFMA-counted peak.

The per-unit constants are MEASURED, not hand counts. oracle/port/flopcount.cpp
runs the port (the bitwise restatement of the reference) on an op-counting double
over BASELINE config 3 scenarios (N = 30/60/120, both controller models) and
divides each phase's flops by its units. tests/test_workmodel.py re-measures
them. They count the work the kernels execute, which differs from the
reference's in two exact savings:
- drift and jacobian share one exp per RK stage, where the reference evaluates it twice;
- state-only shooting runs where only F is consumed.
The N-dependence of the IPM and SQP figures is below 1 % (NX = 1) and 4 % (NX = 3);
the N = 60 values are used.
"""
EXP, LOG, SINCOS = 20.0, 20.0, 40.0

# measured, per controller state dimension (flopcount: N=60, config 3)
_MEASURED = {
    # shoot_full/ekf_step: port count with two exps per RK stage, minus the
    # 20 exps per interval/step that the kernels share
    1: dict(shoot_full=2176.0 - 20 * EXP, shoot_fonly=866.0, ipm_stage=262.5, sqp_stage=159.1,
            ekf_step=2203.0 - 20 * EXP, plant_step=1925.0),
    3: dict(shoot_full=5436.0 - 20 * EXP, shoot_fonly=1176.0, ipm_stage=852.5, sqp_stage=447.0,
            ekf_step=8061.0 - 20 * EXP, plant_step=1925.0),
}

#: plant + measurement per control step (measure, simulate_interval with Ns=10
#: Euler-Maruyama substeps on the 3-state truth, 31 normals)
PLANT_STEP = _MEASURED[1]["plant_step"]
#: PI law per control step (pi_step, controllers.cpp:12-23)
PI_STEP = 13.0
#: one shooting stage interval with forward sensitivities (Nc=5 RK4 steps)
SHOOT_FULL = _MEASURED[1]["shoot_full"]
#: one state-only stage interval (xi_from_inputs)
SHOOT_FONLY = _MEASURED[1]["shoot_fonly"]
#: one stage of one Mehrotra IPM iteration (residuals, factor, two solves,
#: expand, step length, update)
IPM_STAGE = _MEASURED[1]["ipm_stage"]
#: SQP glue per stage per iteration (Lagrangian gradient, KKT test, BFGS,
#: merit, line-search bookkeeping)
SQP_STAGE = _MEASURED[1]["sqp_stage"]
#: CD-EKF update + predict per control step (np=5 RK4 steps)
EKF_STEP = _MEASURED[1]["ekf_step"]


def pi_flops(control_steps: int) -> float:
    return control_steps * (PLANT_STEP + PI_STEP)


def nmpc_flops(counters, nx: int = 1) -> float:
    """Total algorithmic flops of an NMPC launch from the per-sample device
    counters (numpy structured array, abi.COUNTERS_DTYPE); nx = controller
    model state dimension (1: K3 / K3w / K3g one-state, 3: K3w / K3g three-state)."""
    m = _MEASURED[nx]
    c = {k: float(counters[k].sum()) for k in counters.dtype.names}
    return (c["control_steps"] * (m["plant_step"] + m["ekf_step"])
            + c["shoot_full"] * m["shoot_full"]
            + c["shoot_fonly"] * m["shoot_fonly"]
            + c["ipm_stage_iters"] * m["ipm_stage"]
            + c["sqp_stage_iters"] * m["sqp_stage"])
