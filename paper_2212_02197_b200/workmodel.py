"""Algorithmic FP64 work per unit, for the roofline (SURVEY.md §8d convention).

Convention: +, -, *, /, sqrt = 1 flop each; transcendental weights
exp = log = 20, sincos = 40; Philox integer work not counted. The kernels
compile with --fmad=false (bit parity), so every flop is a separate
instruction: the attainable ceiling is the FP64 *issue* rate, i.e. half the
DFMA-counted peak.

Per-unit constants are hand counts from the reference source (+-10%, the
survey's figures), adjusted for the work this implementation actually
executes (drift and its jacobian share one exp; F-only shooting where only F
is consumed; the accepted line-search trial is not re-evaluated):
"""
EXP, LOG, SINCOS = 20.0, 20.0, 40.0

#: plant + measurement per control step (measure, simulate_interval with Ns=10
#: Euler-Maruyama substeps on the 3-state truth, 31 normals): survey §8d
PLANT_STEP = 866.0 + 10 * EXP + 15.5 * LOG + 15.5 * SINCOS
#: PI law per control step (pi_step, controllers.cpp:12-23)
PI_STEP = 13.0
#: one shooting stage interval with forward sensitivities (Nc=5 RK4 steps,
#: 20 stage evaluations, one exp each): survey's 1,415 flops + 20 exp
SHOOT_FULL = 1415.0 + 20 * EXP
#: one state-only stage interval (xi_from_inputs): 20 drift evaluations
#: (~15 flops + exp) + RK combination
SHOOT_FONLY = 20 * (15.0 + EXP) + 55.0
#: one stage of one Mehrotra IPM iteration (residuals, factor, two solves,
#: expand, step length, update): survey's 253
IPM_STAGE = 253.0
#: SQP glue per stage per iteration (Lagrangian gradient, KKT test, BFGS,
#: merit, line-search bookkeeping): survey's 150
SQP_STAGE = 150.0
#: CD-EKF update + predict per control step (np=5 RK4 steps, 20 exp)
EKF_STEP = 2255.0 - 20 * EXP


def pi_flops(control_steps: int) -> float:
    return control_steps * (PLANT_STEP + PI_STEP)


def nmpc_flops(counters) -> float:
    """Total algorithmic flops of an NMPC launch from the per-sample device
    counters (numpy structured array, abi.COUNTERS_DTYPE)."""
    c = {k: float(counters[k].sum()) for k in counters.dtype.names}
    return (c["control_steps"] * (PLANT_STEP + EKF_STEP)
            + c["shoot_full"] * SHOOT_FULL
            + c["shoot_fonly"] * SHOOT_FONLY
            + c["ipm_stage_iters"] * IPM_STAGE
            + c["sqp_stage_iters"] * SQP_STAGE)
