"""B200-native batched closed-loop Monte Carlo for the stochastic CSTR of
arXiv 2212.02197 (PI and NMPC regulators), drop-in for the reference's
run_monte_carlo path. See DESIGN.md."""
from . import abi, configs  # noqa: F401
from .engine import (  # noqa: F401
    Context, DomainError, Histogram, LengthMismatch, McResult, NonFiniteState,
    NotPositiveDefinite, SimResult, Unsupported, aggregate_stats, library,
    phi_histogram, run_closed_loop, run_monte_carlo, validate_scenario)
