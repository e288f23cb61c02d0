// nmpcmc/gpu_backend.hpp -- the reference-side adapter.
//
// What a maintainer of the reference adds next to montecarlo.hpp
// (/root/reference/proj/core/include/nmpcmc/montecarlo.hpp) to route its
// Monte Carlo loop to the B200 engine. It compiles against the reference's
// own headers and the C++ facade over the C ABI (include/nmpcmc_gpu.hpp), and
// returns the reference's own result types. tests/test_integration.py builds
// it with the reference's sources and compares it with the reference's
// run_monte_carlo (oracle/adapter_check.cpp).
//
// The reference's Scenario holds the CSTR as type-erased std::function models
// (model.hpp:28-46, built by make_cstr_model, cstr.cpp:67-128); the device
// cannot recover the plant from them, so the adapter also takes the
// CstrParams / CstrVariant the two models were built from.
#pragma once

#include <cstdint>
#include <limits>
#include <string>
#include <vector>

#include "nmpcmc/cstr.hpp"
#include "nmpcmc/errors.hpp"
#include "nmpcmc/montecarlo.hpp"
#include "nmpcmc_gpu.hpp"

namespace nmpcmc {

struct GpuCstrModels {
    CstrParams truth;
    CstrVariant truth_variant = CstrVariant::three_state;
    CstrParams ctrl;
    CstrVariant ctrl_variant = CstrVariant::one_state;
};

inline nmpcmc_cstr_params to_gpu(const CstrParams& p) {
    return {p.V, p.k0, p.EaR, p.beta, p.cA_in, p.cB_in, p.cT_in, p.sigmaA, p.sigmaB, p.sigmaT, p.u_min, p.u_max};
}

inline int32_t to_gpu(CstrVariant v) {
    return v == CstrVariant::one_state ? NMPCMC_ONE_STATE : NMPCMC_THREE_STATE;
}

/// The POD the C ABI takes, from the reference's Scenario (montecarlo.hpp:27-55).
/// Throws the reference's DimensionMismatch where the case study's single
/// input / output / measurement does not hold.
inline nmpcmc_scenario to_gpu_scenario(const Scenario& sc, const GpuCstrModels& m) {
    nmpcmc_scenario g{};
    auto one = [](const Matrix& a, const char* what) {
        if (a.rows() != 1 || a.cols() != 1) throw DimensionMismatch(std::string("gpu backend: ") + what + " must be 1x1");
        return a(0, 0);
    };
    if (sc.u_min.size() != 1 || sc.u_max.size() != 1) throw DimensionMismatch("gpu backend: n_u must be 1");
    if (sc.setpoints.times.size() > NMPCMC_MAX_SETPOINTS)
        throw DimensionMismatch("gpu backend: too many setpoint breakpoints");
    g.controller = sc.controller == ControllerType::pi ? NMPCMC_CTRL_PI : NMPCMC_CTRL_NMPC;
    g.truth_variant = to_gpu(m.truth_variant);
    g.ctrl_variant = to_gpu(m.ctrl_variant);
    g.truth = to_gpu(m.truth);
    g.ctrl = to_gpu(m.ctrl);
    g.has_noise_R = sc.noise.R.rows() > 0;
    g.noise_R = g.has_noise_R ? one(sc.noise.R, "NoiseSpec::R") : 0.0;
    g.R_filter = sc.R_filter.rows() > 0 ? one(sc.R_filter, "R_filter") : 0.0;
    g.Qz = sc.Qz.rows() > 0 ? one(sc.Qz, "Qz") : 0.0;
    g.horizon_Ts = sc.horizon.Ts;
    g.N = sc.horizon.N;
    g.Nc = sc.horizon.Nc;
    g.np = sc.np;
    g.Ns = sc.Ns;
    g.sqp = {sc.sqp.eps, sc.sqp.c1, sc.sqp.backtrack_factor, sc.sqp.qp_tol,
             sc.sqp.max_iter, sc.sqp.max_backtracks, sc.sqp.qp_max_iter, 0};
    g.pi = {sc.pi.kP, sc.pi.kI, sc.pi.kaw, sc.pi.u_bar, sc.pi.I_hat};
    g.u_min = sc.u_min[0];
    g.u_max = sc.u_max[0];
    g.t0 = sc.t0;
    g.tf = sc.tf;
    g.Ts = sc.Ts;
    g.n_setpoints = static_cast<int32_t>(sc.setpoints.times.size());
    for (int i = 0; i < g.n_setpoints; ++i) {
        if (sc.setpoints.values[i].size() != 1) throw DimensionMismatch("gpu backend: n_z must be 1");
        g.sp_times[i] = sc.setpoints.times[i];
        g.sp_values[i] = sc.setpoints.values[i][0];
    }
    for (std::size_t i = 0; i < sc.x0.size() && i < 3; ++i) g.x0[i] = sc.x0[i];
    for (std::size_t i = 0; i < sc.x0_hat.size() && i < 3; ++i) g.x0_hat[i] = sc.x0_hat[i];
    for (int c = 0; c < sc.P0.cols() && c < 3; ++c)
        for (int r = 0; r < sc.P0.rows() && r < 3; ++r) g.P0[c * sc.P0.rows() + r] = sc.P0(r, c);
    g.base_seed = sc.base_seed;
    g.record_trajectories = sc.record_trajectories ? 1 : 0;
    g.record_stride = sc.record_stride;
    return g;
}

/// Rethrow a facade error as the reference's exception of the same name
/// (errors.hpp:9-32).
template <class F>
auto with_reference_errors(F&& f) -> decltype(f()) {
    try {
        return f();
    } catch (const gpu::DimensionMismatch& e) {
        throw DimensionMismatch(e.what());
    } catch (const gpu::NotPositiveDefinite& e) {
        throw NotPositiveDefinite(e.what());
    } catch (const gpu::NonFiniteState& e) {
        throw NonFiniteState(e.what());
    } catch (const gpu::DomainError& e) {
        throw DomainError(e.what());
    } catch (const gpu::LengthMismatch& e) {
        throw LengthMismatch(e.what());
    }
}

/// Drop-in for run_monte_carlo(sc, n_sims, workers) (montecarlo.hpp:121,
/// montecarlo.cpp:213-251): the worker count becomes a GPU count (devices
/// 0 .. n_devices-1; 0 = all visible). Records are index-ordered and bitwise
/// the reference's in exact-libm mode; the aggregate is the
/// reference's aggregate_stats of those records, computed on the device (K4)
/// with the same operation order. With sc.record_trajectories the sampled
/// closed loop of every simulation comes back as the reference's Trajectory
/// (montecarlo.cpp:126-146).
inline McResult run_monte_carlo_gpu(const Scenario& sc, const GpuCstrModels& m, int n_sims, int n_devices = 0) {
    return with_reference_errors([&]() {
        const nmpcmc_scenario g = to_gpu_scenario(sc, m);
        if (n_sims < 1) throw gpu::DomainError(NMPCMC_DOMAIN_ERROR, "run_monte_carlo: n_sims must be at least 1");
        McResult out;
        out.sims.resize(static_cast<std::size_t>(n_sims));
        if (!g.record_trajectories) {
            const gpu::McResult r = gpu::run_monte_carlo(g, n_sims, n_devices);
            for (std::size_t i = 0; i < r.sims.size(); ++i) {
                SimResult& s = out.sims[i];
                s.sim_index = r.sims[i].sim_index;
                s.phi = r.sims[i].phi;
                s.failed = r.sims[i].failed;
                s.ocp_solves = r.sims[i].ocp_solves;
                s.ocp_failures = r.sims[i].ocp_failures;
            }
            const gpu::McAggregate& a = r.aggregate;
            out.aggregate.n_sims = a.n_sims;
            out.aggregate.n_failed = a.n_failed;
            out.aggregate.mean = a.mean;
            out.aggregate.variance = a.variance;
            out.aggregate.min = a.min;
            out.aggregate.max = a.max;
            out.aggregate.deciles = a.deciles;
            out.aggregate.ocp_solves = a.ocp_solves;
            out.aggregate.ocp_failures = a.ocp_failures;
            out.aggregate.ocp_success_pct = a.ocp_success_pct;
            out.wall_seconds = r.wall_seconds;
            return out;
        }
        // trajectories: one device (the per-sample rows dominate the copy)
        gpu::Context ctx(0);
        const int rows = nmpcmc_gpu_traj_rows(&g);
        std::vector<nmpcmc_sim_record> rec(static_cast<std::size_t>(n_sims));
        std::vector<double> traj(static_cast<std::size_t>(n_sims) * rows * 5);
        gpu::check(nmpcmc_gpu_run_traj(ctx.get(), &g, 0, n_sims, rec.data(), traj.data()), "run_monte_carlo",
                   ctx.get());
        for (int i = 0; i < n_sims; ++i) {
            SimResult& s = out.sims[static_cast<std::size_t>(i)];
            s.sim_index = static_cast<std::uint64_t>(i);
            s.phi = rec[i].phi;
            s.failed = rec[i].failed != 0;
            s.ocp_solves = rec[i].ocp_solves;
            s.ocp_failures = rec[i].ocp_failures;
            const double* t = traj.data() + static_cast<std::size_t>(i) * rows * 5;
            for (int k = 0; k < rows; ++k) {
                const double* row = t + 5 * k;
                if (row[0] != row[0]) break;  // unused rows of a failed run are NaN
                s.trajectory.t.push_back(row[0]);
                s.trajectory.z.push_back(Vec{row[1]});
                s.trajectory.z_bar.push_back(Vec{row[2]});
                s.trajectory.u.push_back(Vec{row[3]});
                s.trajectory.y.push_back(Vec{row[4]});
            }
        }
        out.aggregate = aggregate_stats(out.sims);
        return out;
    });
}

/// Drop-in for run_closed_loop(sc, sim_index) (montecarlo.hpp:92).
inline SimResult run_closed_loop_gpu(const Scenario& sc, const GpuCstrModels& m, std::uint64_t sim_index) {
    return with_reference_errors([&]() {
        const nmpcmc_scenario g = to_gpu_scenario(sc, m);
        gpu::Context ctx(0);
        const gpu::SimResult r = gpu::run_closed_loop(ctx, g, sim_index);
        SimResult s;
        s.sim_index = r.sim_index;
        s.phi = r.phi;
        s.failed = r.failed;
        s.ocp_solves = r.ocp_solves;
        s.ocp_failures = r.ocp_failures;
        return s;
    });
}

}  // namespace nmpcmc
