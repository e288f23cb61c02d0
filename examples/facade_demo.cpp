// Minimal C++ client of the facade: a reference-style program that runs the
// PI case study through nmpcmc::gpu (build: see tests/test_cpp_facade.py).
#include <cstdio>
#include <cstring>

#include "nmpcmc_gpu.hpp"

int main(int argc, char** argv) {
    nmpcmc::gpu::Scenario sc;
    std::memset(&sc, 0, sizeof sc);
    sc.controller = NMPCMC_CTRL_PI;
    sc.truth_variant = NMPCMC_THREE_STATE;
    sc.ctrl_variant = NMPCMC_ONE_STATE;
    const nmpcmc_cstr_params p = {0.105, 0x1.679cb6b1d419cp+35, 8500.0, 560.0 / 4.186, 0.8, 1.2, 273.65,
                                  0.0, 0.0, 2.5, 0.0, 1000.0};
    sc.truth = p;
    sc.ctrl = p;
    sc.has_noise_R = 1;
    sc.noise_R = 0.01;
    sc.R_filter = 0.01;
    sc.Qz = 1.0;
    sc.horizon_Ts = 10.0;
    sc.N = 60;
    sc.Nc = 5;
    sc.np = 5;
    sc.Ns = 10;
    sc.sqp = {1e-6, 1e-4, 0.5, 1e-12, 20, 30, 50, 0};
    sc.pi = {-10.0, -0.1, -0.1, 600.0, 0.0};
    sc.u_min = 0.0;
    sc.u_max = 1000.0;
    sc.t0 = 0.0;
    sc.tf = 7200.0;
    sc.Ts = 10.0;
    sc.n_setpoints = 1;
    sc.sp_times[0] = 0.0;
    sc.sp_values[0] = 335.0;
    const double T0 = 335.0;
    sc.x0[0] = (p.cA_in - (T0 - p.cT_in) / p.beta) * p.V;
    sc.x0[1] = (p.cB_in - 2.0 * (T0 - p.cT_in) / p.beta) * p.V;
    sc.x0[2] = T0 * p.V;
    sc.x0_hat[0] = T0 * p.V;
    sc.P0[0] = 1e-6;
    sc.base_seed = 12345;
    sc.record_stride = 1;
    std::printf("N_bar = %d\n", nmpcmc::gpu::validate_scenario(sc));
    if (argc > 1 && std::strcmp(argv[1], "--validate-only") == 0) return 0;
    nmpcmc::gpu::Context ctx(0);
    const auto r = nmpcmc::gpu::run_monte_carlo(ctx, sc, 1000);
    std::printf("mean phi %.6f, failed %d\n", r.aggregate.mean, r.aggregate.n_failed);
    // the reference's run_monte_carlo(sc, n_sims, workers) shape: a GPU count
    // (every visible device here), records bitwise independent of it
    const auto rm = nmpcmc::gpu::run_monte_carlo(sc, 1000, 0);
    bool same = rm.sims.size() == r.sims.size() && rm.aggregate.mean == r.aggregate.mean;
    for (std::size_t i = 0; same && i < r.sims.size(); ++i)
        same = std::memcmp(&rm.sims[i].phi, &r.sims[i].phi, sizeof(double)) == 0;
    // two blocks on the same device through the multi-device context
    nmpcmc::gpu::Context two({0, 0});
    const auto r2 = nmpcmc::gpu::run_monte_carlo(two, sc, 1000);
    for (std::size_t i = 0; same && i < r.sims.size(); ++i)
        same = std::memcmp(&r2.sims[i].phi, &r.sims[i].phi, sizeof(double)) == 0;
    std::printf("multi-device records identical %d (devices %d)\n", same ? 1 : 0, two.num_devices());
    // standalone QP service: min 1/2 u^2 + 2u + 1/2 x1^2, x1 = 0.5 u, u in [-1, 10]
    nmpcmc::gpu::QpStage s0, s1;
    s0.R = {1.0};
    s0.r = {2.0};
    s0.Ju = {0.5};
    s0.b = {0.0};
    s0.lb = {-1.0};
    s0.ub = {10.0};
    s1.Q = {1.0};
    s1.q = {0.0};
    const auto qp = nmpcmc::gpu::solve_qp_batch(ctx, {{s0, s1}}, 1, 1);
    std::printf("qp status %d u %.9f iterations %d\n", qp[0].status, qp[0].delta_xi[0], qp[0].iterations);
    // OCP service on the NMPC variant of the scenario, cold start at T = 335 K
    sc.controller = NMPCMC_CTRL_NMPC;
    const auto ocp = nmpcmc::gpu::solve_ocp_batch(ctx, sc, {T0 * p.V}, {0.0});
    std::printf("ocp converged %d u0 %.6f\n", ocp[0].converged ? 1 : 0, ocp[0].xi[0]);
    // controller-level API: four NMPC controllers stepping on measurements
    nmpcmc::gpu::NmpcBatch ctl(ctx, sc, 4);
    std::vector<nmpcmc_nmpc_diag> dg;
    std::vector<double> u;
    for (int j = 0; j < 3; ++j) u = ctl.step({10.0 * j, 10.0 * j, 10.0 * j, 10.0 * j}, {335.0, 336.0, 334.0, 335.5}, &dg);
    std::printf("nmpc_step warm %d status %d u finite %d\n", dg[0].warm_started, dg[0].status, u[0] == u[0] ? 1 : 0);
    return 0;
}
