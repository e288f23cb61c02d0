// adapter_check.cpp -- TEST INFRASTRUCTURE: exercises the reference-side
// adapter integration/nmpcmc/gpu_backend.hpp from the reference's side.
//
// Built by oracle/Makefile (target `ref`) against the reference's own headers
// and its exact-libm object code (oracle/_ref/obj/xlibm), linked with
// libnmpcmc_gpu.so. Each case builds a Scenario with the reference's own API
// (make_cstr_model, cstr.cpp:67-128; the study parameters of
// /root/reference/proj/tests/support/cstr_fixtures.hpp:13-28), runs the
// reference's run_monte_carlo (montecarlo.cpp:213-251) on the host and
// run_monte_carlo_gpu through the adapter, and compares every SimResult,
// every trajectory row and the McAggregate bit for bit. Prints one line per
// case and exits non-zero on the first difference.
//
//   adapter_check            run every case (needs a GPU)
//   adapter_check --host     only build the scenarios and check the adapter's
//                            POD mapping and error translation (no GPU)
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "nmpcmc/gpu_backend.hpp"

using namespace nmpcmc;

namespace {

const double kK0 = 0x1.679cb6b1d419cp+35;  // RN(exp(24.6)), as configs.K0

CstrParams study(double sigmaT) {
    CstrParams p;
    p.V = 0.105;
    p.k0 = kK0;
    p.EaR = 8500.0;
    p.beta = 560.0 / 4.186;
    p.cA_in = 0.8;
    p.cB_in = 1.2;
    p.cT_in = 273.65;
    p.sigmaA = 0.0;
    p.sigmaB = 0.0;
    p.sigmaT = sigmaT;
    p.u_min = 0.0;
    p.u_max = 1000.0;
    return p;
}

struct Case {
    const char* name;
    ControllerType ctrl;
    CstrVariant ctrl_variant;
    int n_steps, N, n_sims;
    bool record;
};

Scenario build(const Case& c, GpuCstrModels& m) {
    m.truth = study(2.5);
    m.ctrl = study(2.5);
    m.truth_variant = CstrVariant::three_state;
    m.ctrl_variant = c.ctrl_variant;
    Scenario sc;
    sc.truth = make_cstr_model(m.truth, m.truth_variant);
    sc.noise.R = Matrix::from_rows({{0.01}});
    sc.noise.n_w = sc.truth.n_w;
    sc.controller = c.ctrl;
    sc.ctrl_model = make_cstr_model(m.ctrl, m.ctrl_variant);
    sc.horizon = Horizon{c.N, 10.0, 5};
    sc.Qz = Matrix::from_rows({{1.0}});
    sc.R_filter = Matrix::from_rows({{0.01}});
    const double T0 = 335.0;
    const CstrParams& p = m.truth;
    const double cA = p.cA_in - (T0 - p.cT_in) / p.beta, cB = p.cB_in - 2.0 * (T0 - p.cT_in) / p.beta;
    const Vec n = {cA * p.V, cB * p.V, T0 * p.V};
    const int nxc = c.ctrl_variant == CstrVariant::one_state ? 1 : 3;
    sc.x0_hat.assign(n.end() - nxc, n.end());
    sc.P0 = Matrix(nxc, nxc);
    for (int i = 0; i < nxc; ++i) sc.P0(i, i) = 1e-6;
    sc.np = 5;
    sc.sqp.eps = 1e-6;
    sc.sqp.max_iter = 20;
    sc.sqp.max_backtracks = 30;
    sc.sqp.c1 = 1e-4;
    sc.sqp.backtrack_factor = 0.5;
    sc.sqp.qp_tol = 1e-12;
    sc.sqp.qp_max_iter = 50;
    sc.pi.kP = -10.0;
    sc.pi.kI = -0.1;
    sc.pi.kaw = -0.1;
    sc.pi.u_bar = 600.0;
    sc.u_min = {0.0};
    sc.u_max = {1000.0};
    sc.t0 = 0.0;
    sc.Ts = 10.0;
    sc.tf = c.n_steps * 10.0;
    const double v[4] = {335.0, 340.0, 330.0, 340.0};
    for (int i = 0; i < 4; ++i) {
        sc.setpoints.times.push_back(sc.tf * 0.25 * i);
        sc.setpoints.values.push_back(Vec{v[i]});
    }
    sc.Ns = 10;
    sc.x0 = n;
    sc.base_seed = 12345;
    sc.record_trajectories = c.record;
    sc.record_stride = 1;
    return sc;
}

bool same(double a, double b) { return std::bit_cast<std::uint64_t>(a) == std::bit_cast<std::uint64_t>(b); }

int fail(const char* name, const std::string& what) {
    std::printf("ADAPTER MISMATCH %s: %s\n", name, what.c_str());
    return 1;
}

bool same_vecs(const std::vector<Vec>& a, const std::vector<Vec>& b) {
    if (a.size() != b.size()) return false;
    for (std::size_t i = 0; i < a.size(); ++i) {
        if (a[i].size() != b[i].size()) return false;
        for (std::size_t j = 0; j < a[i].size(); ++j)
            if (!same(a[i][j], b[i][j])) return false;
    }
    return true;
}

int compare(const Case& c, const McResult& ref, const McResult& gpu) {
    if (ref.sims.size() != gpu.sims.size()) return fail(c.name, "sim count");
    int n_failed = 0;
    for (std::size_t i = 0; i < ref.sims.size(); ++i) {
        const SimResult &a = ref.sims[i], &b = gpu.sims[i];
        n_failed += a.failed;
        if (a.sim_index != b.sim_index || !same(a.phi, b.phi) || a.failed != b.failed ||
            a.ocp_solves != b.ocp_solves || a.ocp_failures != b.ocp_failures)
            return fail(c.name, "record " + std::to_string(i));
        if (c.record) {
            const Trajectory &ta = a.trajectory, &tb = b.trajectory;
            if (ta.t.size() != tb.t.size()) return fail(c.name, "trajectory length " + std::to_string(i));
            for (std::size_t k = 0; k < ta.t.size(); ++k)
                if (!same(ta.t[k], tb.t[k])) return fail(c.name, "trajectory t " + std::to_string(i));
            if (!same_vecs(ta.z, tb.z) || !same_vecs(ta.z_bar, tb.z_bar) || !same_vecs(ta.u, tb.u) ||
                !same_vecs(ta.y, tb.y))
                return fail(c.name, "trajectory rows " + std::to_string(i));
        }
    }
    const McAggregate &A = ref.aggregate, &B = gpu.aggregate;
    if (A.n_sims != B.n_sims || A.n_failed != B.n_failed || !same(A.mean, B.mean) || !same(A.variance, B.variance) ||
        !same(A.min, B.min) || !same(A.max, B.max) || A.ocp_solves != B.ocp_solves ||
        A.ocp_failures != B.ocp_failures || !same(A.ocp_success_pct, B.ocp_success_pct) ||
        A.deciles.size() != B.deciles.size())
        return fail(c.name, "aggregate");
    for (std::size_t i = 0; i < A.deciles.size(); ++i)
        if (!same(A.deciles[i], B.deciles[i])) return fail(c.name, "decile " + std::to_string(i));
    std::printf("ADAPTER OK %s: %zu sims (%d failed) bitwise, aggregate bitwise (mean phi %.9g)%s\n", c.name,
                ref.sims.size(), n_failed, A.mean, c.record ? ", trajectories bitwise" : "");
    return 0;
}

int host_checks() {
    // error translation: tf not a multiple of Ts is the reference's DomainError
    // on both sides (validate_scenario, montecarlo.cpp:34-63)
    const Case c{"bad_tf", ControllerType::pi, CstrVariant::one_state, 10, 30, 4, false};
    GpuCstrModels m;
    Scenario sc = build(c, m);
    sc.tf = 95.0;
    bool ref_threw = false, gpu_threw = false;
    try {
        validate_scenario(sc);
    } catch (const DomainError&) {
        ref_threw = true;
    }
    try {
        gpu::validate_scenario(to_gpu_scenario(sc, m));
    } catch (const gpu::DomainError&) {
        gpu_threw = true;
    }
    if (!ref_threw || !gpu_threw) return fail(c.name, "validation does not throw DomainError on both sides");
    sc.tf = 100.0;
    sc.u_min = {0.0, 0.0};
    try {
        to_gpu_scenario(sc, m);
        return fail(c.name, "n_u = 2 accepted");
    } catch (const DimensionMismatch&) {
    }
    // the POD agrees with the reference's own checks
    sc.u_min = {0.0};
    const int nbar_ref = validate_scenario(sc);
    const int nbar_gpu = gpu::validate_scenario(to_gpu_scenario(sc, m));
    if (nbar_ref != nbar_gpu) return fail(c.name, "N_bar");
    std::printf("ADAPTER HOST OK: DomainError / DimensionMismatch translated, N_bar %d on both sides\n", nbar_ref);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (host_checks()) return 1;
    if (argc > 1 && std::strcmp(argv[1], "--host") == 0) return 0;
    const int workers = static_cast<int>(std::thread::hardware_concurrency());
    const Case cases[] = {
        {"pi_config0_720", ControllerType::pi, CstrVariant::one_state, 720, 60, 128, false},
        {"nmpc_n30_60steps", ControllerType::nmpc, CstrVariant::one_state, 60, 30, 32, false},
        {"nmpc_n60_traj", ControllerType::nmpc, CstrVariant::one_state, 40, 60, 8, true},
        {"nmpc3_n30_30steps", ControllerType::nmpc, CstrVariant::three_state, 30, 30, 8, false},
        {"pi_traj", ControllerType::pi, CstrVariant::one_state, 720, 60, 16, true},
    };
    for (const Case& c : cases) {
        GpuCstrModels m;
        const Scenario sc = build(c, m);
        const McResult ref = run_monte_carlo(sc, c.n_sims, workers > 0 ? workers : 1);
        const McResult gpu = run_monte_carlo_gpu(sc, m, c.n_sims, 1);
        if (compare(c, ref, gpu)) return 1;
    }
    // run_closed_loop drop-in on one index
    {
        const Case c{"closed_loop_17", ControllerType::nmpc, CstrVariant::one_state, 60, 30, 1, false};
        GpuCstrModels m;
        const Scenario sc = build(c, m);
        const SimResult a = run_closed_loop(sc, 17), b = run_closed_loop_gpu(sc, m, 17);
        if (!same(a.phi, b.phi) || a.failed != b.failed || a.ocp_solves != b.ocp_solves ||
            a.ocp_failures != b.ocp_failures)
            return fail(c.name, "run_closed_loop");
        std::printf("ADAPTER OK %s: run_closed_loop bitwise\n", c.name);
    }
    std::printf("ADAPTER ALL OK\n");
    return 0;
}
