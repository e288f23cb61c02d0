// ref_driver.cpp -- C-ABI driver around the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE (oracle): linked against the reference core compiled
// from /root/reference/proj/core/src/*.cpp by oracle/Makefile into
// oracle/_ref/. It translates the POD nmpcmc_scenario of include/nmpcmc_gpu.h
// into the reference's Scenario (montecarlo.hpp:27-55) and calls the
// reference's own entry points:
//   run_closed_loop  (montecarlo.cpp:80-157)   -> nmpcmc_ref_run_closed_loop
//   run_monte_carlo  (montecarlo.cpp:213-251)  -> nmpcmc_ref_run_batch
//   aggregate_stats  (montecarlo.cpp:172-211)  -> nmpcmc_ref_aggregate
//   phi_histogram    (montecarlo.cpp:268-304)  -> nmpcmc_ref_histogram
//   solve_qp / riccati_factor_solve (qp.cpp:157-423) -> nmpcmc_ref_solve_qp_batch
//   sqp_solve on the regulator OcpProblem (sqp.cpp:182-411)  -> nmpcmc_ref_solve_ocp_batch
// and, for unit-level pins, CounterRng / pi_step / nmpc_step.
// Only tests/, __graft_entry__.smoke() and bench.py's CPU arm load it.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

#include "nmpcmc/controllers.hpp"
#include "nmpcmc/cstr.hpp"
#include "nmpcmc/errors.hpp"
#include "nmpcmc/montecarlo.hpp"
#include "nmpcmc/ocp.hpp"
#include "nmpcmc/qp.hpp"
#include "nmpcmc/sqp.hpp"
#include "nmpcmc/rng.hpp"
#include "nmpcmc_gpu.h"

using namespace nmpcmc;

namespace {

CstrParams to_params(const nmpcmc_cstr_params& p) {
    CstrParams q;
    q.V = p.V;
    q.k0 = p.k0;
    q.EaR = p.EaR;
    q.beta = p.beta;
    q.cA_in = p.cA_in;
    q.cB_in = p.cB_in;
    q.cT_in = p.cT_in;
    q.sigmaA = p.sigmaA;
    q.sigmaB = p.sigmaB;
    q.sigmaT = p.sigmaT;
    q.u_min = p.u_min;
    q.u_max = p.u_max;
    return q;
}

CstrVariant to_variant(int v) { return v == NMPCMC_ONE_STATE ? CstrVariant::one_state : CstrVariant::three_state; }
int nx_of(int v) { return v == NMPCMC_ONE_STATE ? 1 : 3; }

/// Per-sample truth parameters: the BASELINE perturbation rule of
/// include/nmpcmc_gpu.h, drawn with the reference's own CounterRng.
CstrParams truth_params(const nmpcmc_scenario& s, std::uint64_t sim_index) {
    CstrParams p = to_params(s.truth);
    if (s.perturb) {
        CounterRng prng(s.base_seed, sim_index | 0x8000000000000000ULL);
        const double z0 = prng.normal();
        const double z1 = prng.normal();
        const double z2 = prng.normal();
        p.cA_in = p.cA_in * (1.0 + s.perturb_rel_std[0] * z0);
        p.cB_in = p.cB_in * (1.0 + s.perturb_rel_std[1] * z1);
        p.EaR = p.EaR * (1.0 + s.perturb_rel_std[2] * z2);
    }
    return p;
}

/// nmpcmc_ref_set_ctrl_fd: build the controller model without its analytic
/// jacobians, so the reference takes its finite-difference fallbacks
/// (model.cpp:54-124) -- the counterpart of NMPCMC_OPT_CTRL_JACOBIANS = FD.
int g_ctrl_fd = 0;

Scenario make_scenario(const nmpcmc_scenario& s, std::uint64_t sim_index) {
    Scenario sc;
    sc.truth = make_cstr_model(truth_params(s, sim_index), to_variant(s.truth_variant));
    if (s.has_noise_R) sc.noise.R = Matrix::from_rows({{s.noise_R}});
    sc.noise.n_w = sc.truth.n_w;
    sc.controller = s.controller == NMPCMC_CTRL_PI ? ControllerType::pi : ControllerType::nmpc;
    sc.ctrl_model = make_cstr_model(to_params(s.ctrl), to_variant(s.ctrl_variant));
    if (g_ctrl_fd) {
        sc.ctrl_model.drift_jacobian_x = nullptr;
        sc.ctrl_model.drift_jacobian_u = nullptr;
        sc.ctrl_model.measurement_jacobian_x = nullptr;
        sc.ctrl_model.output_jacobian_x = nullptr;
    }
    sc.horizon = Horizon{s.N, s.horizon_Ts, s.Nc};
    sc.Qz = Matrix::from_rows({{s.Qz}});
    sc.R_filter = Matrix::from_rows({{s.R_filter}});
    const int nxc = nx_of(s.ctrl_variant);
    sc.x0_hat.assign(s.x0_hat, s.x0_hat + nxc);
    sc.P0 = Matrix(nxc, nxc);
    for (int c = 0; c < nxc; ++c)
        for (int r = 0; r < nxc; ++r) sc.P0(r, c) = s.P0[c * nxc + r];
    sc.np = s.np;
    sc.sqp.eps = s.sqp.eps;
    sc.sqp.max_iter = s.sqp.max_iter;
    sc.sqp.max_backtracks = s.sqp.max_backtracks;
    sc.sqp.c1 = s.sqp.c1;
    sc.sqp.backtrack_factor = s.sqp.backtrack_factor;
    sc.sqp.qp_tol = s.sqp.qp_tol;
    sc.sqp.qp_max_iter = s.sqp.qp_max_iter;
    sc.pi.kP = s.pi.kP;
    sc.pi.kI = s.pi.kI;
    sc.pi.kaw = s.pi.kaw;
    sc.pi.u_bar = s.pi.u_bar;
    sc.pi.I_hat = s.pi.I_hat;
    sc.u_min = {s.u_min};
    sc.u_max = {s.u_max};
    sc.t0 = s.t0;
    sc.tf = s.tf;
    sc.Ts = s.Ts;
    sc.Ns = s.Ns;
    for (int i = 0; i < s.n_setpoints; ++i) {
        sc.setpoints.times.push_back(s.sp_times[i]);
        sc.setpoints.values.push_back(Vec{s.sp_values[i]});
    }
    sc.x0.assign(s.x0, s.x0 + nx_of(s.truth_variant));
    sc.base_seed = s.base_seed;
    sc.record_trajectories = s.record_trajectories != 0;
    sc.record_stride = s.record_stride;
    return sc;
}

void to_record(const SimResult& r, nmpcmc_sim_record* out) {
    out->phi = r.phi;
    out->failed = r.failed ? 1 : 0;
    out->ocp_solves = r.ocp_solves;
    out->ocp_failures = r.ocp_failures;
    out->status = r.failed ? -1 : 0;  // the reference swallows the cause
}

/// The worker body of run_monte_carlo (montecarlo.cpp:226-236): anything
/// run_closed_loop does not absorb still only fails this one simulation.
void run_one(const nmpcmc_scenario& s, std::uint64_t idx, nmpcmc_sim_record* out, double* traj,
             int rows) {
    try {
        const Scenario sc = make_scenario(s, idx);
        const SimResult r = run_closed_loop(sc, idx);
        to_record(r, out);
        if (traj != nullptr) {
            const Trajectory& tr = r.trajectory;
            const double nan = std::numeric_limits<double>::quiet_NaN();
            for (int i = 0; i < rows; ++i) {
                const bool have = static_cast<std::size_t>(i) < tr.t.size();
                traj[i * 5 + 0] = have ? tr.t[i] : nan;
                traj[i * 5 + 1] = have ? tr.z[i][0] : nan;
                traj[i * 5 + 2] = have ? tr.z_bar[i][0] : nan;
                traj[i * 5 + 3] = have ? tr.u[i][0] : nan;
                traj[i * 5 + 4] = have ? tr.y[i][0] : nan;
            }
        }
    } catch (...) {
        out->phi = std::numeric_limits<double>::quiet_NaN();
        out->failed = 1;
        out->ocp_solves = 0;
        out->ocp_failures = 0;
        out->status = -2;
        if (traj != nullptr)
            for (int i = 0; i < rows * 5; ++i) traj[i] = std::numeric_limits<double>::quiet_NaN();
    }
}

}  // namespace

extern "C" {

void nmpcmc_ref_set_ctrl_fd(int on) { g_ctrl_fd = on ? 1 : 0; }

int nmpcmc_ref_validate(const nmpcmc_scenario* s, int* nbar) {
    try {
        *nbar = validate_scenario(make_scenario(*s, 0));
        return 0;
    } catch (const DomainError&) {
        return NMPCMC_DOMAIN_ERROR;
    } catch (...) {
        return NMPCMC_INVALID_ARGUMENT;
    }
}

/// run_closed_loop for one global index; traj (nullable) gets rows*5 doubles.
int nmpcmc_ref_run_closed_loop(const nmpcmc_scenario* s, std::uint64_t sim_index,
                               nmpcmc_sim_record* out, double* traj, int rows) {
    run_one(*s, sim_index, out, traj, rows);
    return 0;
}

/// Batch over [first, first+n) on `workers` threads. With no per-sample
/// parameters and first == 0 this IS the reference's run_monte_carlo;
/// otherwise the same atomic-counter pool over per-sample Scenarios.
int nmpcmc_ref_run_batch(const nmpcmc_scenario* s, std::uint64_t first, std::int64_t n,
                         int workers, nmpcmc_sim_record* out, double* wall_seconds) {
    if (n < 1 || workers < 1) return NMPCMC_DOMAIN_ERROR;
    if (!s->perturb && first == 0 && n <= std::numeric_limits<int>::max()) {
        const Scenario sc = make_scenario(*s, 0);
        const McResult r = run_monte_carlo(sc, static_cast<int>(n), workers);
        for (std::int64_t i = 0; i < n; ++i) to_record(r.sims[static_cast<std::size_t>(i)], &out[i]);
        if (wall_seconds) *wall_seconds = r.wall_seconds;
        return 0;
    }
    std::atomic<std::int64_t> next{0};
    const auto start = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    const int nt = static_cast<int>(std::min<std::int64_t>(workers, n));
    for (int w = 0; w < nt; ++w)
        pool.emplace_back([&]() {
            for (;;) {
                const std::int64_t i = next.fetch_add(1, std::memory_order_relaxed);
                if (i >= n) return;
                run_one(*s, first + static_cast<std::uint64_t>(i), &out[i], nullptr, 0);
            }
        });
    for (auto& th : pool) th.join();
    if (wall_seconds)
        *wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    return 0;
}

int nmpcmc_ref_aggregate(const nmpcmc_sim_record* rec, std::int64_t n, nmpcmc_aggregate* out) {
    std::vector<SimResult> sims(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) {
        sims[i].phi = rec[i].phi;
        sims[i].failed = rec[i].failed != 0;
        sims[i].ocp_solves = rec[i].ocp_solves;
        sims[i].ocp_failures = rec[i].ocp_failures;
    }
    const McAggregate a = aggregate_stats(sims);
    out->n_sims = a.n_sims;
    out->n_failed = a.n_failed;
    out->mean = a.mean;
    out->variance = a.variance;
    out->min = a.min;
    out->max = a.max;
    for (int d = 0; d < 11; ++d) out->deciles[d] = a.deciles[static_cast<std::size_t>(d)];
    out->ocp_solves = a.ocp_solves;
    out->ocp_failures = a.ocp_failures;
    out->ocp_success_pct = a.ocp_success_pct;
    return 0;
}

int nmpcmc_ref_histogram(const double* phi, std::int64_t n, int bins, double* edges,
                         int* counts, int* nbins) {
    const Histogram h = phi_histogram(std::vector<double>(phi, phi + n), bins);
    *nbins = static_cast<int>(h.counts.size());
    for (std::size_t i = 0; i < h.edges.size(); ++i) edges[i] = h.edges[i];
    for (std::size_t i = 0; i < h.counts.size(); ++i) counts[i] = h.counts[i];
    return 0;
}

void nmpcmc_ref_philox_block(const std::uint32_t* in, std::uint32_t* out) {
    const auto r = CounterRng::philox_block({in[0], in[1], in[2], in[3]}, {in[4], in[5]});
    for (int i = 0; i < 4; ++i) out[i] = r[static_cast<std::size_t>(i)];
}

void nmpcmc_ref_normals(std::uint64_t seed, std::uint64_t stream, std::int64_t n, double* out) {
    CounterRng rng(seed, stream);
    for (std::int64_t i = 0; i < n; ++i) out[i] = rng.normal();
}

/// pi_step (controllers.cpp:12-23): state[8] = kP,kI,kaw,Ts,u_bar,u_min,u_max,I_hat;
/// out[7] = e, P, I, u_hat, u, I_aw, next.I_hat.
void nmpcmc_ref_pi_step(const double* st, double y, double ybar, double* out) {
    PiState s;
    s.kP = st[0];
    s.kI = st[1];
    s.kaw = st[2];
    s.Ts = st[3];
    s.u_bar = st[4];
    s.u_min = st[5];
    s.u_max = st[6];
    s.I_hat = st[7];
    const PiStepResult r = pi_step(s, y, ybar);
    out[0] = r.e;
    out[1] = r.P;
    out[2] = r.I;
    out[3] = r.u_hat;
    out[4] = r.u;
    out[5] = r.I_aw;
    out[6] = r.next.I_hat;
}

/// The reference's make_nmpc_state (controllers.cpp:25-48) + nmpc_step
/// (controllers.cpp:114-212) for B independent controllers over T steps:
/// instance b steps with (t[b*T + j], y[b*T + j]) and setpoints
/// sp[(b*T + j)*N + k] (NULL: the scenario's profile at t + (k+1) Ts). An
/// exception fails only that step (status, NaN input); the NmpcState keeps
/// whatever the reference left in it and the next step continues from there.
/// Outputs per step: u, and the diagnostics in the layout of nmpcmc_nmpc_diag;
/// per instance the final state (x_hat, P, last_xi, last duals, warm).
int nmpcmc_ref_nmpc_steps(const nmpcmc_scenario* s, std::int64_t B, int T, const double* x0_hat, const double* P0,
                          const double* t, const double* y, const double* sp, double* u_out, nmpcmc_nmpc_diag* diag,
                          double* xhat_out, double* P_out, double* xi_out, double* lam_out, double* pil_out,
                          double* piu_out, std::int32_t* warm_out) {
    const int nx = nx_of(s->ctrl_variant), N = s->N, L = N * (1 + nx);
    SqpOptions opts;
    opts.eps = s->sqp.eps;
    opts.max_iter = s->sqp.max_iter;
    opts.max_backtracks = s->sqp.max_backtracks;
    opts.c1 = s->sqp.c1;
    opts.backtrack_factor = s->sqp.backtrack_factor;
    opts.qp_tol = s->sqp.qp_tol;
    opts.qp_max_iter = s->sqp.qp_max_iter;
    SetpointProfile prof;
    for (int i = 0; i < s->n_setpoints; ++i) {
        prof.times.push_back(s->sp_times[i]);
        prof.values.push_back(Vec{s->sp_values[i]});
    }
    const double nan = std::numeric_limits<double>::quiet_NaN();
    for (std::int64_t b = 0; b < B; ++b) {
        Vec xh(nx);
        Matrix p0(nx, nx);
        for (int i = 0; i < nx; ++i) xh[i] = x0_hat ? x0_hat[b * nx + i] : s->x0_hat[i];
        for (int c = 0; c < nx; ++c)
            for (int r = 0; r < nx; ++r) p0(r, c) = P0 ? P0[b * nx * nx + c * nx + r] : s->P0[c * nx + r];
        NmpcState st = make_nmpc_state(make_cstr_model(to_params(s->ctrl), to_variant(s->ctrl_variant)),
                                       Horizon{N, s->horizon_Ts, s->Nc}, Vec{s->u_min}, Vec{s->u_max},
                                       Matrix::from_rows({{s->Qz}}), Matrix::from_rows({{s->R_filter}}), xh, p0,
                                       s->np, opts);
        for (int j = 0; j < T; ++j) {
            const std::int64_t q = b * T + j;
            std::vector<Vec> spv;
            for (int k = 0; k < N; ++k)
                spv.push_back(sp ? Vec{sp[q * N + k]} : prof.at(t[q] + (k + 1) * s->Ts));
            NmpcDiagnostics dg;
            nmpcmc_nmpc_diag& d = diag[q];
            std::memset(&d, 0, sizeof d);
            for (int i = 0; i < nx; ++i) d.x_filtered[i] = nan;
            for (int i = 0; i < nx * nx; ++i) d.P_filtered[i] = nan;
            d.innovation = std::isfinite(y[q]) ? y[q] - st.filter.x_hat[nx - 1] / s->ctrl.V : nan;
            d.warm_started = static_cast<int>(st.last_xi.size()) == L ? 1 : 0;
            try {
                const Vec u = nmpc_step(st, t[q], Vec{y[q]}, spv, Vec{}, &dg);
                u_out[q] = u[0];
                for (int i = 0; i < nx; ++i) d.x_filtered[i] = dg.filtered.x_hat[i];
                for (int c = 0; c < nx; ++c)
                    for (int r = 0; r < nx; ++r) d.P_filtered[c * nx + r] = dg.filtered.P(r, c);
                d.innovation = dg.innovation[0];
                d.converged = dg.sqp.converged ? 1 : 0;
                d.sqp_iterations = dg.sqp.iterations;
                d.status = 0;
            } catch (const NotPositiveDefinite&) {
                u_out[q] = nan, d.status = NMPCMC_NOT_POSITIVE_DEFINITE;
            } catch (const NonFiniteState&) {
                u_out[q] = nan, d.status = NMPCMC_NON_FINITE_STATE;
            } catch (const DomainError&) {
                u_out[q] = nan, d.status = NMPCMC_DOMAIN_ERROR;
            }
        }
        for (int i = 0; i < nx; ++i) xhat_out[b * nx + i] = st.filter.x_hat[i];
        for (int c = 0; c < nx; ++c)
            for (int r = 0; r < nx; ++r) P_out[b * nx * nx + c * nx + r] = st.filter.P(r, c);
        const bool w = static_cast<int>(st.last_xi.size()) == L;
        warm_out[b] = w ? 1 : 0;
        for (int i = 0; i < L; ++i) xi_out[b * L + i] = w ? st.last_xi[i] : 0.0;
        for (int i = 0; i < N * nx; ++i) lam_out[b * N * nx + i] = w ? st.last_duals.lambda[i] : 0.0;
        for (int i = 0; i < N; ++i) pil_out[b * N + i] = w ? st.last_duals.pi_l[i] : 0.0;
        for (int i = 0; i < N; ++i) piu_out[b * N + i] = w ? st.last_duals.pi_u[i] : 0.0;
    }
    return 0;
}

/// A stagewise quadratic NLP through the reference's SqpProblem interface
/// (sqp.hpp:15-25), as its SQP tests pose plain QPs: the packed layout and the
/// evaluation order of nmpcmc_gpu_sqp_solve_qnlp_batch (include/nmpcmc_gpu.h,
/// Qnlp in csrc/nmpc_gen_kernel.cuh). Test infrastructure: the thing under
/// test is the reference's sqp_solve run on it.
class QnlpProblem final : public SqpProblem {
public:
    QnlpProblem(const double* data, int N, int nx) : d_(data), N_(N), nx_(nx) {
        lay_.N = N;
        lay_.n_x = nx;
        lay_.n_u = 1;
        umin_ = {data[nx]};
        umax_ = {data[nx + 1]};
    }
    XiLayout layout() const override { return lay_; }
    const Vec& u_min() const override { return umin_; }
    const Vec& u_max() const override { return umax_; }
    double objective(const Vec& xi, Vec* grad) const override {
        const int nx = nx_;
        double phi = 0.0;
        for (int k = 0; k < N_; ++k) {
            const double* P = stage(k);
            const double u = xi[lay_.u_offset(k)];
            const double su = P[0] * u;
            phi = phi + (0.5 * (u * su) + P[1] * u);
            double xQx = 0.0, qx = 0.0;
            for (int i = 0; i < nx; ++i) {
                double qxi = 0.0;
                for (int j = 0; j < nx; ++j) qxi += P[2 + j * nx + i] * xi[lay_.x_offset(k + 1) + j];
                const double xv = xi[lay_.x_offset(k + 1) + i];
                xQx += xv * qxi;
                qx += P[2 + nx * nx + i] * xv;
            }
            phi = phi + (0.5 * xQx + qx);
        }
        if (grad != nullptr) {
            grad->assign(static_cast<std::size_t>(lay_.size()), 0.0);
            for (int k = 0; k < N_; ++k) {
                const double* P = stage(k);
                const double u = xi[lay_.u_offset(k)];
                (*grad)[lay_.u_offset(k)] = P[0] * u + P[1];
                for (int i = 0; i < nx; ++i) {
                    double qxi = 0.0;
                    for (int j = 0; j < nx; ++j) qxi += P[2 + j * nx + i] * xi[lay_.x_offset(k + 1) + j];
                    (*grad)[lay_.x_offset(k + 1) + i] = qxi + P[2 + nx * nx + i];
                }
            }
        }
        return phi;
    }
    ConstraintBlocks constraints(const Vec& xi) const override {
        const int nx = nx_;
        ConstraintBlocks cb;
        cb.g.assign(static_cast<std::size_t>(N_ * nx), 0.0);
        for (int k = 0; k < N_; ++k) {
            const double* P = stage(k);
            const double* A = P + 2 + nx * nx + nx;
            const double* B = A + nx * nx;
            const double* c = B + nx;
            Matrix Fx(nx, nx), Fu(nx, 1);
            Vec b(nx);
            for (int i = 0; i < nx; ++i) {
                double F = 0.0;
                for (int j = 0; j < nx; ++j) F += A[j * nx + i] * (k == 0 ? d_[j] : xi[lay_.x_offset(k) + j]);
                F = F + B[i] * xi[lay_.u_offset(k)];
                F = F + c[i];
                const double nxt = xi[lay_.x_offset(k + 1) + i];
                cb.g[k * nx + i] = nxt - F;
                b[i] = F - nxt;
                Fu(i, 0) = B[i];
                for (int j = 0; j < nx; ++j) Fx(i, j) = A[j * nx + i];
            }
            cb.dF_dx.push_back(Fx);
            cb.dF_du.push_back(Fu);
            cb.b.push_back(b);
        }
        return cb;
    }

private:
    const double* stage(int k) const { return d_ + nx_ + 2 + static_cast<std::ptrdiff_t>(k) * (2 + 2 * nx_ * nx_ + 3 * nx_); }
    const double* d_;
    int N_, nx_;
    XiLayout lay_;
    Vec umin_, umax_;
};

/// The reference's sqp_solve on a batch of QnlpProblems (layout of
/// nmpcmc_gpu_sqp_solve_qnlp_batch); status NMPCMC_DOMAIN_ERROR etc. where it throws.
int nmpcmc_ref_sqp_solve_qnlp_batch(const nmpcmc_qnlp_dims* d, std::int64_t batch, const double* problems,
                                    const double* xi0_in, double* xi_out, double* lam_out, double* pil_out,
                                    double* piu_out, std::int32_t* converged, std::int32_t* iters,
                                    std::int32_t* status) {
    const int N = d->N, nx = d->n_x, L = N * (1 + nx);
    const std::int64_t stride = nx + 2 + static_cast<std::int64_t>(N) * (2 + 2 * nx * nx + 3 * nx);
    SqpOptions opts;
    opts.eps = d->sqp.eps;
    opts.max_iter = d->sqp.max_iter;
    opts.max_backtracks = d->sqp.max_backtracks;
    opts.c1 = d->sqp.c1;
    opts.backtrack_factor = d->sqp.backtrack_factor;
    opts.qp_tol = d->sqp.qp_tol;
    opts.qp_max_iter = d->sqp.qp_max_iter;
    for (std::int64_t b = 0; b < batch; ++b) {
        const QnlpProblem prob(problems + b * stride, N, nx);
        Vec xi0(static_cast<std::size_t>(L), 0.0);
        if (xi0_in != nullptr) xi0.assign(xi0_in + b * L, xi0_in + (b + 1) * L);
        std::fill(xi_out + b * L, xi_out + (b + 1) * L, 0.0);
        std::fill(lam_out + b * N * nx, lam_out + (b + 1) * N * nx, 0.0);
        std::fill(pil_out + b * N, pil_out + (b + 1) * N, 0.0);
        std::fill(piu_out + b * N, piu_out + (b + 1) * N, 0.0);
        converged[b] = 0;
        iters[b] = 0;
        try {
            const SqpReport rep = sqp_solve(prob, xi0, opts, SqpWarmStart{});
            std::copy(rep.xi.begin(), rep.xi.end(), xi_out + b * L);
            std::copy(rep.lambda.begin(), rep.lambda.end(), lam_out + b * N * nx);
            std::copy(rep.pi_l.begin(), rep.pi_l.end(), pil_out + b * N);
            std::copy(rep.pi_u.begin(), rep.pi_u.end(), piu_out + b * N);
            converged[b] = rep.converged ? 1 : 0;
            iters[b] = rep.iterations;
            status[b] = 0;
        } catch (const DomainError&) {
            status[b] = NMPCMC_DOMAIN_ERROR;
        } catch (const NonFiniteState&) {
            status[b] = NMPCMC_NON_FINITE_STATE;
        } catch (const NotPositiveDefinite&) {
            status[b] = NMPCMC_NOT_POSITIVE_DEFINITE;
        }
    }
    return 0;
}

/// reaction_rate (cstr.cpp:36-40) on the three-state variant; NaN on DomainError.
double nmpcmc_ref_reaction_rate(const nmpcmc_cstr_params* p, const double* c) {
    const CstrParams q = to_params(*p);
    try {
        return reaction_rate({c[0], c[1], c[2]}, q, stoich_config(CstrVariant::three_state, q));
    } catch (...) {
        return std::numeric_limits<double>::quiet_NaN();
    }
}

/// The reference's solve_qp (mode 0) / riccati_factor_solve (mode 1) over a
/// batch in the packed layout of nmpcmc_gpu_solve_qp_batch (include/nmpcmc_gpu.h).
int nmpcmc_ref_solve_qp_batch(const nmpcmc_qp_dims* d, std::int64_t batch, const double* stages,
                              double* solutions, std::int32_t* status, std::int32_t* iterations) {
    const int N = d->N, nx = d->n_x, nu = d->n_u;
    const int SB = 2 * nx * nx + 2 * nx * nu + nu * nu + 2 * nx + 3 * nu;
    const std::int64_t SO = (std::int64_t)N * (nu + nx) + (std::int64_t)N * nx + 2 * (std::int64_t)N * nu;
    auto mat = [](const double* p, int r, int c) {
        Matrix m(r, c);
        for (int j = 0; j < c; ++j)
            for (int i = 0; i < r; ++i) m(i, j) = p[j * r + i];
        return m;
    };
    auto vec = [](const double* p, int n) { return Vec(p, p + n); };
    for (std::int64_t b = 0; b < batch; ++b) {
        std::vector<QpStageData> st(N + 1);
        for (int k = 0; k <= N; ++k) {
            const double* p = stages + (b * (N + 1) + k) * SB;
            const int oM = nx * nx, oR = oM + nx * nu, oq = oR + nu * nu, orr = oq + nx, oJx = orr + nu,
                      oJu = oJx + nx * nx, ob = oJu + nx * nu, olb = ob + nx, oub = olb + nu;
            QpStageData& s = st[k];
            if (k == N) {
                s.Q = mat(p, nx, nx);
                s.q = vec(p + oq, nx);
                continue;
            }
            if (k >= 1) {
                s.Q = mat(p, nx, nx);
                s.M = mat(p + oM, nx, nu);
                s.q = vec(p + oq, nx);
                s.Jx = mat(p + oJx, nx, nx);
            }
            s.R = mat(p + oR, nu, nu);
            s.r = vec(p + orr, nu);
            s.Ju = mat(p + oJu, nx, nu);
            s.b = vec(p + ob, nx);
            s.lb = vec(p + olb, nu);
            s.ub = vec(p + oub, nu);
        }
        double* o = solutions + b * SO;
        std::fill(o, o + SO, 0.0);
        const std::int64_t L = (std::int64_t)N * (nu + nx), NX = (std::int64_t)N * nx, NV = (std::int64_t)N * nu;
        iterations[b] = 0;
        try {
            if (d->mode == 1) {
                const auto [dxi, mu] = riccati_factor_solve(st);
                std::copy(dxi.begin(), dxi.end(), o);
                std::copy(mu.begin(), mu.end(), o + L);
                status[b] = NMPCMC_QP_OPTIMAL;
            } else {
                const QpSolution sol = solve_qp(st, d->tol, d->max_iter);
                std::copy(sol.delta_xi.begin(), sol.delta_xi.end(), o);
                std::copy(sol.mu.begin(), sol.mu.end(), o + L);
                std::copy(sol.nu_l.begin(), sol.nu_l.end(), o + L + NX);
                std::copy(sol.nu_u.begin(), sol.nu_u.end(), o + L + NX + NV);
                status[b] = sol.status == QpStatus::Optimal ? NMPCMC_QP_OPTIMAL
                            : sol.status == QpStatus::MaxIter ? NMPCMC_QP_MAXITER
                                                              : NMPCMC_QP_FAILED;
                iterations[b] = sol.iterations;
            }
        } catch (const DomainError&) {
            status[b] = NMPCMC_QP_DOMAIN_ERROR;
        } catch (const NotPositiveDefinite&) {
            status[b] = NMPCMC_QP_NOT_POSITIVE_DEFINITE;
        }
    }
    return 0;
}

/// The reference's sqp_solve on the regulator OcpProblem of the scenario's
/// controller model for each (x0[b], t0[b]): NlpInstance as nmpc_step builds it
/// (controllers.cpp:134-145) and its cold start (controllers.cpp:166-185) when
/// xi0 is NULL, else the given iterate with zero duals. status[b]: 0, or
/// NMPCMC_DOMAIN_ERROR if a DomainError escaped.
int nmpcmc_ref_solve_ocp_batch_traced(const nmpcmc_scenario* s, std::int64_t batch, const double* x0,
                                      const double* t0, const double* xi0_in, double* xi_out, double* lam_out,
                                      double* pil_out, double* piu_out, std::int32_t* converged,
                                      std::int32_t* status, std::int32_t* iterations, std::int32_t max_trace,
                                      nmpcmc_sqp_iter_log* trace, std::int32_t* trace_len);

int nmpcmc_ref_solve_ocp_batch(const nmpcmc_scenario* s, std::int64_t batch, const double* x0, const double* t0,
                               const double* xi0_in, double* xi_out, double* lam_out, double* pil_out,
                               double* piu_out, std::int32_t* converged, std::int32_t* status) {
    return nmpcmc_ref_solve_ocp_batch_traced(s, batch, x0, t0, xi0_in, xi_out, lam_out, pil_out, piu_out, converged,
                                             status, nullptr, 0, nullptr, nullptr);
}

/// As nmpcmc_ref_solve_ocp_batch, plus SqpReport::iterations and the
/// SqpReport::trace records (sqp.hpp:64-90) in the layout of
/// nmpcmc_sqp_iter_log (any of the three may be NULL).
int nmpcmc_ref_solve_ocp_batch_traced(const nmpcmc_scenario* s, std::int64_t batch, const double* x0,
                                      const double* t0, const double* xi0_in, double* xi_out, double* lam_out,
                                      double* pil_out, double* piu_out, std::int32_t* converged,
                                      std::int32_t* status, std::int32_t* iterations, std::int32_t max_trace,
                                      nmpcmc_sqp_iter_log* trace, std::int32_t* trace_len) {
    const int nx = nx_of(s->ctrl_variant), N = s->N, L = N * (1 + nx);
    SqpOptions opts;
    opts.eps = s->sqp.eps;
    opts.max_iter = s->sqp.max_iter;
    opts.max_backtracks = s->sqp.max_backtracks;
    opts.c1 = s->sqp.c1;
    opts.backtrack_factor = s->sqp.backtrack_factor;
    opts.qp_tol = s->sqp.qp_tol;
    opts.qp_max_iter = s->sqp.qp_max_iter;
    SetpointProfile prof;
    for (int i = 0; i < s->n_setpoints; ++i) {
        prof.times.push_back(s->sp_times[i]);
        prof.values.push_back(Vec{s->sp_values[i]});
    }
    for (std::int64_t b = 0; b < batch; ++b) {
        NlpInstance nlp;
        nlp.horizon = Horizon{N, s->horizon_Ts, s->Nc};
        nlp.model = make_cstr_model(to_params(s->ctrl), to_variant(s->ctrl_variant));
        nlp.t0 = t0[b];
        nlp.x0.assign(x0 + b * nx, x0 + (b + 1) * nx);
        nlp.u_min = {s->u_min};
        nlp.u_max = {s->u_max};
        for (int k = 1; k <= N; ++k) nlp.setpoints.push_back(prof.at(t0[b] + k * s->Ts));
        nlp.Qz = Matrix::from_rows({{s->Qz}});
        double* xo = xi_out + b * L;
        std::fill(xo, xo + L, 0.0);
        std::fill(lam_out + b * N * nx, lam_out + (b + 1) * N * nx, 0.0);
        std::fill(pil_out + b * N, pil_out + (b + 1) * N, 0.0);
        std::fill(piu_out + b * N, piu_out + (b + 1) * N, 0.0);
        converged[b] = 0;
        if (iterations) iterations[b] = 0;
        if (trace_len) trace_len[b] = 0;
        try {
            const OcpProblem problem(std::move(nlp));
            Vec xi0;
            if (xi0_in != nullptr) {
                xi0.assign(xi0_in + b * L, xi0_in + (b + 1) * L);
            } else {  // cold start (controllers.cpp:166-185), nominal_input (:58-66)
                const bool fl = std::isfinite(s->u_min), fh = std::isfinite(s->u_max);
                const double un = fl && fh ? 0.5 * (s->u_min + s->u_max) : std::max(s->u_min, std::min(s->u_max, 0.0));
                try {
                    xi0 = xi_from_inputs(problem.nlp(), std::vector<Vec>(N, Vec{un}));
                } catch (const NonFiniteState&) {
                    xi0.assign(L, 0.0);
                    for (int k = 0; k < N; ++k) {
                        xi0[k * (1 + nx)] = un;
                        for (int i = 0; i < nx; ++i) xi0[k * (1 + nx) + 1 + i] = problem.nlp().x0[i];
                    }
                }
            }
            const SqpReport rep = sqp_solve(problem, xi0, opts, SqpWarmStart{});
            if (iterations) iterations[b] = rep.iterations;
            if (trace_len) trace_len[b] = static_cast<std::int32_t>(rep.trace.size());
            for (std::size_t q = 0; trace && q < rep.trace.size() && q < static_cast<std::size_t>(max_trace); ++q) {
                const SqpIterationLog& lg = rep.trace[q];
                nmpcmc_sqp_iter_log& d = trace[b * max_trace + static_cast<std::int64_t>(q)];
                d = nmpcmc_sqp_iter_log{};
                d.alpha = lg.alpha;
                d.merit_before = lg.merit_before;
                d.merit_after = lg.merit_after;
                d.directional_derivative = lg.directional_derivative;
                d.grad_l_inf = lg.grad_l_inf;
                d.g_inf = lg.g_inf;
                d.step_inf = lg.step_inf;
                d.ls_evals = lg.ls_evals;
                d.qp_iterations = lg.qp_iterations;
                d.qp_status = static_cast<std::int32_t>(lg.qp_status);
                d.armijo_exhausted = lg.armijo_exhausted ? 1 : 0;
                d.bfgs_reset = lg.bfgs_reset ? 1 : 0;
            }
            std::copy(rep.xi.begin(), rep.xi.end(), xo);
            std::copy(rep.lambda.begin(), rep.lambda.end(), lam_out + b * N * nx);
            std::copy(rep.pi_l.begin(), rep.pi_l.end(), pil_out + b * N);
            std::copy(rep.pi_u.begin(), rep.pi_u.end(), piu_out + b * N);
            converged[b] = rep.converged ? 1 : 0;
            status[b] = 0;
        } catch (const DomainError&) {
            status[b] = NMPCMC_DOMAIN_ERROR;
        } catch (const NonFiniteState&) {
            status[b] = NMPCMC_NON_FINITE_STATE;
        }
    }
    return 0;
}

}  // extern "C"
