// nmpcmc_gpu.hpp -- C++ facade with the reference's names and result types
// over the C ABI (nmpcmc_gpu.h). Header-only; link libnmpcmc_gpu.so.
//
// A caller of the reference (/root/reference/proj/core/include/nmpcmc/montecarlo.hpp)
//     nmpcmc::McResult r = nmpcmc::run_monte_carlo(scenario, n_sims, workers);
// switches to
//     nmpcmc::gpu::McResult r = nmpcmc::gpu::run_monte_carlo(gpu_scenario, n_sims);
// where gpu_scenario carries the CSTR parameters explicitly (the reference's
// Scenario holds std::function models the GPU cannot use, model.hpp:28-46).
// Field-by-field mapping: INTEGRATION.md.
#pragma once

#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "nmpcmc_gpu.h"

namespace nmpcmc {
namespace gpu {

using Scenario = nmpcmc_scenario;

/// Exception classes of errors.hpp:9-32, thrown from status codes.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};
struct DimensionMismatch : Error { using Error::Error; };
struct NotPositiveDefinite : Error { using Error::Error; };
struct NonFiniteState : Error { using Error::Error; };
struct DomainError : Error { using Error::Error; };
struct LengthMismatch : Error { using Error::Error; };

inline void check(int rc, const char* what, const nmpcmc_gpu_ctx* ctx = nullptr) {
    if (rc == NMPCMC_OK) return;
    std::string msg = std::string(what) + ": " + (ctx ? nmpcmc_gpu_last_error(ctx) : "status " + std::to_string(rc));
    switch (rc) {
        case NMPCMC_DIMENSION_MISMATCH: throw DimensionMismatch(rc, msg);
        case NMPCMC_NOT_POSITIVE_DEFINITE: throw NotPositiveDefinite(rc, msg);
        case NMPCMC_NON_FINITE_STATE: throw NonFiniteState(rc, msg);
        case NMPCMC_DOMAIN_ERROR: throw DomainError(rc, msg);
        case NMPCMC_LENGTH_MISMATCH: throw LengthMismatch(rc, msg);
        default: throw Error(rc, msg);
    }
}

/// SimResult (montecarlo.hpp:72-79), trajectory omitted.
struct SimResult {
    std::uint64_t sim_index = 0;
    double phi = 0.0;
    bool failed = false;
    int ocp_solves = 0;
    int ocp_failures = 0;
};

/// McAggregate (montecarlo.hpp:95-106).
struct McAggregate {
    int n_sims = 0, n_failed = 0;
    double mean = 0.0, variance = 0.0, min = 0.0, max = 0.0;
    std::vector<double> deciles;
    long long ocp_solves = 0, ocp_failures = 0;
    double ocp_success_pct = 100.0;
};

/// McResult (montecarlo.hpp:112-116).
struct McResult {
    std::vector<SimResult> sims;
    McAggregate aggregate;
    double wall_seconds = 0.0;
};

/// Histogram (montecarlo.hpp:136-141).
struct Histogram {
    std::vector<double> edges;
    std::vector<int> counts;
};

/// RAII device context: one GPU and one stream, or -- from a list of device
/// ids -- one sub-context per GPU with NCCL between them
/// (nmpcmc_gpu_ctx_create_multi). The multi-device form replaces the worker
/// pool of run_monte_carlo (montecarlo.cpp:218-245).
class Context {
public:
    explicit Context(int device = 0) { check(nmpcmc_gpu_ctx_create(device, &ctx_), "ctx_create"); }
    explicit Context(const std::vector<int>& device_ids) {
        if (device_ids.empty()) throw DomainError(NMPCMC_DOMAIN_ERROR, "Context: no device ids");
        check(nmpcmc_gpu_ctx_create_multi(device_ids.data(), static_cast<int>(device_ids.size()), &ctx_),
              "ctx_create_multi");
    }
    int num_devices() const { return nmpcmc_gpu_ctx_num_devices(ctx_); }
    ~Context() { nmpcmc_gpu_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    nmpcmc_gpu_ctx* get() const { return ctx_; }

private:
    nmpcmc_gpu_ctx* ctx_ = nullptr;
};

/// validate_scenario (montecarlo.cpp:34-63): N_bar.
inline int validate_scenario(const Scenario& sc) {
    int32_t nbar = 0;
    check(nmpcmc_gpu_validate(&sc, &nbar), "validate_scenario");
    return nbar;
}

inline McAggregate to_aggregate(const nmpcmc_aggregate& a) {
    McAggregate out;
    out.n_sims = a.n_sims;
    out.n_failed = a.n_failed;
    out.mean = a.mean;
    out.variance = a.variance;
    out.min = a.min;
    out.max = a.max;
    out.deciles.assign(a.deciles, a.deciles + 11);
    out.ocp_solves = a.ocp_solves;
    out.ocp_failures = a.ocp_failures;
    out.ocp_success_pct = a.ocp_success_pct;
    return out;
}

inline McAggregate aggregate_stats(const std::vector<nmpcmc_sim_record>& rec) {
    nmpcmc_aggregate a{};
    check(nmpcmc_gpu_aggregate(rec.data(), static_cast<int64_t>(rec.size()), &a), "aggregate_stats");
    return to_aggregate(a);
}

/// run_monte_carlo (montecarlo.cpp:213-251) for samples [first, first + n).
/// On a multi-device context the samples are sharded by global index over
/// the GPUs and the aggregate is computed on device_ids[0] after the NCCL
/// gather (K4); records are bitwise independent of the device count.
inline McResult run_monte_carlo(Context& ctx, const Scenario& sc, int n_sims, std::uint64_t first = 0) {
    if (n_sims < 1) throw DomainError(NMPCMC_DOMAIN_ERROR, "run_monte_carlo: n_sims must be at least 1");
    std::vector<nmpcmc_sim_record> rec(static_cast<std::size_t>(n_sims));
    nmpcmc_aggregate a{};
    const auto t0 = std::chrono::steady_clock::now();
    check(nmpcmc_gpu_run(ctx.get(), &sc, first, n_sims, rec.data(), nullptr, &a), "run_monte_carlo", ctx.get());
    McResult r;
    r.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    r.sims.resize(rec.size());
    for (std::size_t i = 0; i < rec.size(); ++i) {
        r.sims[i].sim_index = first + i;
        r.sims[i].phi = rec[i].phi;
        r.sims[i].failed = rec[i].failed != 0;
        r.sims[i].ocp_solves = rec[i].ocp_solves;
        r.sims[i].ocp_failures = rec[i].ocp_failures;
    }
    r.aggregate = to_aggregate(a);
    return r;
}

/// The reference's signature run_monte_carlo(sc, n_sims, workers)
/// (montecarlo.hpp:121) with the worker count read as a GPU count: devices
/// 0 .. n_devices-1 of this process (0 = every visible device).
inline McResult run_monte_carlo(const Scenario& sc, int n_sims, int n_devices = 0) {
    if (n_devices <= 0) check(nmpcmc_gpu_device_count(&n_devices), "device_count");
    if (n_devices <= 0) throw Error(NMPCMC_CUDA_ERROR, "run_monte_carlo: no CUDA device");
    std::vector<int> ids(static_cast<std::size_t>(n_devices));
    for (int i = 0; i < n_devices; ++i) ids[static_cast<std::size_t>(i)] = i;
    Context ctx(ids);
    return run_monte_carlo(ctx, sc, n_sims);
}

/// run_closed_loop (montecarlo.cpp:80-157) for one global sample index.
inline SimResult run_closed_loop(Context& ctx, const Scenario& sc, std::uint64_t sim_index) {
    return run_monte_carlo(ctx, sc, 1, sim_index).sims.front();
}

/// QpStageData (qp.hpp:24-30), matrices column-major (M is n_x x n_u). The
/// members a stage does not use may stay empty (stage 0: Q M q Jx; stage N:
/// all but Q q).
struct QpStage {
    std::vector<double> Q, M, R, q, r, Jx, Ju, b, lb, ub;
};
/// QpSolution (qp.hpp:34-41); status: NMPCMC_QP_OPTIMAL / MAXITER / FAILED, or
/// NMPCMC_QP_DOMAIN_ERROR / NMPCMC_QP_NOT_POSITIVE_DEFINITE where the
/// reference throws.
struct QpSolution {
    std::vector<double> delta_xi, mu, nu_l, nu_u;
    int iterations = 0;
    int status = NMPCMC_QP_FAILED;
};

/// solve_qp (qp.hpp:52-56) -- or riccati_factor_solve (qp.hpp:42-45) with
/// riccati_only -- for a batch of stagewise QPs of equal dimensions.
inline std::vector<QpSolution> solve_qp_batch(Context& ctx, const std::vector<std::vector<QpStage>>& qps, int n_x,
                                              int n_u, double tol = 1e-10, int max_iter = 50,
                                              bool riccati_only = false) {
    if (qps.empty()) return {};
    const int N = static_cast<int>(qps.front().size()) - 1;
    const int64_t SB = nmpcmc_qp_stage_doubles(n_x, n_u), SO = nmpcmc_qp_solution_doubles(N, n_x, n_u);
    std::vector<double> packed(qps.size() * static_cast<std::size_t>((N + 1) * SB), 0.0);
    const int sizes[10] = {n_x * n_x, n_x * n_u, n_u * n_u, n_x, n_u, n_x * n_x, n_x * n_u, n_x, n_u, n_u};
    for (std::size_t bi = 0; bi < qps.size(); ++bi) {
        if (static_cast<int>(qps[bi].size()) != N + 1)
            throw DimensionMismatch(NMPCMC_DIMENSION_MISMATCH, "solve_qp_batch: unequal stage counts");
        for (int k = 0; k <= N; ++k) {
            const QpStage& st = qps[bi][k];
            const std::vector<double>* parts[10] = {&st.Q, &st.M, &st.R, &st.q, &st.r,
                                                    &st.Jx, &st.Ju, &st.b, &st.lb, &st.ub};
            double* dst = packed.data() + (bi * (N + 1) + k) * SB;
            for (int m = 0; m < 10; ++m) {
                if (!parts[m]->empty()) {
                    if (static_cast<int>(parts[m]->size()) != sizes[m])
                        throw DimensionMismatch(NMPCMC_DIMENSION_MISMATCH, "solve_qp_batch: block size");
                    std::copy(parts[m]->begin(), parts[m]->end(), dst);
                }
                dst += sizes[m];
            }
        }
    }
    const nmpcmc_qp_dims d{N, n_x, n_u, max_iter, tol, riccati_only ? 1 : 0, 0};
    std::vector<double> sol(qps.size() * static_cast<std::size_t>(SO));
    std::vector<int32_t> status(qps.size()), iters(qps.size());
    check(nmpcmc_gpu_solve_qp_batch(ctx.get(), &d, static_cast<int64_t>(qps.size()), packed.data(), sol.data(),
                                    status.data(), iters.data()),
          "solve_qp_batch", ctx.get());
    std::vector<QpSolution> out(qps.size());
    const int L = N * (n_u + n_x), NX = N * n_x, NV = N * n_u;
    for (std::size_t bi = 0; bi < qps.size(); ++bi) {
        const double* s = sol.data() + bi * SO;
        out[bi].delta_xi.assign(s, s + L);
        out[bi].mu.assign(s + L, s + L + NX);
        out[bi].nu_l.assign(s + L + NX, s + L + NX + NV);
        out[bi].nu_u.assign(s + L + NX + NV, s + L + NX + 2 * NV);
        out[bi].iterations = iters[bi];
        out[bi].status = status[bi];
    }
    return out;
}

/// SqpReport (sqp.hpp:79-90) of one OCP instance.
struct OcpSolution {
    std::vector<double> xi, lambda, pi_l, pi_u;
    bool converged = false;
    int status = 0;  // NMPCMC_DOMAIN_ERROR if a DomainError escaped
};

/// sqp_solve (sqp.hpp:148-151) on the regulator OcpProblem of sc's controller
/// model for each (x0[b], t0[b]); x0 holds n_x entries per instance. Cold
/// start as nmpc_step unless xi0 (L entries per instance) is given.
inline std::vector<OcpSolution> solve_ocp_batch(Context& ctx, const Scenario& sc, const std::vector<double>& x0,
                                                const std::vector<double>& t0,
                                                const std::vector<double>* xi0 = nullptr) {
    const int nx = sc.ctrl_variant == NMPCMC_THREE_STATE ? 3 : 1, N = sc.N, L = N * (1 + nx);
    const std::size_t B = t0.size();
    if (x0.size() != B * nx || (xi0 && xi0->size() != B * L))
        throw LengthMismatch(NMPCMC_LENGTH_MISMATCH, "solve_ocp_batch: input lengths");
    std::vector<double> xi(B * L), lam(B * N * nx), pil(B * N), piu(B * N);
    std::vector<int32_t> conv(B), st(B);
    check(nmpcmc_gpu_solve_ocp_batch(ctx.get(), &sc, static_cast<int64_t>(B), x0.data(), t0.data(),
                                     xi0 ? xi0->data() : nullptr, xi.data(), lam.data(), pil.data(), piu.data(),
                                     conv.data(), st.data()),
          "solve_ocp_batch", ctx.get());
    std::vector<OcpSolution> out(B);
    for (std::size_t b = 0; b < B; ++b) {
        out[b].xi.assign(xi.begin() + b * L, xi.begin() + (b + 1) * L);
        out[b].lambda.assign(lam.begin() + b * N * nx, lam.begin() + (b + 1) * N * nx);
        out[b].pi_l.assign(pil.begin() + b * N, pil.begin() + (b + 1) * N);
        out[b].pi_u.assign(piu.begin() + b * N, piu.begin() + (b + 1) * N);
        out[b].converged = conv[b] != 0;
        out[b].status = st[b];
    }
    return out;
}

/// pi_step (controllers.hpp:49) for a batch of PI controllers; states advance
/// to result.next in place.
inline std::vector<nmpcmc_pi_step_result> pi_step_batch(Context& ctx, std::vector<nmpcmc_pi_state>& states,
                                                        const std::vector<double>& y,
                                                        const std::vector<double>& y_bar) {
    if (y.size() != states.size() || y_bar.size() != states.size())
        throw LengthMismatch(NMPCMC_LENGTH_MISMATCH, "pi_step_batch: input lengths");
    std::vector<nmpcmc_pi_step_result> r(states.size());
    check(nmpcmc_gpu_pi_step_batch(ctx.get(), states.data(), y.data(), y_bar.data(),
                                   static_cast<int64_t>(states.size()), r.data()),
          "pi_step_batch", ctx.get());
    return r;
}

/// B device-resident NmpcStates (make_nmpc_state, controllers.hpp:84-86) of
/// the scenario's controller configuration; step() is nmpc_step
/// (controllers.hpp:92-93) on every instance.
class NmpcBatch {
public:
    NmpcBatch(Context& ctx, const Scenario& sc, int64_t batch, const std::vector<double>* x0_hat = nullptr,
              const std::vector<double>* P0 = nullptr)
        : ctx_(ctx), batch_(batch), N_(sc.N) {
        check(nmpcmc_gpu_nmpc_batch_create(ctx.get(), &sc, batch, x0_hat ? x0_hat->data() : nullptr,
                                           P0 ? P0->data() : nullptr, &st_),
              "make_nmpc_state", ctx.get());
    }
    ~NmpcBatch() { nmpcmc_gpu_nmpc_batch_destroy(st_); }
    NmpcBatch(const NmpcBatch&) = delete;
    NmpcBatch& operator=(const NmpcBatch&) = delete;
    /// Applied inputs (NaN where nmpc_step threw; diag[b].status says which).
    std::vector<double> step(const std::vector<double>& t, const std::vector<double>& y,
                             std::vector<nmpcmc_nmpc_diag>* diag = nullptr,
                             const std::vector<double>* setpoints = nullptr) {
        if (static_cast<int64_t>(t.size()) != batch_ || static_cast<int64_t>(y.size()) != batch_ ||
            (setpoints && static_cast<int64_t>(setpoints->size()) != batch_ * N_))
            throw LengthMismatch(NMPCMC_LENGTH_MISMATCH, "nmpc_step: input lengths");
        std::vector<double> u(static_cast<std::size_t>(batch_));
        if (diag) diag->resize(static_cast<std::size_t>(batch_));
        check(nmpcmc_gpu_nmpc_step_batch(ctx_.get(), st_, t.data(), y.data(), setpoints ? setpoints->data() : nullptr,
                                         u.data(), diag ? diag->data() : nullptr),
              "nmpc_step", ctx_.get());
        return u;
    }
    nmpcmc_nmpc_batch* get() const { return st_; }

private:
    Context& ctx_;
    int64_t batch_;
    int N_;
    nmpcmc_nmpc_batch* st_ = nullptr;
};

/// phi_histogram (montecarlo.cpp:268-304).
inline Histogram phi_histogram(const std::vector<double>& phi, int bins = 0) {
    std::vector<double> edges(201);
    std::vector<int32_t> counts(200);
    int32_t nb = 0;
    check(nmpcmc_gpu_histogram(phi.data(), static_cast<int64_t>(phi.size()), bins, edges.data(), counts.data(), &nb),
          "phi_histogram");
    Histogram h;
    h.edges.assign(edges.begin(), edges.begin() + nb + 1);
    h.counts.assign(counts.begin(), counts.begin() + nb);
    return h;
}

}  // namespace gpu
}  // namespace nmpcmc
