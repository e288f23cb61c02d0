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

/// RAII device context (one GPU, one stream).
class Context {
public:
    explicit Context(int device = 0) { check(nmpcmc_gpu_ctx_create(device, &ctx_), "ctx_create"); }
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

inline McAggregate aggregate_stats(const std::vector<nmpcmc_sim_record>& rec) {
    nmpcmc_aggregate a{};
    check(nmpcmc_gpu_aggregate(rec.data(), static_cast<int64_t>(rec.size()), &a), "aggregate_stats");
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

/// run_monte_carlo (montecarlo.cpp:213-251) for samples [first, first + n).
inline McResult run_monte_carlo(Context& ctx, const Scenario& sc, int n_sims, std::uint64_t first = 0) {
    if (n_sims < 1) throw DomainError(NMPCMC_DOMAIN_ERROR, "run_monte_carlo: n_sims must be at least 1");
    std::vector<nmpcmc_sim_record> rec(static_cast<std::size_t>(n_sims));
    check(nmpcmc_gpu_run(ctx.get(), &sc, first, n_sims, rec.data(), nullptr, nullptr), "run_monte_carlo",
          ctx.get());
    McResult r;
    r.sims.resize(rec.size());
    for (std::size_t i = 0; i < rec.size(); ++i) {
        r.sims[i].sim_index = first + i;
        r.sims[i].phi = rec[i].phi;
        r.sims[i].failed = rec[i].failed != 0;
        r.sims[i].ocp_solves = rec[i].ocp_solves;
        r.sims[i].ocp_failures = rec[i].ocp_failures;
    }
    r.aggregate = aggregate_stats(rec);
    return r;
}

/// run_closed_loop (montecarlo.cpp:80-157) for one global sample index.
inline SimResult run_closed_loop(Context& ctx, const Scenario& sc, std::uint64_t sim_index) {
    return run_monte_carlo(ctx, sc, 1, sim_index).sims.front();
}

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
