// host_api.cpp -- host-side parts of the C ABI (include/nmpcmc_gpu.h):
// scenario validation, aggregate statistics and the histogram. These run on
// the per-sample records the kernels produce; they restate the reference's
// serial, index-ordered host code so the aggregate is bitwise what
// aggregate_stats would compute from the same records.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include "nmpcmc_gpu.h"

namespace {

constexpr double kNan = std::numeric_limits<double>::quiet_NaN();

/// quantile_sorted (montecarlo.cpp:161-168).
double quantile_sorted(const std::vector<double>& sorted, double q) {
    if (sorted.empty()) return kNan;
    const double h = q * static_cast<double>(sorted.size() - 1);
    const std::size_t lo = static_cast<std::size_t>(h);
    if (lo + 1 >= sorted.size()) return sorted.back();
    const double w = h - static_cast<double>(lo);
    return sorted[lo] + w * (sorted[lo + 1] - sorted[lo]);
}

}  // namespace

extern "C" {

int nmpcmc_gpu_abi_version(void) { return NMPCMC_GPU_ABI_VERSION; }

int64_t nmpcmc_gpu_struct_size(int which) {
    switch (which) {
        case 0: return sizeof(nmpcmc_scenario);
        case 1: return sizeof(nmpcmc_sim_record);
        case 2: return sizeof(nmpcmc_work_counters);
        case 3: return sizeof(nmpcmc_aggregate);
        default: return -1;
    }
}

/// validate_scenario (montecarlo.cpp:34-63) for the POD scenario, plus the
/// constructor checks the reference performs elsewhere (make_nmpc_state,
/// controllers.cpp:28-34; measure's semidefinite factor, linalg.cpp:80) and
/// what the device path supports.
int nmpcmc_gpu_validate(const nmpcmc_scenario* sc, int32_t* nbar_out) {
    if (sc == nullptr) return NMPCMC_INVALID_ARGUMENT;
    if (sc->Ts <= 0.0) return NMPCMC_DOMAIN_ERROR;
    if (!(sc->tf > sc->t0)) return NMPCMC_DOMAIN_ERROR;
    const double span = sc->tf - sc->t0;
    const int nbar = static_cast<int>(std::llround(span / sc->Ts));
    if (nbar < 1 || std::fabs(nbar * sc->Ts - span) > 1e-9 * std::max(1.0, span))
        return NMPCMC_DOMAIN_ERROR;
    if (sc->Ns < 1) return NMPCMC_DOMAIN_ERROR;
    if (sc->truth_variant != NMPCMC_THREE_STATE && sc->truth_variant != NMPCMC_ONE_STATE)
        return NMPCMC_DOMAIN_ERROR;
    if (sc->n_setpoints < 1 || sc->n_setpoints > NMPCMC_MAX_SETPOINTS) return NMPCMC_DOMAIN_ERROR;
    if (sc->sp_times[0] > sc->t0) return NMPCMC_DOMAIN_ERROR;
    for (int i = 1; i < sc->n_setpoints; ++i)
        if (sc->sp_times[i] < sc->sp_times[i - 1]) return NMPCMC_DOMAIN_ERROR;
    if (sc->has_noise_R) {
        // cholesky_factor_semidefinite throws for a pivot below -tol
        const double tol = 1e-13 * std::max(std::max(0.0, std::fabs(sc->noise_R)), 1.0);
        if (!(std::fabs(sc->noise_R) <= tol) && (sc->noise_R <= 0.0 || !std::isfinite(sc->noise_R)))
            return NMPCMC_NOT_POSITIVE_DEFINITE;
    }
    if (sc->controller == NMPCMC_CTRL_NMPC) {
        if (std::fabs(sc->horizon_Ts - sc->Ts) > 1e-12) return NMPCMC_DOMAIN_ERROR;
        if (sc->N <= 0 || sc->horizon_Ts <= 0.0 || sc->Nc <= 0 || sc->np <= 0)
            return NMPCMC_DOMAIN_ERROR;
        if (sc->ctrl_variant != NMPCMC_ONE_STATE && sc->ctrl_variant != NMPCMC_THREE_STATE)
            return NMPCMC_DOMAIN_ERROR;
        if (sc->N > 4096) return NMPCMC_UNSUPPORTED;  // workspace sanity bound
        if (sc->sqp.max_iter < 0 || sc->sqp.qp_max_iter < 0 || sc->sqp.max_backtracks < 0)
            return NMPCMC_DOMAIN_ERROR;
    } else if (sc->controller == NMPCMC_CTRL_PI) {
        // n_y = n_u = 1 by construction for the CSTR
    } else {
        return NMPCMC_DOMAIN_ERROR;
    }
    if (sc->record_trajectories && sc->record_stride < 1) {
        // run_closed_loop clamps the stride to >= 1 (montecarlo.cpp:103)
    }
    if (nbar_out) *nbar_out = nbar;
    return NMPCMC_OK;
}

int32_t nmpcmc_gpu_traj_rows(const nmpcmc_scenario* sc) {
    int32_t nbar = 0;
    if (nmpcmc_gpu_validate(sc, &nbar) != NMPCMC_OK) return -1;
    const int stride = std::max(1, sc->record_stride);
    return (nbar + stride - 1) / stride + 1;
}

/// aggregate_stats (montecarlo.cpp:172-211).
int nmpcmc_gpu_aggregate(const nmpcmc_sim_record* rec, int64_t n, nmpcmc_aggregate* out) {
    if (rec == nullptr || out == nullptr || n < 0) return NMPCMC_INVALID_ARGUMENT;
    std::memset(out, 0, sizeof *out);
    out->n_sims = static_cast<int32_t>(n);
    std::vector<double> ok;
    ok.reserve(static_cast<std::size_t>(n));
    long long solves = 0, failures = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (rec[i].failed)
            ++out->n_failed;
        else
            ok.push_back(rec[i].phi);
        solves += rec[i].ocp_solves;
        failures += rec[i].ocp_failures;
    }
    out->ocp_solves = solves;
    out->ocp_failures = failures;
    out->ocp_success_pct =
        solves > 0 ? 100.0 * static_cast<double>(solves - failures) / static_cast<double>(solves)
                   : 100.0;
    if (ok.empty()) {
        out->mean = out->variance = out->min = out->max = kNan;
        for (double& d : out->deciles) d = kNan;
        return NMPCMC_OK;
    }
    double sum = 0.0;
    for (double v : ok) sum += v;
    out->mean = sum / static_cast<double>(ok.size());
    double ss = 0.0;
    for (double v : ok) ss += (v - out->mean) * (v - out->mean);
    out->variance = ok.size() > 1 ? ss / static_cast<double>(ok.size() - 1) : 0.0;
    std::vector<double> sorted = ok;
    std::sort(sorted.begin(), sorted.end());
    out->min = sorted.front();
    out->max = sorted.back();
    for (int d = 0; d <= 10; ++d) out->deciles[d] = quantile_sorted(sorted, d / 10.0);
    return NMPCMC_OK;
}

/// phi_histogram (montecarlo.cpp:268-304), Freedman-Diaconis when bins <= 0.
int nmpcmc_gpu_histogram(const double* phi, int64_t n, int32_t bins, double* edges,
                         int32_t* counts, int32_t* nbins_out) {
    if (phi == nullptr || edges == nullptr || counts == nullptr || nbins_out == nullptr)
        return NMPCMC_INVALID_ARGUMENT;
    if (bins > 200) return NMPCMC_INVALID_ARGUMENT;  // output arrays hold 200 bins
    std::vector<double> v;
    v.reserve(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i)
        if (std::isfinite(phi[i])) v.push_back(phi[i]);
    if (v.empty()) {
        edges[0] = 0.0;
        edges[1] = 1.0;
        counts[0] = 0;
        *nbins_out = 1;
        return NMPCMC_OK;
    }
    std::sort(v.begin(), v.end());
    const double lo = v.front(), hi = v.back();
    if (bins <= 0) {
        const double iqr = quantile_sorted(v, 0.75) - quantile_sorted(v, 0.25);
        const double width = 2.0 * iqr / std::cbrt(static_cast<double>(v.size()));
        bins = width > 0.0 ? static_cast<int>(std::ceil((hi - lo) / width)) : 1;
        bins = std::clamp(bins, 1, 200);
    }
    if (hi <= lo) {
        edges[0] = lo;
        edges[1] = lo + 1.0;
        counts[0] = static_cast<int32_t>(v.size());
        *nbins_out = 1;
        return NMPCMC_OK;
    }
    const double width = (hi - lo) / bins;
    for (int b = 0; b <= bins; ++b) edges[b] = lo + b * width;
    edges[bins] = hi;
    for (int b = 0; b < bins; ++b) counts[b] = 0;
    for (double x : v) {
        int b = static_cast<int>((x - lo) / width);
        b = std::clamp(b, 0, bins - 1);
        ++counts[b];
    }
    *nbins_out = bins;
    return NMPCMC_OK;
}

}  // extern "C"
