// stats_kernel.cuh -- K4: the Monte Carlo statistics on the device.
//
// aggregate_stats (montecarlo.cpp:172-211) and phi_histogram
// (montecarlo.cpp:268-304) over DEVICE-resident records, bitwise equal to the
// reference's host code:
//   * integer totals (n_failed, ocp_solves, ocp_failures) and the stable,
//     index-ordered compaction of the non-failed Φ are exact in any order
//     (CUB DeviceSelect keeps the input order);
//   * the two floating-point sums (Σ Φ for the mean, Σ (Φ - mean)² for the
//     variance) are the reference's serial left-to-right chains: one warp
//     streams the values (coalesced, one chunk ahead), every lane adds the
//     broadcast terms in index order. The products (Φ - mean)² are formed
//     lane-parallel -- the same IEEE product either way;
//   * min / max / deciles / quartiles come from a device radix sort
//     (CUB DeviceRadixSort) and quantile_sorted (montecarlo.cpp:161-168),
//     evaluated with the same IEEE operations (--fmad=false);
//   * the histogram's bin count uses std::cbrt on the host from four scalars
//     (the reference's libm call), then one counting kernel with integer
//     atomics (exact in any order).
// The cost is dominated by the two serial chains: ~8 cycles per sample each,
// ~8 ms per 10^6 samples -- against ~40 min of closed-loop work for 10^6
// NMPC samples on one GPU.
#pragma once

#include <cub/cub.cuh>

#include "nmpcmc_gpu.h"

namespace nmpcmc_dev {
namespace k4 {

/// Exact integer totals of one launch.
struct Totals {
    unsigned long long n_failed;
    unsigned long long n_finite;
    long long ocp_solves;
    long long ocp_failures;
};

/// Per-record flags and integer totals (block partials + one atomic each).
__global__ void totals_kernel(const nmpcmc_sim_record* rec, int64_t n, Totals* tot) {
    unsigned long long nf = 0, nfin = 0;
    long long s = 0, f = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const nmpcmc_sim_record r = rec[i];
        nf += r.failed ? 1 : 0;
        nfin += isfinite(r.phi) ? 1 : 0;
        s += r.ocp_solves;
        f += r.ocp_failures;
    }
    typedef cub::BlockReduce<unsigned long long, 256> BRU;
    typedef cub::BlockReduce<long long, 256> BRL;
    __shared__ union {
        typename BRU::TempStorage u;
        typename BRL::TempStorage l;
    } ts;
    unsigned long long a = BRU(ts.u).Sum(nf);
    __syncthreads();
    unsigned long long b = BRU(ts.u).Sum(nfin);
    __syncthreads();
    long long c = BRL(ts.l).Sum(s);
    __syncthreads();
    long long d = BRL(ts.l).Sum(f);
    if (threadIdx.x == 0) {
        atomicAdd(&tot->n_failed, a);
        atomicAdd(&tot->n_finite, b);
        atomicAdd((unsigned long long*)&tot->ocp_solves, (unsigned long long)c);
        atomicAdd((unsigned long long*)&tot->ocp_failures, (unsigned long long)d);
    }
}

/// Φ of non-failed records (aggregate_stats' `ok`, index order preserved by
/// the stable selection) and of finite records (phi_histogram's `v`).
struct PhiOk {
    const nmpcmc_sim_record* rec;
    __device__ double operator()(int64_t i) const { return rec[i].phi; }
};
struct IsOk {
    const nmpcmc_sim_record* rec;
    __device__ bool operator()(int64_t i) const { return rec[i].failed == 0; }
};
struct IsFinite {
    const nmpcmc_sim_record* rec;
    __device__ bool operator()(int64_t i) const { return isfinite(rec[i].phi) != 0; }
};

/// The serial left-to-right sum of v[0..n) (SQUARE_DEV: of (v - shift)²),
/// exactly the reference's `for (double v : ok) sum += ...` chain. One warp:
/// each lane loads one element of a 32-element chunk (the next chunk is loaded
/// while the current one is summed) and the terms are broadcast in order.
template <bool SQUARE_DEV>
__global__ void __launch_bounds__(32) serial_sum_kernel(const double* v, int64_t n, const double* shift,
                                                        double* out) {
    const int lane = threadIdx.x;
    const double m = SQUARE_DEV ? *shift : 0.0;
    double acc = 0.0;
    auto term = [&](int64_t i) {
        if (i >= n) return 0.0;
        const double x = v[i];
        if (SQUARE_DEV) {
            const double d = x - m;
            return d * d;
        }
        return x;
    };
    double cur = term(lane);
    for (int64_t base = 0; base < n; base += 32) {
        const double nxt = term(base + 32 + lane);
        const int cnt = n - base < 32 ? (int)(n - base) : 32;
#pragma unroll 8
        for (int j = 0; j < cnt; ++j) acc += __shfl_sync(0xffffffffu, cur, j);
        cur = nxt;
    }
    if (lane == 0) *out = acc;
}

/// quantile_sorted (montecarlo.cpp:161-168).
__device__ __forceinline__ double quantile_sorted(const double* s, int64_t n, double q) {
    const double h = q * (double)(n - 1);
    const uint64_t lo = (uint64_t)h;
    if (lo + 1 >= (uint64_t)n) return s[n - 1];
    const double w = h - (double)lo;
    return s[lo] + w * (s[lo + 1] - s[lo]);
}

/// Assemble McAggregate (montecarlo.hpp:95-106) from the totals, the two
/// serial sums and the sorted ok values; also the quartiles / extremes of the
/// sorted finite values for phi_histogram (scal[0..3] = lo, hi, q25, q75).
__global__ void finish_kernel(const Totals* tot, int64_t n, const double* sum, const double* ss,
                              const double* sorted_ok, const double* sorted_fin, nmpcmc_aggregate* agg,
                              double* scal) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    nmpcmc_aggregate a;
    a.n_sims = (int32_t)n;
    a.n_failed = (int32_t)tot->n_failed;
    a.ocp_solves = tot->ocp_solves;
    a.ocp_failures = tot->ocp_failures;
    a.ocp_success_pct = a.ocp_solves > 0 ? 100.0 * (double)(a.ocp_solves - a.ocp_failures) / (double)a.ocp_solves
                                         : 100.0;
    const int64_t n_ok = n - (int64_t)tot->n_failed;
    if (n_ok == 0) {
        a.mean = a.variance = a.min = a.max = nan;
        for (int d = 0; d <= 10; ++d) a.deciles[d] = nan;
    } else {
        a.mean = *sum / (double)n_ok;  // ss was formed with this mean (same division)
        a.variance = n_ok > 1 ? *ss / (double)(n_ok - 1) : 0.0;
        a.min = sorted_ok[0];
        a.max = sorted_ok[n_ok - 1];
        for (int d = 0; d <= 10; ++d) a.deciles[d] = quantile_sorted(sorted_ok, n_ok, d / 10.0);
    }
    *agg = a;
    const int64_t nf = (int64_t)tot->n_finite;
    if (scal != nullptr && nf > 0) {
        scal[0] = sorted_fin[0];
        scal[1] = sorted_fin[nf - 1];
        scal[2] = quantile_sorted(sorted_fin, nf, 0.25);
        scal[3] = quantile_sorted(sorted_fin, nf, 0.75);
    }
}

/// mean = sum / n_ok on the device, the shift of the variance chain.
__global__ void mean_kernel(const Totals* tot, int64_t n, const double* sum, double* mean) {
    const int64_t n_ok = n - (int64_t)tot->n_failed;
    *mean = n_ok > 0 ? *sum / (double)n_ok : 0.0;
}

/// phi_histogram's counting loop (montecarlo.cpp:296-301): exact integer
/// atomics, so the order of the values does not matter.
__global__ void hist_kernel(const double* v, int64_t n, double lo, double width, int bins, int* counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int b = (int)((v[i] - lo) / width);
        b = b < 0 ? 0 : (b > bins - 1 ? bins - 1 : b);
        atomicAdd(&counts[b], 1);
    }
}

}  // namespace k4
}  // namespace nmpcmc_dev
