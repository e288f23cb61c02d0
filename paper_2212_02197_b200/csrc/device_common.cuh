// device_common.cuh -- per-sample device building blocks shared by the PI
// and NMPC closed-loop kernels: Philox4x32-10 + Box-Muller stream, the CSTR
// SDE model, setpoint lookup, Euler-Maruyama plant, measurement.
//
// Every function restates one reference routine with the reference's exact
// floating-point operation order (compiled with --fmad=false, so nothing is
// contracted). The "1.0*s + 1.0*y" and "0.0 + a*b" forms are kept where the
// reference's gemm/gemv epilogue produces them (linalg.cpp:156-161,186-187):
// they differ from the bare product only in the sign of zero, but that is
// cheap to keep and makes the restatement auditable line by line.
#pragma once

#include <stdint.h>

#include "nmpcmc_gpu.h"
#include "xlibm.h"

namespace nmpcmc_dev {

// ---------------------------------------------------------------- status
// Per-sample failure codes (nmpcmc_status); 0 = running.
enum : int {
    ST_OK = 0,
    ST_NPD = NMPCMC_NOT_POSITIVE_DEFINITE,
    ST_NONFINITE = NMPCMC_NON_FINITE_STATE,
    ST_DOMAIN = NMPCMC_DOMAIN_ERROR,
};

__device__ __forceinline__ bool dfinite(double x) { return isfinite(x); }

// std::max / std::min exactly as libstdc++ defines them (a<b ? b : a), which
// fixes the NaN and signed-zero behaviour.
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }

// gemm/gemv epilogue (linalg.cpp:161,187): alpha*s + (beta==0 ? 0 : beta*c)
// for the 1x1 products that occur with alpha = +-1, beta in {0, 1}.
__device__ __forceinline__ double dot1(double a, double b) { return 0.0 + a * b; }
__device__ __forceinline__ double epi0(double s) { return 1.0 * s + 0.0; }
__device__ __forceinline__ double epi1(double s, double c) { return 1.0 * s + 1.0 * c; }
__device__ __forceinline__ double epim1(double s, double c) { return -1.0 * s + 1.0 * c; }

// ------------------------------------------------------------- Philox RNG
// CounterRng::philox_block (rng.cpp:31-43), constants rng.cpp:10-13.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

/// CounterRng (rng.hpp:18-48) restricted to normal(): every Box-Muller pair
/// consumes exactly one Philox block (two uniforms of two words each), so the
/// stream is (block index, cached spare) -- SURVEY.md Appendix A.5.
struct NormalStream {
    uint64_t seed;
    uint64_t stream;
    uint64_t block;
    double spare;
    bool have_spare;

    __device__ void init(uint64_t seed_, uint64_t stream_) {
        seed = seed_;
        stream = stream_;
        block = 0;
        spare = 0.0;
        have_spare = false;
    }

    /// rng.cpp:78-91: u1 = 1 - U, u2 = U, r = sqrt(-2 ln u1), a = 2 pi u2,
    /// return r cos a, cache r sin a (GCC emits one sincos call).
    __device__ __noinline__ double normal() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        const uint4 ctr = make_uint4((uint32_t)block, (uint32_t)(block >> 32), (uint32_t)stream,
                                     (uint32_t)(stream >> 32));
        const uint4 b = philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
        ++block;
        const uint64_t w0 = ((uint64_t)b.x << 32) | b.y;  // next_u64: high word first
        const uint64_t w1 = ((uint64_t)b.z << 32) | b.w;
        const double U0 = (double)(w0 >> 11) * 0x1.0p-53;
        const double U1 = (double)(w1 >> 11) * 0x1.0p-53;
        const double u1 = 1.0 - U0;
        const double u2 = U1;
        const double radius = sqrt(-2.0 * xlibm_log(u1));
        const double angle = 0x1.921fb54442d18p+2 * u2;  // 2.0 * std::numbers::pi folded
        double s, c;
        xlibm_sincos(angle, &s, &c);
        spare = radius * s;
        have_spare = true;
        return radius * c;
    }
};

/// Box-Muller pair p of stream (seed, stream) -- the two normals
/// NormalStream::normal() returns from Philox block p (rng.cpp:78-91):
/// c = r cos a (returned first), s = r sin a (the cached spare).
__device__ __forceinline__ void normal_pair(uint64_t seed, uint64_t stream, uint64_t p, double& c, double& s) {
    const uint4 ctr = make_uint4((uint32_t)p, (uint32_t)(p >> 32), (uint32_t)stream, (uint32_t)(stream >> 32));
    const uint4 b = philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t w0 = ((uint64_t)b.x << 32) | b.y;
    const uint64_t w1 = ((uint64_t)b.z << 32) | b.w;
    const double u1 = 1.0 - (double)(w0 >> 11) * 0x1.0p-53;
    const double u2 = (double)(w1 >> 11) * 0x1.0p-53;
    const double radius = sqrt(-2.0 * xlibm_log(u1));
    const double angle = 0x1.921fb54442d18p+2 * u2;
    double sn, cs;
    xlibm_sincos(angle, &sn, &cs);
    s = radius * sn;
    c = radius * cs;
}

/// Normal n of stream (seed, stream) alone: component n & 1 of pair n >> 1
/// (c for even n, s for odd n), bitwise the value normal_pair produces for
/// it -- only the needed half of the sincos is kept.
__device__ __forceinline__ double normal_one(uint64_t seed, uint64_t stream, uint64_t n) {
    const uint64_t p = n >> 1;
    const uint4 ctr = make_uint4((uint32_t)p, (uint32_t)(p >> 32), (uint32_t)stream, (uint32_t)(stream >> 32));
    const uint4 b = philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t w0 = ((uint64_t)b.x << 32) | b.y;
    const uint64_t w1 = ((uint64_t)b.z << 32) | b.w;
    const double u1 = 1.0 - (double)(w0 >> 11) * 0x1.0p-53;
    const double u2 = (double)(w1 >> 11) * 0x1.0p-53;
    const double radius = sqrt(-2.0 * xlibm_log(u1));
    const double angle = 0x1.921fb54442d18p+2 * u2;
    return radius * ((n & 1) ? xlibm_sin(angle) : xlibm_cos(angle));
}

/// W consecutive pairs from pair0 into buf (element j at buf[j * stride]):
/// W independent Philox / log / sincos chains, so they overlap (ILP).
template <int W>
__device__ __noinline__ void fill_normal_pairs(double* buf, int stride, uint64_t seed, uint64_t stream,
                                               uint64_t pair0) {
#pragma unroll
    for (int j = 0; j < W; ++j) {
        double c, s;
        normal_pair(seed, stream, pair0 + j, c, s);
        buf[(2 * j) * stride] = c;
        buf[(2 * j + 1) * stride] = s;
    }
}

/// The normal stream of NormalStream, consumed through a window of W pairs
/// generated ahead (fill_normal_pairs) instead of one pair per call: the same
/// sequence bit for bit (normal k is component k & 1 of pair k >> 1), but
/// the generation leaves the plant's serial Euler-Maruyama chain.
///
/// G > 1: the window is shared by a group of G consecutive lanes that run the
/// same sample in lockstep (every lane holds the same k); lane r of the group
/// generates pairs r, r + G, ... of each refill, so a refill costs each lane
/// W / G chains. Refills must be warp-uniform (the caller keeps every group
/// of the warp at the same k at each refill point): __syncwarp of the whole
/// warp orders the shared-memory windows without splitting it.
template <int W, int G = 1>
struct NormalWindow {
    double* buf;
    int stride;
    uint64_t seed, stream;
    uint64_t base;  // normal index of buf[0] (even)
    uint64_t k;     // next normal index
    unsigned gmask; // lanes that refill together (the whole warp)
    int r;          // rank in the group
    __device__ void fill(uint64_t pair0) {
        if (G == 1) {
            fill_normal_pairs<W>(buf, stride, seed, stream, pair0);
            return;
        }
        __syncwarp(gmask);  // every lane of the group is done reading the old window
#pragma unroll
        for (int j = 0; j < W; j += G) {
            double c, s;
            normal_pair(seed, stream, pair0 + j + r, c, s);
            buf[(2 * (j + r)) * stride] = c;
            buf[(2 * (j + r) + 1) * stride] = s;
        }
        __syncwarp(gmask);
    }
    __device__ void init(double* b, int st, uint64_t seed_, uint64_t stream_) {
        buf = b;
        stride = st;
        seed = seed_;
        stream = stream_;
        k = 0;
        base = 0;
        r = G == 1 ? 0 : (int)(threadIdx.x & (G - 1));
        gmask = 0xffffffffu;
        fill(0);
    }
    /// One control step's refill when only some of its normals are read: the
    /// measurement normal k0 (has_R) and the third of every plant substep's
    /// three, k0 + has_R + 3 j + 2 (the three-state plant with zero diffusion
    /// on c_A, c_B: simulate_interval<NX, true>). The others are skipped
    /// (skip()), never read. Needs has_R + 3 ns <= 2W - 1. Warp-uniform.
    __device__ void fill_sparse(uint64_t k0, int has_R, int ns) {
        k = k0;
        base = k0 & ~1ULL;
        if (G > 1) __syncwarp(gmask);
        const int count = has_R + ns;
#pragma unroll 4
        for (int m = r; m < count; m += G) {
            const uint64_t n = (has_R && m == 0) ? k0 : k0 + (uint64_t)(has_R + 3 * (m - has_R) + 2);
            buf[(int)(n - base) * stride] = normal_one(seed, stream, n);
        }
        if (G > 1) __syncwarp(gmask);
    }
    __device__ __forceinline__ void skip() { ++k; }
    /// make normals k .. k+m-1 resident (m <= 2W - 1) with at most one refill
    __device__ __forceinline__ void reserve(int m) {
        if (k + (uint64_t)m > base + 2 * W) {
            base = k & ~1ULL;
            fill(base >> 1);
        }
    }
    __device__ __forceinline__ double normal() {
        if (k >= base + 2 * W) {
            base = k & ~1ULL;
            fill(base >> 1);
        }
        const double z = buf[(int)(k - base) * stride];
        ++k;
        return z;
    }
};

// ------------------------------------------------------------ CSTR model
constexpr double kMlMinToLs = 1e-3 / 60.0;  // cstr.hpp:46

struct Cstr {
    double V, k0, EaR, beta, cA_in, cB_in, cT_in, sigmaA, sigmaB, sigmaT;
};

__device__ __forceinline__ Cstr load_cstr(const nmpcmc_cstr_params& p) {
    return Cstr{p.V, p.k0, p.EaR, p.beta, p.cA_in, p.cB_in, p.cT_in, p.sigmaA, p.sigmaB, p.sigmaT};
}

/// Per-sample truth parameters (include/nmpcmc_gpu.h perturbation rule).
__device__ __forceinline__ Cstr sample_truth(const nmpcmc_scenario& sc, uint64_t sim_index) {
    Cstr p = load_cstr(sc.truth);
    if (sc.perturb) {
        NormalStream prng;
        prng.init(sc.base_seed, sim_index | 0x8000000000000000ULL);
        const double z0 = prng.normal();
        const double z1 = prng.normal();
        const double z2 = prng.normal();
        p.cA_in = p.cA_in * (1.0 + sc.perturb_rel_std[0] * z0);
        p.cB_in = p.cB_in * (1.0 + sc.perturb_rel_std[1] * z1);
        p.EaR = p.EaR * (1.0 + sc.perturb_rel_std[2] * z2);
    }
    return p;
}

/// Three-state drift cstr_drift (cstr.cpp:42-53) with reaction_rate
/// (cstr.cpp:36-40). Returns ST_DOMAIN when c_T <= 0 (cstr.cpp:38).
__device__ __forceinline__ int drift3(const Cstr& p, const double n[3], double u, double dn[3]) {
    const double f = u * kMlMinToLs;
    const double c0 = n[0] / p.V, c1 = n[1] / p.V, c2 = n[2] / p.V;
    if (c2 <= 0.0) return ST_DOMAIN;
    const double r = p.k0 * xlibm_exp(-p.EaR / c2) * c0 * c1;
    dn[0] = p.cA_in * f - c0 * f + -1.0 * r * p.V;
    dn[1] = p.cB_in * f - c1 * f + -2.0 * r * p.V;
    dn[2] = p.cT_in * f - c2 * f + p.beta * r * p.V;
    return ST_OK;
}

/// One-state reduction concentrations (cstr.cpp:13-17).
struct Conc1 {
    double cA, cB, cT;
};
__device__ __forceinline__ Conc1 conc1(const Cstr& p, double cT) {
    return Conc1{p.cA_in - (cT - p.cT_in) / p.beta, p.cB_in - 2.0 * (cT - p.cT_in) / p.beta, cT};
}

/// One-state drift (cstr.cpp:42-53, variant one_state).
__device__ __forceinline__ int drift1(const Cstr& p, double n, double u, double* dn) {
    const double f = u * kMlMinToLs;
    const double c = n / p.V;
    const Conc1 cc = conc1(p, c);
    if (cc.cT <= 0.0) return ST_DOMAIN;
    const double r = p.k0 * xlibm_exp(-p.EaR / cc.cT) * cc.cA * cc.cB;
    *dn = p.cT_in * f - c * f + p.beta * r * p.V;
    return ST_OK;
}

// ------------------------------------------------------------- setpoints
/// SetpointProfile::at (montecarlo.cpp:26-32): values[upper_bound(t) - 1].
/// Validation guarantees times[0] <= t for every query.
__device__ __forceinline__ double setpoint_at(const nmpcmc_scenario& sc, double t) {
    int idx = 0;
    while (idx < sc.n_setpoints && !(t < sc.sp_times[idx])) ++idx;
    return sc.sp_values[idx - 1];
}

// ------------------------------------------------------------ plant loop
/// cholesky_factor_semidefinite of the 1x1 R (linalg.cpp:69-103, tol :80).
/// Host validation rejects R < -tol, so the throwing branch cannot occur.
__device__ __forceinline__ double chol_semidef_1x1(double R) {
    const double scale = smax(0.0, fabs(R));
    const double tol = 1e-13 * smax(scale, 1.0);
    const double d = R;
    if (fabs(d) <= tol) return 0.0;
    return sqrt(d);
}

/// Truth state for either variant; n_x = 3 or 1.
template <int NX>
struct Plant {
    double x[NX];
};

/// measure (model.cpp:39-48): y = g(x) + L_R zeta, one normal per call when R
/// has rows; g = x_T / V (cstr.cpp:86-89).
template <int NX, class Rng>
__device__ __forceinline__ double measure(const Cstr& p, const Plant<NX>& pl, bool has_R, double lR, Rng& rng) {
    double y = pl.x[NX - 1] / p.V;
    if (has_R) {
        const double zeta = rng.normal();
        y = epi1(dot1(lR, zeta), y);
    }
    return y;
}

/// simulate_interval (model.cpp:26-37) + euler_maruyama_step (model.cpp:13-24)
/// for the CSTR (diffusion diag(F sigma_bar), cstr.cpp:55-65). Returns a status.
/// SPARSE (NX = 3, sigma_A = sigma_B = 0): the c_A, c_B increments are not
/// drawn but skipped and taken as 0. Bitwise the same states: in the gemv
/// below their terms are (+-0) * dw in every row, the row sums start at +0.0,
/// and +0 + (+-0) = +0, so no row depends on dw_A or dw_B.
/// simulate_interval_d: the same with the drift supplied by the caller,
/// drift(x, u, dn) -> status (simulate_interval passes drift3 / drift1).
template <int NX, class Rng, bool SPARSE, class Drift>
__device__ __forceinline__ int simulate_interval_d(const Cstr& p, Plant<NX>& pl, double t0, double t1,
                                                   double u, int ns, Rng& rng, const Drift& drift) {
    const double dt = (t1 - t0) / ns;
    const double sqrt_dt = sqrt(dt);
    const double f = u * kMlMinToLs;
    double sig[NX];
    if (NX == 3) {
        sig[0] = f * p.sigmaA;
        sig[1] = f * p.sigmaB;
        sig[NX - 1] = f * p.sigmaT;
    } else {
        sig[0] = f * p.sigmaT;
    }
    for (int k = 0; k < ns; ++k) {
        double dw[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) {
            if constexpr (SPARSE) {
                if (j < NX - 1) {
                    rng.skip();
                    dw[j] = 0.0;
                    continue;
                }
            }
            dw[j] = sqrt_dt * rng.normal();
        }
        double dn[NX];
        const int st = drift(pl.x, u, dn);
        if (st != ST_OK) return st;
        double next[NX];
#pragma unroll
        for (int i = 0; i < NX; ++i) next[i] = pl.x[i] + dt * dn[i];  // axpy
        bool fin = true;
#pragma unroll
        for (int i = 0; i < NX; ++i) {  // gemv_into(1, sigma, dw, 1, next)
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += (i == j ? sig[i] : 0.0) * dw[j];
            next[i] = epi1(s, next[i]);
            fin = fin && dfinite(next[i]);
        }
        if (!fin) return ST_NONFINITE;
#pragma unroll
        for (int i = 0; i < NX; ++i) pl.x[i] = next[i];
    }
    return ST_OK;
}

template <int NX, class Rng, bool SPARSE = false>
__device__ __forceinline__ int simulate_interval(const Cstr& p, Plant<NX>& pl, double t0, double t1,
                                                 double u, int ns, Rng& rng) {
    return simulate_interval_d<NX, Rng, SPARSE>(p, pl, t0, t1, u, ns, rng,
                                                [&](const double* x, double uu, double* dn) -> int {
                                                    if (NX == 3) return drift3(p, x, uu, dn);
                                                    return drift1(p, x[0], uu, dn);
                                                });
}

}  // namespace nmpcmc_dev
