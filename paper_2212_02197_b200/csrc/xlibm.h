// xlibm.h -- portable exp / log / sincos, bit-identical on host and device.
//
// Why this exists: the reference
// (/root/reference/proj/core/src/cstr.cpp:39 exp; rng.cpp:91-95 log, sin, cos)
// calls glibc's libm, whose results neither CUDA libdevice nor any other libm
// reproduces bit-for-bit, and the NMPC loop amplifies 1-ulp differences into
// >1e-5 changes of the closed-loop cost. One source compiled for both sides
// fixes that: the CUDA kernels call these functions, and the oracle's
// "exact-libm" link variant redirects the reference objects' exp/log/sincos
// symbols to them (oracle/Makefile). Only IEEE +,-,*,/ and explicit fma()
// are used; compile with nvcc --fmad=false and gcc -ffp-contract=off so no
// other contraction happens. Accuracy is ~0.5 ulp (tests/test_xlibm.py
// measures it against mpmath).
//
// Algorithms (standard, restated): exp -- 2^(j/128) table + degree-5
// polynomial on |r| <= ln2/256; log -- 128-entry reciprocal table on
// z in [0x1.6p-1, 0x1.6p0) + double-double reconstruction + degree-10
// log1p polynomial; sincos -- reduction by pi/64 in three Cody-Waite parts
// (valid for |x| < 2^19), sin/cos(j pi/64) double-double table, degree-9/8
// polynomials, compensated reconstruction.
#pragma once

#include <stdint.h>
#include <string.h>
#include <math.h>

#include "xlibm_tables.h"

#if defined(__CUDACC__)
#define XLIBM_FN __host__ __device__ static inline
#else
#define XLIBM_FN static inline
#endif

#if defined(__CUDACC__)
#define XLIBM_DECLARE_TABLE(name, DATA)                       \
    __device__ static const double xlibm_d_##name[128] = {DATA}; \
    static const double xlibm_h_##name[128] = {DATA};
#else
#define XLIBM_DECLARE_TABLE(name, DATA) static const double xlibm_h_##name[128] = {DATA};
#endif

XLIBM_DECLARE_TABLE(exp_hi, XLIBM_EXP_HI_DATA)
XLIBM_DECLARE_TABLE(exp_tail, XLIBM_EXP_TAIL_DATA)
XLIBM_DECLARE_TABLE(log_invc, XLIBM_LOG_INVC_DATA)
XLIBM_DECLARE_TABLE(log_logc_hi, XLIBM_LOG_LOGC_HI_DATA)
XLIBM_DECLARE_TABLE(log_logc_lo, XLIBM_LOG_LOGC_LO_DATA)
XLIBM_DECLARE_TABLE(sin_hi, XLIBM_SIN_HI_DATA)
XLIBM_DECLARE_TABLE(sin_lo, XLIBM_SIN_LO_DATA)
XLIBM_DECLARE_TABLE(cos_hi, XLIBM_COS_HI_DATA)
XLIBM_DECLARE_TABLE(cos_lo, XLIBM_COS_LO_DATA)

#if defined(__CUDA_ARCH__)
#define XLIBM_T(name, i) __ldg(&xlibm_d_##name[(i)])
#else
#define XLIBM_T(name, i) (xlibm_h_##name[(i)])
#endif

XLIBM_FN uint64_t xlibm_asu64(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, sizeof u);
    return u;
#endif
}

XLIBM_FN double xlibm_asf64(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, sizeof x);
    return x;
#endif
}

XLIBM_FN double xlibm_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}

#define XLIBM_SHIFT 0x1.8p52
#define XLIBM_INF HUGE_VAL

/// Knuth TwoSum: s = RN(a+b), *err = (a+b) - s exactly.
XLIBM_FN double xlibm_two_sum(double a, double b, double* err) {
    double s = a + b;
    double bb = s - a;
    *err = (a - (s - bb)) + (b - bb);
    return s;
}

XLIBM_FN double xlibm_exp(double x) {
    if (x != x) return x + x;
    if (x > 0x1.62e42fefa39efp+9) return XLIBM_INF;  // > ln(DBL_MAX)
    if (x < -0x1.74910d52d3052p+9) return 0.0;       // < ln(2^-1075)
    double z = x * XLIBM_EXP_INV_LN2N;
    double kds = z + XLIBM_SHIFT;
    // kds = SHIFT + round(z) exactly (|z| < 2^18 here): the integer is the
    // difference of the bit patterns, so no float-to-int conversion sits on
    // the dependency chain; kd = round(z) as before
    int64_t k = (int64_t)(xlibm_asu64(kds) - xlibm_asu64(XLIBM_SHIFT));
    double kd = kds - XLIBM_SHIFT;
    double r = xlibm_fma(-kd, XLIBM_EXP_LN2N_HI, x);
    r = xlibm_fma(-kd, XLIBM_EXP_LN2N_LO, r);
    int j = (int)(k & 127);
    int64_t e = (k - j) / 128;
    double tail = XLIBM_T(exp_tail, j);
    double hi = XLIBM_T(exp_hi, j);
    double r2 = r * r;
    double tmp = tail + r + r2 * (XLIBM_EXP_C2 + r * XLIBM_EXP_C3) +
                 (r2 * r2) * (XLIBM_EXP_C4 + r * XLIBM_EXP_C5);
    if (e > 1020 || e < -1020) {
        if (e > 0) {
            double scale = xlibm_asf64(xlibm_asu64(hi) + ((uint64_t)(e - 2) << 52));
            return 4.0 * (scale + scale * tmp);
        }
        double scale = xlibm_asf64(xlibm_asu64(hi) + ((uint64_t)(e + 1000) << 52));
        return (scale + scale * tmp) * 0x1p-1000;
    }
    double scale = xlibm_asf64(xlibm_asu64(hi) + ((uint64_t)e << 52));
    return scale + scale * tmp;
}

XLIBM_FN double xlibm_log(double x) {
    uint64_t ix = xlibm_asu64(x);
    if (x != x) return x + x;
    if (x < 0.0) return (x - x) / (x - x);  // NaN
    if (x == 0.0) return -XLIBM_INF;
    if (x == XLIBM_INF) return x;
    int64_t kadj = 0;
    if (ix < 0x0010000000000000ULL) {  // subnormal: scale into the normal range
        x = x * 0x1p52;
        ix = xlibm_asu64(x);
        kadj = -52;
    }
    const uint64_t off = 0x3fe6000000000000ULL;
    uint64_t tmp = ix - off;
    int i = (int)((tmp >> 45) & 127);
    int64_t k = ((int64_t)tmp >> 52) + kadj;
    uint64_t iz = ix - (tmp & (0xfffULL << 52));
    double z = xlibm_asf64(iz);
    double invc = XLIBM_T(log_invc, i);
    double logc_hi = XLIBM_T(log_logc_hi, i);
    double logc_lo = XLIBM_T(log_logc_lo, i);
    double r = xlibm_fma(z, invc, -1.0);
    double kd = (double)k;
    double werr, herr;
    double w = xlibm_two_sum(kd * XLIBM_LN2_HI, logc_hi, &werr);
    double hi = xlibm_two_sum(w, r, &herr);
    double r2 = r * r;
    double q = XLIBM_LOG_C3 +
               r * (XLIBM_LOG_C4 +
                    r * (XLIBM_LOG_C5 +
                         r * (XLIBM_LOG_C6 +
                              r * (XLIBM_LOG_C7 +
                                   r * (XLIBM_LOG_C8 + r * (XLIBM_LOG_C9 + r * XLIBM_LOG_C10))))));
    double p = -0.5 * r2 + (r2 * r) * q;
    double lo = herr + werr + kd * XLIBM_LN2_LO + logc_lo + p;
    return hi + lo;
}

/// sin and cos of one argument, as glibc's sincos(x, &s, &c).
XLIBM_FN void xlibm_sincos(double x, double* s_out, double* c_out) {
    if (!(x - x == 0.0)) {  // inf or nan
        *s_out = x - x;
        *c_out = x - x;
        return;
    }
    double nds = x * XLIBM_INV_PIO64 + XLIBM_SHIFT;
    int64_t n = (int64_t)(xlibm_asu64(nds) - xlibm_asu64(XLIBM_SHIFT));  // as in xlibm_exp
    double nd = nds - XLIBM_SHIFT;
    // r + r_lo = x - n pi/64: the P1 product and difference are exact, the
    // P2 step is a TwoSum, P3 only feeds the low word.
    double t = xlibm_fma(-nd, XLIBM_PIO64_1, x);
    double e1;
    double r = xlibm_two_sum(t, -(nd * XLIBM_PIO64_2), &e1);
    double r_lo = e1 - nd * XLIBM_PIO64_3;
    int j = (int)(n & 127);
    double sh = XLIBM_T(sin_hi, j), sl = XLIBM_T(sin_lo, j);
    double ch = XLIBM_T(cos_hi, j), cl = XLIBM_T(cos_lo, j);
    double r2 = r * r;
    double sr_tail = (r * r2) * (XLIBM_SIN_S3 + r2 * (XLIBM_SIN_S5 + r2 * (XLIBM_SIN_S7 + r2 * XLIBM_SIN_S9)));
    double cr1 = r2 * (XLIBM_COS_C2 + r2 * (XLIBM_COS_C4 + r2 * (XLIBM_COS_C6 + r2 * XLIBM_COS_C8)));
    // sin(a + r) = S + C r + [S (cos r - 1) + C (sin r - r) + S_lo + C_lo r]
    double p = ch * r;
    double perr = xlibm_fma(ch, r, -p);
    double serr;
    double s = xlibm_two_sum(sh, p, &serr);
    double stail = serr + perr + ch * r_lo + sl + cl * r + sh * cr1 + ch * sr_tail;
    // cos(a + r) = C - S r + [C (cos r - 1) - S (sin r - r) + C_lo - S_lo r]
    double q = sh * r;
    double qerr = xlibm_fma(sh, r, -q);
    double cerr;
    double c = xlibm_two_sum(ch, -q, &cerr);
    double ctail = cerr - qerr - sh * r_lo + cl - sl * r + ch * cr1 - sh * sr_tail;
    *s_out = s + stail;
    *c_out = c + ctail;
}

XLIBM_FN double xlibm_sin(double x) {
    double s, c;
    xlibm_sincos(x, &s, &c);
    return s;
}

XLIBM_FN double xlibm_cos(double x) {
    double s, c;
    xlibm_sincos(x, &s, &c);
    return c;
}
