// certified_math.cuh -- certified fast FP64 sqrt / division for the serial
// Riccati recursions (K3, K3g/K3w). A Markstein step from a hardware
// reciprocal(-sqrt) seed gives the correctly rounded result almost always; an
// exact fma residual then PROVES it (certificate), and any uncertified result
// is replayed with IEEE operations by the caller, so results stay bitwise
// those of the reference's IEEE sqrt and division.
#pragma once

#include "device_common.cuh"

namespace nmpcmc_dev {

// ------------------------------------------- certified fast sqrt / division
// Certificates work on the high words only (cheap integer ops). Windows:
// the Cholesky pivot l in [2^-200, 2^200), numerators in [2^-400, 2^400),
// so every quotient lies in [2^-600, 2^600): residuals are exact, half-ulps
// are normal, nothing under/overflows.
__device__ __forceinline__ bool hi_window(double x, unsigned lo_e, unsigned span) {
    const unsigned e = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;
    return (e - lo_e) < span;
}
/// ulp(x)/2 for |x| in the window: 2^(E-1023-53).
__device__ __forceinline__ double half_ulp_hi(double x) {
    return __hiloint2double((__double2hiint(x) & 0x7ff00000) - (53 << 20), 0);
}
__device__ __forceinline__ bool mant_nonzero(double x) {
    return ((__double2hiint(x) & 0x000fffff) | __double2loint(x)) != 0;
}

#ifndef NMPCMC_SQRT_ONE_NEWTON
#define NMPCMC_SQRT_ONE_NEWTON 1
#endif
/// l ~ sqrt(h) and y ~ 1/l for h > 0: one Newton step (default; two with
/// NMPCMC_SQRT_ONE_NEWTON=0) on the hardware rsqrt seed and
/// a Markstein correction. Not yet certified (see cert_sqrt).
__device__ __forceinline__ void fast_sqrt(double h, double& l, double& y) {
    double y0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(h));
    const double hh = 0.5 * h;
    double e = __fma_rn(-hh, y0 * y0, 0.5);
    y0 = __fma_rn(y0, e, y0);
#if !NMPCMC_SQRT_ONE_NEWTON
    e = __fma_rn(-hh, y0 * y0, 0.5);
    y0 = __fma_rn(y0, e, y0);
#endif
    const double s = h * y0;
    const double d = __fma_rn(-s, s, h);
    l = __fma_rn(d, 0.5 * y0, s);
    y = y0;
}
/// q ~ a / b from y ~ 1/b (Markstein correction); 3 dependent operations.
/// Not yet certified (see cert_div).
__device__ __forceinline__ double fast_div(double a, double b, double y) {
    const double q0 = a * y;
    const double e0 = __fma_rn(-b, q0, a);
    return __fma_rn(e0, y, q0);
}
/// True only if l is RN(sqrt(h)): the exact residual h - l^2 lies strictly
/// inside (-l ulp(l), l ulp(l)) shrunk by 2^-50, l is not a power of two and
/// inside its window.
__device__ __forceinline__ bool cert_sqrt(double h, double l) {
    const double r = __fma_rn(-l, l, h);
    const double bound = (l * (1.0 - 0x1.0p-50)) * (2.0 * half_ulp_hi(l));
    return hi_window(l, 1023u - 200u, 400u) && mant_nonzero(l) && fabs(r) < bound;
}
/// True only if q is RN(a / b) for b > 0: the exact residual a - b q lies
/// strictly inside b ulp(q) / 2 (shrunk), q not a power of two, a and b
/// inside their windows.
__device__ __forceinline__ bool cert_div(double a, double b, double q) {
    const double e = __fma_rn(-b, q, a);
    return hi_window(a, 1023u - 400u, 800u) && hi_window(b, 1023u - 200u, 400u) && mant_nonzero(q) &&
           fabs(e) < (b * (1.0 - 0x1.0p-50)) * half_ulp_hi(q);
}

/// Branch-free forms of the certificates (bitwise &): for use inside serial
/// dependency chains, where a short-circuit would split the chain into
/// convergence regions.
__device__ __forceinline__ bool cert_sqrt_bf(double h, double l) {
    const double r = __fma_rn(-l, l, h);
    const double bound = (l * (1.0 - 0x1.0p-50)) * (2.0 * half_ulp_hi(l));
    return hi_window(l, 1023u - 200u, 400u) & mant_nonzero(l) & (fabs(r) < bound);
}
__device__ __forceinline__ bool cert_div_bf(double a, double b, double q) {
    const double e = __fma_rn(-b, q, a);
    return hi_window(a, 1023u - 400u, 800u) & hi_window(b, 1023u - 200u, 400u) & mant_nonzero(q) &
           (fabs(e) < (b * (1.0 - 0x1.0p-50)) * half_ulp_hi(q));
}
/// a / b from y ~ 1/b with its certificate folded into ok. A zero numerator
/// is exact as a * y, which also carries the IEEE sign of the zero.
__device__ __forceinline__ double cdiv_seed(double a, double b, double y, bool& ok) {
    const double q0 = a * y;
    const double q = __fma_rn(__fma_rn(-b, q0, a), y, q0);
    const bool z = (a == 0.0);
    ok &= z | cert_div_bf(a, b, q);
    return z ? q0 : q;
}

}  // namespace nmpcmc_dev
