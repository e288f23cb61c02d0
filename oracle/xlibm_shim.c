/* Exported wrappers around the portable libm (paper_2212_02197_b200/csrc/xlibm.h).
 *
 * Test infrastructure only. Two uses:
 *  - the "exact-libm" variant of the reference build redirects the reference
 *    objects' exp/log/sin/cos/sincos symbols to these (objcopy --redefine-sym,
 *    oracle/Makefile), so the CPU oracle rounds exactly like the device;
 *  - tests/test_xlibm.py loads them via ctypes to measure ulp error.
 * Compile with -ffp-contract=off (no implicit FMA), like the device build's
 * --fmad=false. */
#include "../paper_2212_02197_b200/csrc/xlibm.h"

double nmx_exp(double x) { return xlibm_exp(x); }
double nmx_log(double x) { return xlibm_log(x); }
double nmx_sin(double x) { return xlibm_sin(x); }
double nmx_cos(double x) { return xlibm_cos(x); }
void nmx_sincos(double x, double* s, double* c) { xlibm_sincos(x, s, c); }
