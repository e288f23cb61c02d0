// nmpc_kernel.cuh -- K3: NMPC closed loop, one warp per sample.
//
// Restates, for the one-state controller model (cstr.cpp one_state variant,
// the paper/reference default), the reference's NMPC branch of
// run_closed_loop (montecarlo.cpp:80-157):
//   nmpc_step          controllers.cpp:114-212 (filter, warm/cold start, SQP, predict)
//   filter_update      ekf.cpp:59-96            predict      ekf.cpp:26-57
//   shoot              ocp.cpp:9-74             eval_objective / eval_constraints ocp.cpp:76-135
//   xi_from_inputs     ocp.cpp:137-154
//   sqp_solve          sqp.cpp:182-411 (+ line_search :22-59, bfgs_block_update :61-84,
//                      check_convergence :86-96, lagrangian_gradient :102-128)
//   solve_qp           qp.cpp:173-423 (+ riccati_factor :73-110, riccati_solve_vectors :116-155)
// with the reference's floating-point operation order everywhere, so that with
// the shared portable libm the per-sample results are bitwise those of the
// reference's exact-libm build (tests/test_gpu_nmpc.py).
//
// Execution model (K3):
//  * one warp = one block = one sample at a time; persistent blocks pull
//    sample indices from an atomic counter. The workspace is split: the 22
//    arrays the serial Riccati sweeps and ordered reductions read live in
//    shared memory (ST doubles each, ST = compile-time stride >= N+1), the 25
//    arrays only lane-parallel loops touch live in a per-block global region
//    that stays L2-resident -- which doubles the samples resident per SM;
//  * stage-parallel work (the N independent shooting intervals, residuals,
//    expand / step-length / update loops, BFGS blocks) is spread over the 32
//    lanes, k = lane, lane+32, ...;
//  * the serial recursions (Riccati sweeps, ordered reductions,
//    xi_from_inputs, EKF, plant) run redundantly on all 32 lanes in lockstep;
//  * the Riccati sweeps -- the latency-critical chain -- use a certified fast
//    square root and division (Markstein correction from the hardware
//    reciprocal-sqrt seed; an exact fma residual certifies that each result is
//    the IEEE correctly rounded one). A sweep whose certificate fails anywhere
//    is replayed with IEEE sqrt/division, so results are always bitwise IEEE;
//  * phases are __noinline__ functions with one call site each, which keeps
//    the kernel small enough for the instruction cache;
//  * exceptions become per-sample status codes with the reference's catch
//    scopes.
#pragma once

#include "certified_math.cuh"
#include "device_common.cuh"

#ifndef NMPCMC_QP_LOCAL_OCP
#define NMPCMC_QP_LOCAL_OCP 1
#endif
// In solve_qp a by-value copy of the Ocp keeps o.gws / o.N in registers for
// the inlined expand / step / certificate helpers; through the reference they
// are reloaded from local memory after every store (+0.6 %). Copying it in
// every phase measured 6.5 % slower (larger frames, register pressure).
#if NMPCMC_QP_LOCAL_OCP
#define NMPCMC_LOCAL_OCP(name, src) const Ocp name = src
#else
#define NMPCMC_LOCAL_OCP(name, src) const Ocp& name = src
#endif

// Unroll factors of the serial Riccati / rollout loops (experiments; 1 =
// the measured default, the kernel is instruction-cache sensitive).
#ifndef NMPCMC_UNROLL_FACTOR
#define NMPCMC_UNROLL_FACTOR 1
#endif
#ifndef NMPCMC_UNROLL_VECTOR
#define NMPCMC_UNROLL_VECTOR 1
#endif
#ifndef NMPCMC_UNROLL_ROLLOUT
#define NMPCMC_UNROLL_ROLLOUT 1
#endif

// Unroll factors of the lane-parallel stage loops (k = lane, lane + 32, ...)
// of solve_qp and of the shooting loop (experiments; 1 = the default).
#ifndef NMPCMC_UNROLL_QP_LANES
#define NMPCMC_UNROLL_QP_LANES 1
#endif
#ifndef NMPCMC_UNROLL_SHOOT_LANES
#define NMPCMC_UNROLL_SHOOT_LANES 1
#endif

namespace nmpcmc_dev {

constexpr int kUnrollQpLanes = NMPCMC_UNROLL_QP_LANES;
constexpr int kUnrollShootLanes = NMPCMC_UNROLL_SHOOT_LANES;
constexpr unsigned FULLMASK = 0xffffffffu;
constexpr int kUnrollFactor = NMPCMC_UNROLL_FACTOR;
constexpr int kUnrollVector = NMPCMC_UNROLL_VECTOR;
constexpr int kUnrollRollout = NMPCMC_UNROLL_ROLLOUT;
#define kNaN __longlong_as_double(0x7ff8000000000000LL)
constexpr double kEpsMach = 0x1.0p-52;  // numeric_limits<double>::epsilon (sqp.cpp:71)

// ------------------------------------------------------------ warp helpers
/// inf_norm fold (linalg.cpp:204-208): m = max(m, |x|) with std::max, so NaN
/// entries are ignored; partials never become NaN, hence order-independent.
__device__ __forceinline__ double fold_absmax(double m, double x) {
    const double a = fabs(x);
    return (m < a) ? a : m;
}
__device__ __forceinline__ double warp_max(double m) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double v = __shfl_xor_sync(FULLMASK, m, o);
        m = (m < v) ? v : m;
    }
    return m;
}
/// std::min fold starting from a non-NaN value (max_step, qp.cpp:321-337).
__device__ __forceinline__ double warp_min(double m) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double v = __shfl_xor_sync(FULLMASK, m, o);
        m = (v < m) ? v : m;
    }
    return m;
}
__device__ __forceinline__ int warp_min_int(int v) { return __reduce_min_sync(FULLMASK, v); }
__device__ __forceinline__ int warp_sum_int(int v) { return __reduce_add_sync(FULLMASK, v); }
__device__ __forceinline__ bool warp_any(bool p) { return __any_sync(FULLMASK, p); }
/// Exact warp min / max of NON-NEGATIVE doubles via REDUX on the bit
/// patterns (IEEE order is the unsigned order of the words for x >= 0):
/// two single-instruction reductions instead of ten shuffles.
__device__ __forceinline__ double warp_min_pos(double a) {
    const unsigned hi = (unsigned)__double2hiint(a), lo = (unsigned)__double2loint(a);
    const unsigned mh = __reduce_min_sync(FULLMASK, hi);
    const unsigned ml = __reduce_min_sync(FULLMASK, hi == mh ? lo : 0xffffffffu);
    return __hiloint2double((int)mh, (int)ml);
}
__device__ __forceinline__ double warp_max_pos(double a) {
    const unsigned hi = (unsigned)__double2hiint(a), lo = (unsigned)__double2loint(a);
    const unsigned mh = __reduce_max_sync(FULLMASK, hi);
    const unsigned ml = __reduce_max_sync(FULLMASK, hi == mh ? lo : 0u);
    return __hiloint2double((int)mh, (int)ml);
}

// ------------------------------------------------------- one-state model
/// One stage evaluation of the controller model: drift (cstr.cpp:42-53),
/// drift_jacobian_x (cstr.cpp:99-119, one_state branch) and drift_jacobian_u
/// (cstr.cpp:120-127). exp(-EaR/cT) is evaluated once: drift and jac_x compute
/// it from bitwise identical arguments.
struct Stage1 {
    double k, a, b;
};

__device__ __forceinline__ int eval1(const Cstr& p, double x, double u, Stage1& s, bool want_jac) {
    const double f = u * kMlMinToLs;
    const double c = x / p.V;
    const Conc1 cc = conc1(p, c);
    if (cc.cT <= 0.0) return ST_DOMAIN;
    const double ex = xlibm_exp(-p.EaR / cc.cT);
    const double r = p.k0 * ex * cc.cA * cc.cB;
    s.k = p.cT_in * f - c * f + p.beta * r * p.V;
    if (want_jac) {
        const double k = p.k0 * ex;
        const double drdcT = k * (p.EaR / (cc.cT * cc.cT)) * cc.cA * cc.cB +
                             k * (-cc.cB / p.beta - 2.0 * cc.cA / p.beta);
        s.a = -f / p.V + p.beta * drdcT;
        s.b = (p.cT_in - x / p.V) * kMlMinToLs;
    }
    return ST_OK;
}

/// shoot (ocp.cpp:9-74), one-state: Nc RK4 steps with forward sensitivities.
/// WITH_SENS = false computes F only (xi_from_inputs never reads the
/// sensitivities; the exception behaviour is identical because jac_x throws
/// exactly when drift does).
template <bool WITH_SENS>
__device__ __forceinline__ int shoot1(const Cstr& p, double x, double u, double h, int nc, double& F,
                                      double& Sx, double& Su) {
    F = x;
    Sx = 1.0;
    Su = 0.0;
    const double h2 = 0.5 * h;
    const double h6 = h / 6.0;
#pragma unroll 1
    for (int step = 0; step < nc; ++step) {
        // stage j evaluates at (F, Sx, Su) + c_j h (k, kx, ku)_{j-1} with
        // c_j h = 0, h/2, h/2, 1.0*h (advanced / advanced_sens, ocp.cpp:39-46);
        // the weighted sum k1 + 2 k2 + 2 k3 + k4 accumulates left to right,
        // exactly the reference's expression order (ocp.cpp:51-60)
        double pk = 0.0, pkx = 0.0, pku = 0.0, acc = 0.0, accx = 0.0, accu = 0.0;
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
            double xs = F, sx = Sx, su = Su;
            if (j > 0) {
                const double ch = (j == 3) ? 1.0 * h : h2;
                xs = F + ch * pk;
                if (WITH_SENS) {
                    sx = Sx + ch * pkx;
                    su = Su + ch * pku;
                }
            }
            Stage1 s;
            const int st = eval1(p, xs, u, s, WITH_SENS);
            if (st) return st;
            double kx = 0.0, ku = 0.0;
            if (WITH_SENS) {
                kx = epi0(dot1(s.a, sx));
                ku = epi1(dot1(s.a, su), s.b);
            }
            if (j == 0) {
                acc = s.k;
                accx = kx;
                accu = ku;
            } else if (j < 3) {
                acc = acc + 2.0 * s.k;
                accx = accx + 2.0 * kx;
                accu = accu + 2.0 * ku;
            } else {
                acc = acc + s.k;
                accx = accx + kx;
                accu = accu + ku;
            }
            pk = s.k;
            pkx = kx;
            pku = ku;
        }
        F += h6 * acc;
        if (WITH_SENS) {
            Sx += h6 * accx;
            Su += h6 * accu;
        }
    }
    if (!dfinite(F)) return ST_NONFINITE;
    return ST_OK;
}

/// joint_rhs (ekf.cpp:12-22), one-state: dx = f, dP = A P + P A' + s s'.
__device__ __forceinline__ int joint_rhs1(const Cstr& p, double x, double P, double u, double& dx,
                                          double& dP) {
    Stage1 s;
    const int st = eval1(p, x, u, s, true);
    if (st) return st;
    dx = s.k;
    dP = epi0(dot1(s.a, P));
    dP = epi1(dot1(P, s.a), dP);
    const double sg = u * kMlMinToLs * p.sigmaT;  // cstr_diffusion
    dP = epi1(dot1(sg, sg), dP);
    return ST_OK;
}

// ----------------------------------------------------------- workspace
/// Full per-sample array set (the retired one-thread-per-sample K3b laid all of them out)
/// in global memory. Stage arrays are indexed by k; for the interleaved
/// decision vector xi = (u_0, x_1, ..., u_{N-1}, x_N) (ocp.hpp:37-43)
/// U[k] = u_k and X[k] = x_{k+1}. W blocks: Wr[0] = block 0 (u_0),
/// (Wq, Wm, Wr)[k] = block k = [x_k, u_k] (k = 1..N-1), Wq[N] = block N.
enum ArrayId {
    A_U, A_X, A_LAM, A_PIL, A_PIU,
    A_GX, A_G, A_JX, A_JU, A_TGX, A_TG, A_TJX, A_TJU,
    A_WQ, A_WM, A_WR, A_SIG, A_SP,
    A_DU, A_DX, A_MU, A_NL, A_NU, A_SL, A_SU,
    A_RSU, A_RSX, A_RDYN, A_RCL, A_RCU,
    A_DDU, A_DDX, A_DDMU,
    A_CHOLH, A_RINV, A_GAIN, A_GMAT, A_VAL, A_PVEC, A_DFF, A_RHAT, A_BAR,
    A_TMP,  // two strides
    kWsArrays = A_TMP + 2
};

__host__ __device__ inline int ws_stride_for(int N) { return N < 32 ? 32 : N < 64 ? 64 : (N < 128 ? 128 : 256); }

/// K3 splits the workspace by access pattern. Shared memory holds what the
/// serial Riccati sweeps and ordered reductions read (their latency is on the
/// critical path); a per-block region of global memory (L2-resident: ~12 KB
/// per resident sample) holds the rest, touched only by lane-parallel loops.
extern __shared__ __align__(16) double smem_nmpc[];

// NMPCMC_IPM_SMEM = 1 places the interior-point state and direction arrays
// (touched by every lane-parallel IPM phase) in shared memory, 0 in L2.
#ifndef NMPCMC_IPM_SMEM
#define NMPCMC_IPM_SMEM 0
#endif
// NMPCMC_CERT_SMEM = 1 keeps the certificate inputs of the fast Riccati
// sweeps (written by the serial sweeps, read by the lane-parallel certify
// loops) in shared memory instead of the L2 slab -- at strides up to 64, where
// it measured +1 % (profiles/r02/r02o_k3_cert_ab.txt). At stride 128 the four
// extra arrays cost two resident samples per SM (8 instead of 10) and 8 %
// (r02f2_k3_n120_cert_ab.txt), so there they stay in the slab. The layout is
// therefore a function of the stride: S_TMP, S_IPM0, G_IPM0 and the array
// counts below are expressions in the template parameter ST.
#ifndef NMPCMC_CERT_SMEM
#define NMPCMC_CERT_SMEM 1
#endif
__host__ __device__ constexpr bool cert_in_smem(int stride) { return NMPCMC_CERT_SMEM && stride <= 64; }
enum SmemId {
    S_JX, S_JU, S_WQ, S_WM, S_WR, S_BAR, S_RDYN, S_RHAT, S_RSX,
    S_CHOLH, S_RINV, S_VAL, S_GAIN, S_GMAT, S_PVEC, S_DFF,
    S_DDU, S_DDX,
    S_CHH, S_CA1, S_CQ1, S_CG1,  // only if cert_in_smem(ST)
    kSmemFixed = S_CHH
};
enum GlobId {
    G_U, G_X, G_TU, G_TX, G_LAM, G_PIL, G_PIU,
    G_GX, G_G, G_TGX, G_TG, G_TJX, G_TJU,
    G_SIG, G_SP,
    G_CHH, G_CA1, G_CQ1, G_CG1,  // certificate inputs of the fast Riccati sweeps, unless cert_in_smem(ST)
    kGlobFixed = G_CHH
};
__host__ __device__ constexpr int smem_tmp(int stride) { return kSmemFixed + (cert_in_smem(stride) ? 4 : 0); }
__host__ __device__ constexpr int smem_arrays(int stride) {
    return smem_tmp(stride) + 3 + (NMPCMC_IPM_SMEM ? 14 : 0);
}
__host__ __device__ constexpr int glob_ipm0(int stride) { return kGlobFixed + (cert_in_smem(stride) ? 0 : 4); }
__host__ __device__ constexpr int glob_arrays(int stride) {
    return glob_ipm0(stride) + (NMPCMC_IPM_SMEM ? 0 : 14);
}
#define S_TMP smem_tmp(ST)  // three strides
#define S_IPM0 (smem_tmp(ST) + 3)
#define G_IPM0 glob_ipm0(ST)
/// interior-point arrays: DU DX MU NL NU SL SU RSU RCL RCU DSL DSU DNL DNU
enum IpmId { I_DU, I_DX, I_MU, I_NL, I_NU, I_SL, I_SU, I_RSU, I_RCL, I_RCU, I_DSL, I_DSU, I_DNL, I_DNU };
#if NMPCMC_IPM_SMEM
#define IA(id) (smem_nmpc + (S_IPM0 + (id)) * ST)
#else
#define IA(id) (o.gws + (G_IPM0 + (id)) * ST)
#endif

/// Out-of-line IEEE division for the lane-parallel loops: one call site per
/// use instead of an inlined ~25-instruction sequence keeps the hot code small
/// (the kernel is instruction-cache bound; see profiles/).
static __device__ __noinline__ double qdiv(double a, double b) { return a / b; }

#define SA(id) (smem_nmpc + (id) * ST)
#define GA(id) (o.gws + (id) * ST)
#define CA(name) (cert_in_smem(ST) ? SA(S_##name) : GA(G_##name))

__host__ __device__ inline size_t ws_bytes_for(int ST) { return (size_t)smem_arrays(ST) * ST * sizeof(double); }
__host__ __device__ inline size_t gws_bytes_for(int ST) { return (size_t)glob_arrays(ST) * ST * sizeof(double); }

/// Scalars of one NMPC problem instance (NlpInstance, ocp.hpp:25-34).
struct Ocp {
    Cstr p;        // controller model parameters
    int N, Nc;
    double Ts;     // horizon.Ts
    double h;      // Ts / Nc (ocp.cpp:13)
    double x0;     // filtered estimate
    double umin, umax;
    double Qz;
    double inv_V;  // output / measurement jacobian 1/V (cstr.cpp:92-95)
    double* gws;   // K3: this block's global workspace
};

/// Work counters accumulated per sample (lane-uniform).
struct Cnt {
    long long steps, shoot_full, shoot_fonly, ipm_stage, sqp_stage, qp, sqp, ls;
};

// ------------------------------------------------------------ OCP evals
/// eval_objective (ocp.cpp:76-99): phi in k order; gradient only on the x
/// slots, gX[k] = d phi / d x_{k+1}.
template <int ST>
__device__ __noinline__ double eval_objective(const Ocp& o, const double* X, double* gX) {
    const int lane = threadIdx.x & 31;
    double* tmp = SA(S_TMP);
    const double* sp = GA(G_SP);
    const double ts = o.Ts;
#pragma unroll 1
    for (int k = lane; k < o.N; k += 32) {
        const double res = X[k] / o.p.V - sp[k];  // output(x) - zbar
        const double qres = epi0(dot1(o.Qz, res));
        tmp[k] = ts * dot1(res, qres);
        const double gx = epi0(dot1(o.inv_V, qres));
        gX[k] = 0.0 + 2.0 * ts * gx;
    }
    __syncwarp();
    double phi = 0.0;
#pragma unroll 1
    for (int k = 0; k < o.N; ++k) phi += tmp[k];
    __syncwarp();
    return phi;
}

/// eval_constraints (ocp.cpp:101-135) into (g, Jx, Ju), plus the status of the
/// first failing stage in k order (the reference throws at the first failing
/// shoot). g[k] = x_{k+1} - F_k.
template <int ST>
__device__ __noinline__ int eval_constraints(const Ocp& o, const double* U, const double* X, double* g, double* Jx,
                                             double* Ju, Cnt* cnt) {
    const int lane = threadIdx.x & 31;
    int first_bad = 0x7fffffff;
#pragma unroll kUnrollShootLanes
    for (int k = lane; k < o.N; k += 32) {
        const double xk = (k == 0) ? o.x0 : X[k - 1];
        double F, Sx, Su;
        const int st = shoot1<true>(o.p, xk, U[k], o.h, o.Nc, F, Sx, Su);
        if (st) {
            first_bad = min(first_bad, (k << 4) | st);
        } else {
            g[k] = X[k] - F;
            Jx[k] = Sx;
            Ju[k] = Su;
        }
    }
    cnt->shoot_full += o.N;
    first_bad = warp_min_int(first_bad);
    __syncwarp();
    return first_bad == 0x7fffffff ? ST_OK : (first_bad & 15);
}

/// xi_from_inputs (ocp.cpp:137-154): forward shooting from x0 with inputs U,
/// states into X; serial in k, all lanes.
template <int ST>
__device__ __noinline__ int xi_from_inputs(const Ocp& o, const double* U, double* X, Cnt* cnt) {
    double xk = o.x0;
    int st = ST_OK;
    int k = 0;
#pragma unroll 1
    for (; k < o.N; ++k) {
        double F, Sx, Su;
        st = shoot1<false>(o.p, xk, U[k], o.h, o.Nc, F, Sx, Su);
        if (st) break;
        X[k] = F;
        xk = F;
    }
    cnt->shoot_fonly += (k < o.N) ? k + 1 : o.N;
    __syncwarp();
    return st;
}

// ------------------------------------------------------------------- QP
/// b_k = F_k - x_{k+1} recovered from g_k = x_{k+1} - F_k: IEEE subtraction is
/// antisymmetric, and an exact-zero defect is +0 either way.
__device__ __forceinline__ double bneg(double g) { return g == 0.0 ? 0.0 : -g; }

enum { QP_OPTIMAL = 0, QP_MAXITER = 1, QP_FAILED = 2, QP_DOMAIN = -1 };

// Inside the Riccati sweeps and rollouts the reference's 1x1 gemm/gemv
// epilogues "0.0 + a*b" / "1.0*s + 0.0" are evaluated as a*b / s. The two can
// differ only in the sign of an exact zero; in this path a signed zero never
// reaches a divisor (the divisors are Cholesky pivots, slacks, sws/sr > eps,
// V, beta, c_T > 0), a comparison outcome, or an output (phi is a sum of
// squares), so every nonzero result is bitwise that of the reference -- the
// GPU parity tests check exactly this.

/// riccati_factor (qp.cpp:73-110) fused with the affine backward vector sweep
/// of riccati_solve_vectors (qp.cpp:122-141). Serial in k, all lanes.
/// Returns true on NotPositiveDefinite. FAST: sqrt and the four divisions by
/// each pivot use the 3-operation fast forms; their inputs are stashed so that
/// certify_factor_k() can prove every result is the IEEE one afterwards (the
/// caller replays FAST = false otherwise).
template <int ST, bool FAST>
__device__ __noinline__ bool factor_sweep(const Ocp& o) {
    const int N = o.N;
    const double* Ju = SA(S_JU);
    const double* Jx = SA(S_JX);
    const double* Wq = SA(S_WQ);
    const double* Wm = SA(S_WM);
    const double* Wr = SA(S_WR);
    const double* bar = SA(S_BAR);
    const double* rdyn = SA(S_RDYN);
    const double* rhat = SA(S_RHAT);
    const double* rsx = SA(S_RSX);
    double* cholh = SA(S_CHOLH);
    double* rinv = SA(S_RINV);
    double* val = SA(S_VAL);
    double* gain = SA(S_GAIN);
    double* gmat = SA(S_GMAT);
    double* pvec = SA(S_PVEC);
    double* dff = SA(S_DFF);
    double* chh = CA(CHH);
    double* ca1 = CA(CA1);
    double* cq1 = CA(CQ1);
    double* cg1 = CA(CG1);
    double P = Wq[N];
    double pv = rsx[N - 1];  // pvec[N] = qhat[N]
    val[N] = P;
    pvec[N] = pv;
    // the head of the P chain (ju, Wr, bar) is loaded one stage ahead
    double ju = Ju[N - 1], wr = Wr[N - 1], br = bar[N - 1];
#pragma unroll kUnrollFactor
    for (int k = N - 1; k >= 0; --k) {
        const int kn = k > 0 ? k - 1 : 0;
        const double jun = Ju[kn], wrn = Wr[kn], brn = bar[kn];
        double hh = ju * (P * ju);
        hh = hh + wr;
        hh = hh + br;
        // cholesky_factor -> QP Failed (qp.cpp:358-364); tested at the end of
        // the stage so the branch does not sit on the chain (a failing stage's
        // values are never used)
        const bool npd = hh <= 0.0 || !dfinite(hh);
        double l, y;
        if (FAST) {
            fast_sqrt(hh, l, y);
            chh[k] = hh;
        } else {
            l = sqrt(hh);
            y = 1.0 / l;  // seed for the corrector sweep's fast division
        }
        cholh[k] = l;
        rinv[k] = y;
        const double tmpv = P * -rdyn[k] + pv;
        double hv = ju * tmpv + rhat[k];
        if (FAST) {
            ca1[k] = hv;
            hv = fast_div(hv, l, y);
            cq1[k] = hv;
            hv = fast_div(hv, l, y);
        } else {
            hv = hv / l;
            hv = hv / l;
        }
        hv = -hv;
        dff[k] = hv;
        if (k >= 1) {
            const double jx = Jx[k];
            const double pjx = P * jx;
            double gg = ju * pjx;
            gg = gg + Wm[k];
            double gn;
            if (FAST) {
                gn = fast_div(gg, l, y);
                cg1[k] = gn;
                gn = fast_div(gn, l, y);
            } else {
                gn = gg / l;
                gn = gn / l;
            }
            const double gk = -gn;
            double pn = jx * pjx;
            pn = pn + Wq[k];
            pn = gg * gk + pn;
            val[k] = pn;
            gain[k] = gk;
            gmat[k] = gg;
            double pvn = jx * tmpv + rsx[k - 1];
            pvn = gg * hv + pvn;
            pvec[k] = pvn;
            P = pn;
            pv = pvn;
        }
        if (npd) return true;
        ju = jun;
        wr = wrn;
        br = brn;
    }
    return false;
}

/// Certificate of stage k of a FAST factor_sweep (fused into a later loop).
template <int ST>
__device__ __forceinline__ bool certify_factor_k(const Ocp& o, int k) {
    const double l = SA(S_CHOLH)[k];
    const double q1 = CA(CQ1)[k];
    bool ok = cert_sqrt(CA(CHH)[k], l) && cert_div(CA(CA1)[k], l, q1) && cert_div(q1, l, -SA(S_DFF)[k]);
    if (k >= 1) {
        const double g1 = CA(CG1)[k];
        ok = ok && cert_div(SA(S_GMAT)[k], l, g1) && cert_div(g1, l, -SA(S_GAIN)[k]);
    }
    return ok;
}
/// Certificate of stage k of a FAST vector_sweep.
template <int ST>
__device__ __forceinline__ bool certify_vector_k(const Ocp& o, int k) {
    const double l = SA(S_CHOLH)[k];
    const double q1 = CA(CQ1)[k];
    return cert_div(CA(CA1)[k], l, q1) && cert_div(q1, l, -SA(S_DFF)[k]);
}

/// Corrector backward vector sweep with the cached factor (qp.cpp:122-141);
/// FAST stashes the division inputs for certify_vector_k().
template <int ST, bool FAST>
__device__ __noinline__ void vector_sweep(const Ocp& o) {
    const int N = o.N;
    const double* Ju = SA(S_JU);
    const double* Jx = SA(S_JX);
    const double* rdyn = SA(S_RDYN);
    const double* rhat = SA(S_RHAT);
    const double* rsx = SA(S_RSX);
    const double* cholh = SA(S_CHOLH);
    const double* rinv = SA(S_RINV);
    const double* val = SA(S_VAL);
    const double* gmat = SA(S_GMAT);
    double* pvec = SA(S_PVEC);
    double* dff = SA(S_DFF);
    double* ca1 = CA(CA1);
    double* cq1 = CA(CQ1);
    double pv = rsx[N - 1];
    pvec[N] = pv;
    // operands at the head of the pv chain are loaded one stage ahead
    double vl = val[N], rd = rdyn[N - 1], ju = Ju[N - 1], rh = rhat[N - 1];
#pragma unroll kUnrollVector
    for (int k = N - 1; k >= 0; --k) {
        const int kn = k > 0 ? k - 1 : 0;
        const double vln = val[kn + 1], rdn = rdyn[kn], jun = Ju[kn], rhn = rhat[kn];
        const double l = cholh[k];
        const double tmpv = vl * -rd + pv;
        double hv = ju * tmpv + rh;
        if (FAST) {
            const double y = rinv[k];
            ca1[k] = hv;
            hv = fast_div(hv, l, y);
            cq1[k] = hv;
            hv = fast_div(hv, l, y);
        } else {
            hv = hv / l;
            hv = hv / l;
        }
        hv = -hv;
        dff[k] = hv;
        if (k >= 1) {
            double pvn = Jx[k] * tmpv + rsx[k - 1];
            pvn = gmat[k] * hv + pvn;
            pvec[k] = pvn;
            pv = pvn;
        }
        vl = vln;
        rd = rdn;
        ju = jun;
        rh = rhn;
    }
}

/// Forward rollout (qp.cpp:142-155): step dxi (DDU, DDX). The multiplier step
/// dmu_k = -(P_{k+1} dx_k + p_{k+1}) (qp.cpp:153) is off the dx chain and is
/// formed where it is consumed (the update loop of solve_qp).
template <int ST>
__device__ __noinline__ void rollout(int N) {
    const double* Ju = SA(S_JU);
    const double* Jx = SA(S_JX);
    const double* rdyn = SA(S_RDYN);
    const double* gain = SA(S_GAIN);
    const double* dff = SA(S_DFF);
    double* ddU = SA(S_DDU);
    double* ddX = SA(S_DDX);
    double dx = -rdyn[0] + Ju[0] * dff[0];  // k = 0 (no state feedback)
    ddU[0] = dff[0];
    ddX[0] = dx;
    // the loop is latency-bound on the dx chain: stage k+1's operands are
    // loaded while stage k computes, so no shared-memory latency sits on it
    double g = gain[1], f = dff[1], jx = Jx[1], rd = rdyn[1], ju = Ju[1];
#pragma unroll kUnrollRollout
    for (int k = 1; k < N; ++k) {
        const int kn = k + 1 < N ? k + 1 : k;
        const double gn = gain[kn], fn = dff[kn], jxn = Jx[kn], rdn = rdyn[kn], jun = Ju[kn];
        const double du = g * dx + f;
        double dxn = jx * dx + -rd;
        dxn = ju * du + dxn;
        dx = dxn;
        ddU[k] = du;
        ddX[k] = dx;
        g = gn;
        f = fn;
        jx = jxn;
        rd = rdn;
        ju = jun;
    }
    __syncwarp();
}

/// expand (qp.cpp:308-317) of stage k from the step in DDU, given rl/ru;
/// stored in G_DSL.. for the later loops of the iteration.
struct Dir {
    double dsl, dsu, dnl, dnu;
};
template <int ST>
__device__ __forceinline__ Dir expand_k(const Ocp& o, int k, bool fl, bool fu, double rl, double ru) {
    const double dv = SA(S_DDU)[k];
    Dir d;
    d.dsl = fl ? dv + rl : 0.0;
    d.dsu = fu ? ru - dv : 0.0;
    d.dnl = fl ? qdiv(IA(I_RCL)[k] - IA(I_NL)[k] * d.dsl, IA(I_SL)[k]) : 0.0;
    d.dnu = fu ? qdiv(IA(I_RCU)[k] - IA(I_NU)[k] * d.dsu, IA(I_SU)[k]) : 0.0;
    IA(I_DSL)[k] = d.dsl;
    IA(I_DSU)[k] = d.dsu;
    IA(I_DNL)[k] = d.dnl;
    IA(I_DNU)[k] = d.dnu;
    return d;
}
template <int ST>
__device__ __forceinline__ Dir load_dir(const Ocp& o, int k) {
    return Dir{IA(I_DSL)[k], IA(I_DSU)[k], IA(I_DNL)[k], IA(I_DNU)[k]};
}
/// max_step's cap (qp.cpp:321-337) for the four (value, direction) pairs of
/// stage k: alpha = min(alpha, -frac value / dir) over dir < 0.
template <int ST>
__device__ __forceinline__ double step_caps(const Ocp& o, int k, bool fl, bool fu, const Dir& d, double frac,
                                            double alpha) {
    if (fl) {
        if (d.dsl < 0.0) alpha = smin(alpha, qdiv(-frac * IA(I_SL)[k], d.dsl));
        if (d.dnl < 0.0) alpha = smin(alpha, qdiv(-frac * IA(I_NL)[k], d.dnl));
    }
    if (fu) {
        if (d.dsu < 0.0) alpha = smin(alpha, qdiv(-frac * IA(I_SU)[k], d.dsu));
        if (d.dnu < 0.0) alpha = smin(alpha, qdiv(-frac * IA(I_NU)[k], d.dnu));
    }
    return alpha;
}

/// solve_qp (qp.cpp:173-423) for the stagewise box QP that build_stages
/// (sqp.cpp:130-171) forms from W, grad f and the defect blocks of the
/// current iterate:  stage k: R = Wr[k], Q = Wq[k], M = Wm[k] (k >= 1),
/// q = gX[k-1], r = 0, Jx, Ju, b = -g[k], lb = umin - u_k, ub = umax - u_k;
/// terminal Q = Wq[N], q = gX[N-1].  Result: step in DU/DX, multipliers MU, NL, NU.
template <int ST>
__device__ __noinline__ int solve_qp(const Ocp& o_in, double tol, int max_iter, Cnt* cnt) {
    NMPCMC_LOCAL_OCP(o, o_in);
    const int lane = threadIdx.x & 31;
    const int N = o.N;
    const double tau = 0.995;
    const double umin = o.umin, umax = o.umax;
    const double* U = GA(G_U);
    const double* gX = GA(G_GX);
    const double* g = GA(G_G);
    const double* Jx = SA(S_JX);
    const double* Ju = SA(S_JU);
    const double* Wq = SA(S_WQ);
    const double* Wm = SA(S_WM);
    const double* Wr = SA(S_WR);
    double* dU = IA(I_DU);
    double* dX = IA(I_DX);
    double* mu = IA(I_MU);
    double* nl = IA(I_NL);
    double* nu = IA(I_NU);
    double* sl = IA(I_SL);
    double* su = IA(I_SU);
    double* rsu = IA(I_RSU);
    double* rcl = IA(I_RCL);
    double* rcu = IA(I_RCU);
    double* rsx = SA(S_RSX);
    double* rdyn = SA(S_RDYN);
    double* rhat = SA(S_RHAT);
    double* bar = SA(S_BAR);
    double* tmp = SA(S_TMP);
    const double* ddU = SA(S_DDU);
    const double* ddX = SA(S_DDX);
    const double* val = SA(S_VAL);
    const double* pvec = SA(S_PVEC);
    // data_scale / bounds / init (qp.cpp:183-226)
    double ds = 1.0;
    int nfin = 0;
    bool bad = false;
#pragma unroll kUnrollQpLanes
    for (int k = lane; k < N; k += 32) {
        const double lb = umin - U[k];
        const double ub = umax - U[k];
        if (lb > ub) bad = true;
        const bool fl = dfinite(lb), fu = dfinite(ub);
        if (fl) {
            ++nfin;
            ds = smax(ds, fabs(lb));
        }
        if (fu) {
            ++nfin;
            ds = smax(ds, fabs(ub));
        }
        ds = smax(ds, fold_absmax(0.0, bneg(g[k])));  // inf_norm(b_k); inf_norm(r_k) = 0
        ds = smax(ds, fold_absmax(0.0, gX[k]));       // inf_norm(q_{k+1})
        dU[k] = 0.0;
        dX[k] = 0.0;
        mu[k] = 0.0;
        sl[k] = fl ? smax(1.0, fabs(lb)) : 0.0;
        nl[k] = fl ? 1.0 : 0.0;
        su[k] = fu ? smax(1.0, fabs(ub)) : 0.0;
        nu[k] = fu ? 1.0 : 0.0;
        rcl[k] = 0.0;
        rcu[k] = 0.0;
    }
    if (warp_any(bad)) return QP_DOMAIN;
    ds = warp_max_pos(ds);  // ds >= 1
    const int m = warp_sum_int(nfin);
    const double eps = tol * ds;
    __syncwarp();

    // rl, ru of stage k at the current iterate (qp.cpp:278-283)
    auto rlru = [&](int k, double u, bool fl, bool fu, double& rl, double& ru) {
        const double v = dU[k];
        rl = fl ? v - sl[k] - (umin - u) : 0.0;
        ru = fu ? (umax - u) - v - su[k] : 0.0;
    };

    int status = QP_MAXITER;
#pragma unroll 1
    for (int iter = 0;; ++iter) {
        // residuals() (qp.cpp:237-284); the gap terms go to TMP for the
        // ordered sums
        double ninf = 0.0, dinf = 0.0, linf = 0.0, uinf = 0.0;
#pragma unroll kUnrollQpLanes
        for (int k = lane; k < N; k += 32) {
            const double ju = Ju[k];
            const double vk = dU[k], muk = mu[k];
            const double dxp = k >= 1 ? dX[k - 1] : 0.0;
            double r = epi1(dot1(Wr[k], vk), 0.0);
            if (k >= 1) r = epi1(dot1(Wm[k], dxp), r);
            r = epim1(dot1(ju, muk), r);
            r += nu[k] - nl[k];
            rsu[k] = r;
            double rd = dX[k] + -1.0 * bneg(g[k]);
            if (k >= 1) rd = epim1(dot1(Jx[k], dxp), rd);
            rd = epim1(dot1(ju, vk), rd);
            rdyn[k] = rd;
            const int kk = k + 1;  // x row of stage k+1
            double rx = epi1(dot1(Wq[kk], dX[k]), gX[k]);
            if (kk < N) {
                rx = epi1(dot1(Wm[kk], dU[kk]), rx);
                rx = epim1(dot1(Jx[kk], mu[kk]), rx);
            }
            rx += muk;
            rsx[k] = rx;
            const double u = U[k];
            const bool fl = dfinite(umin - u), fu = dfinite(umax - u);
            double rl, ru;
            rlru(k, u, fl, fu, rl, ru);
            ninf = fold_absmax(fold_absmax(ninf, r), rx);
            dinf = fold_absmax(dinf, rd);
            linf = fold_absmax(linf, rl);
            uinf = fold_absmax(uinf, ru);
            const double slk = sl[k], suk = su[k], nlk = nl[k], nuk = nu[k];
            tmp[k] = slk * nlk;
            tmp[ST + k] = suk * nuk;
            // barrier diagonal + affine rc + condensed rhs of the next step
            // (qp.cpp:353-372, :288-305), computed speculatively: unused when
            // the iteration stops below
            double bk = 0.0;
            if (fl) bk += qdiv(nlk, slk);
            if (fu) bk += qdiv(nuk, suk);
            bar[k] = bk;
            const double cl = fl ? -slk * nlk : 0.0;
            const double cu = fu ? -suk * nuk : 0.0;
            rcl[k] = cl;
            rcu[k] = cu;
            double v = r;
            if (fl) v -= qdiv(cl - nlk * rl, slk);
            if (fu) v += qdiv(cu - nuk * ru, suk);
            rhat[k] = v;
        }
        // the inf-norms only meet "<= eps": max over lanes <= eps iff every
        // lane's partial max is (partials never hold NaN) -- one vote
        const bool res_ok = __all_sync(FULLMASK, ninf <= eps && dinf <= eps && linf <= eps && uinf <= eps);
        __syncwarp();
        // gap = (dot(sl, nl) + dot(su, nu)) / m: two serial chains, each lane
        // runs both (no shuffles)
        double gap;
        {
            double dl = 0.0, du = 0.0;
#pragma unroll 4
            for (int k = 0; k < N; ++k) {
                dl += tmp[k];
                du += tmp[ST + k];
            }
            gap = m > 0 ? (dl + du) / m : 0.0;
        }
        if (res_ok && gap <= eps) {
            status = QP_OPTIMAL;
            break;
        }
        if (iter >= max_iter) {
            status = QP_MAXITER;
            break;
        }
        // riccati_factor + affine solve (qp.cpp:358-372); the fast sweep's
        // certificate is checked inside the affine expand loop below
        bool npd = factor_sweep<ST, true>(o);
        bool fast_ok = !npd;
        if (npd) npd = factor_sweep<ST, false>(o);  // confirm a fast NPD with IEEE ops
        if (npd) {
            status = QP_FAILED;
            break;
        }
        rollout<ST>(N);
        // affine directions + step length, gap_aff, sigma (qp.cpp:367-386)
        double sigma = 0.0;
        {
            double alpha_aff = 1.0;
            for (int pass = 0;; ++pass) {
                bool cert = true;
                alpha_aff = 1.0;
#pragma unroll kUnrollQpLanes
                for (int k = lane; k < N; k += 32) {
                    if (fast_ok) cert = cert && certify_factor_k<ST>(o, k);
                    const double u = U[k];
                    const bool fl = dfinite(umin - u), fu = dfinite(umax - u);
                    double rl, ru;
                    rlru(k, u, fl, fu, rl, ru);
                    const Dir d = expand_k<ST>(o, k, fl, fu, rl, ru);
                    alpha_aff = step_caps<ST>(o, k, fl, fu, d, 1.0, alpha_aff);
                }
                if (!fast_ok || __all_sync(FULLMASK, cert)) break;
                // a fast sqrt/division was not the IEEE one: replay the
                // factor with IEEE ops (an NPD there is genuine) and redo
                __syncwarp();
                fast_ok = false;
                if (factor_sweep<ST, false>(o)) {
                    npd = true;
                    break;
                }
                rollout<ST>(N);
            }
            if (npd) {
                status = QP_FAILED;
                break;
            }
            alpha_aff = warp_min_pos(alpha_aff);  // step lengths lie in (0, 1]
            if (m > 0 && gap > 0.0) {
#pragma unroll kUnrollQpLanes
                for (int k = lane; k < N; k += 32) {
                    const double u = U[k];
                    const bool fl = dfinite(umin - u), fu = dfinite(umax - u);
                    const Dir d = load_dir<ST>(o, k);
                    tmp[k] = fl ? (sl[k] + alpha_aff * d.dsl) * (nl[k] + alpha_aff * d.dnl) : 0.0;
                    tmp[ST + k] = fu ? (su[k] + alpha_aff * d.dsu) * (nu[k] + alpha_aff * d.dnu) : 0.0;
                }
                __syncwarp();
                // terms of infinite bounds are stored as +0: adding +0 to this
                // sum of non-negative products (never -0) changes nothing
                double gap_aff = 0.0;
#pragma unroll 4
                for (int k = 0; k < N; ++k) {
                    gap_aff += tmp[k];
                    gap_aff += tmp[ST + k];
                }
                gap_aff /= m;
                const double ratio = smax(0.0, gap_aff / gap);
                sigma = smin(1.0, ratio * ratio * ratio);
            }
        }
        __syncwarp();
        // corrector rc + condensed rhs (qp.cpp:390-395, :288-305) from the
        // stored affine directions
#pragma unroll kUnrollQpLanes
        for (int k = lane; k < N; k += 32) {
            const double u = U[k];
            const bool fl = dfinite(umin - u), fu = dfinite(umax - u);
            double rl, ru;
            rlru(k, u, fl, fu, rl, ru);
            const Dir d = load_dir<ST>(o, k);
            const double slk = sl[k], suk = su[k], nlk = nl[k], nuk = nu[k];
            double cl = rcl[k], cu = rcu[k];
            if (fl) cl = sigma * gap - slk * nlk - d.dsl * d.dnl;
            if (fu) cu = sigma * gap - suk * nuk - d.dsu * d.dnu;
            rcl[k] = cl;
            rcu[k] = cu;
            double v = rsu[k];
            if (fl) v -= qdiv(cl - nlk * rl, slk);
            if (fu) v += qdiv(cu - nuk * ru, suk);
            rhat[k] = v;
        }
        __syncwarp();
        vector_sweep<ST, true>(o);
        rollout<ST>(N);
        // corrector directions + step length (qp.cpp:396-397), with the
        // certificate of the fast vector sweep
        double alpha = 1.0;
        for (bool vfast = true;; vfast = false) {
            bool cert = true;
            alpha = 1.0;
#pragma unroll kUnrollQpLanes
            for (int k = lane; k < N; k += 32) {
                if (vfast) cert = cert && certify_vector_k<ST>(o, k);
                const double u = U[k];
                const bool fl = dfinite(umin - u), fu = dfinite(umax - u);
                double rl, ru;
                rlru(k, u, fl, fu, rl, ru);
                const Dir d = expand_k<ST>(o, k, fl, fu, rl, ru);
                alpha = step_caps<ST>(o, k, fl, fu, d, tau, alpha);
            }
            if (!vfast || __all_sync(FULLMASK, cert)) break;
            __syncwarp();
            vector_sweep<ST, false>(o);
            rollout<ST>(N);
        }
        alpha = warp_min_pos(alpha);
        // update (qp.cpp:398-410)
#pragma unroll kUnrollQpLanes
        for (int k = lane; k < N; k += 32) {
            const double u = U[k];
            const bool fl = dfinite(umin - u), fu = dfinite(umax - u);
            const Dir d = load_dir<ST>(o, k);
            dU[k] = dU[k] + alpha * ddU[k];
            dX[k] = dX[k] + alpha * ddX[k];
            const double dmu = -(val[k + 1] * ddX[k] + pvec[k + 1]);  // qp.cpp:153
            mu[k] = mu[k] + alpha * dmu;
            if (fl) {
                sl[k] += alpha * d.dsl;
                nl[k] += alpha * d.dnl;
            }
            if (fu) {
                su[k] += alpha * d.dsu;
                nu[k] += alpha * d.dnu;
            }
        }
        cnt->ipm_stage += N;
        __syncwarp();
    }
    // final clamp (qp.cpp:414-419)
#pragma unroll kUnrollQpLanes
    for (int k = lane; k < N; k += 32) {
        const double lb = umin - U[k], ub = umax - U[k];
        dU[k] = smin(smax(dU[k], lb), ub);
    }
    __syncwarp();
    return status;
}

// ------------------------------------------------------------------ SQP
/// Lagrangian gradient pieces (sqp.cpp:102-128) at stage k.
/// hu = (0 - Ju_k lam_k) [+ (pi_u - pi_l)],
/// hx_k (slot x_{k+1}) = (gX_k + lam_k) - Jx_{k+1} lam_{k+1}.
__device__ __forceinline__ double lag_u(const double* Ju, const double* lam, int k) {
    return 0.0 - Ju[k] * lam[k];
}
__device__ __forceinline__ double lag_x(const double* gX, const double* Jx, const double* lam, int k, int N) {
    double h = gX[k] + lam[k];
    if (k + 1 < N) h -= Jx[k + 1] * lam[k + 1];
    return h;
}

/// check_convergence (sqp.cpp:86-96) of grad_l = lagrangian_gradient
/// (sqp.cpp:118-128) at the current evaluation with multipliers (lam, pl, pu).
template <int ST>
__device__ __noinline__ bool kkt_check(const Ocp& o, const double* lam, const double* pl, const double* pu, int m,
                                       double eps) {
    const int lane = threadIdx.x & 31;
    const int N = o.N;
    const double* gX = GA(G_GX);
    const double* g = GA(G_G);
    const double* Jx = SA(S_JX);
    const double* Ju = SA(S_JU);
    double* tmp = SA(S_TMP);
    double gl = 0.0, gi = 0.0;
#pragma unroll 1
    for (int k = lane; k < N; k += 32) {
        const double lk = lam[k], plk = pl[k], puk = pu[k];
        const double hu = (0.0 - Ju[k] * lk) + (puk - plk);
        const double hx = lag_x(gX, Jx, lam, k, N);
        gl = fold_absmax(fold_absmax(gl, hu), hx);
        gi = fold_absmax(gi, g[k]);
        tmp[k] = fabs(lk);
        tmp[ST + k] = fabs(plk);
        tmp[2 * ST + k] = fabs(puk);
    }
    __syncwarp();
    // mults = one_norm(lam) + one_norm(pi_l) + one_norm(pi_u): three serial
    // chains, all on every lane (no shuffles)
    double n1 = 0.0, n2 = 0.0, n3 = 0.0;
#pragma unroll 1
    for (int k = 0; k < N; ++k) {
        n1 += tmp[k];
        n2 += tmp[ST + k];
        n3 += tmp[2 * ST + k];
    }
    __syncwarp();
    double s_d = 1.0;
    if (m > 0) {
        const double mults = n1 + n2 + n3;
        s_d = smax(100.0, mults / m) / 100.0;
    }
    // max over lanes of gl, divided by s_d > 0, is <= eps iff every lane's is
    // (division by a positive number is monotone under rounding)
    return __all_sync(FULLMASK, gl / s_d <= eps && gi <= eps);
}

/// reset_blocks (sqp.cpp:173-178): identity Hessian blocks.
template <int ST>
__device__ __forceinline__ void reset_blocks(int N) {
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (int k = lane; k <= N; k += 32) {
        SA(S_WQ)[k] = 1.0;
        SA(S_WM)[k] = 0.0;
        SA(S_WR)[k] = 1.0;
    }
    __syncwarp();
}

static __device__ __noinline__ double qdiv(double a, double b);

/// bfgs_block_update (sqp.cpp:61-84) for a block of size n (1 or 2) stored as
/// (q, m, r) = (w00, w01 = w10, w11). Returns -1 on NotPositiveDefinite,
/// 0 if skipped, 1 if updated.
__device__ __forceinline__ int bfgs_block(double& q, double& mm, double& r, int n, const double* s,
                                          const double* y, bool uslot_only) {
    if (n == 1) {
        double& wv = uslot_only ? r : q;
        const double ws = epi0(dot1(wv, s[0]));
        const double sws = dot1(s[0], ws);
        if (!(sws > kEpsMach)) return 0;
        const double sy = dot1(s[0], y[0]);
        const double theta = sy >= 0.2 * sws ? 1.0 : qdiv(0.8 * sws, sws - sy);
        const double rr = theta * y[0] + (1.0 - theta) * ws;
        const double sr = dot1(s[0], rr);
        if (!(smin(sws, sr) > kEpsMach)) return 0;
        wv += qdiv(rr * rr, sr) - qdiv(ws * ws, sws);
        if (wv <= 0.0 || !dfinite(wv)) return -1;
        return 1;
    }
    const double ws0 = epi0(0.0 + q * s[0] + mm * s[1]);
    const double ws1 = epi0(0.0 + mm * s[0] + r * s[1]);
    const double sws = 0.0 + s[0] * ws0 + s[1] * ws1;
    if (!(sws > kEpsMach)) return 0;
    const double sy = 0.0 + s[0] * y[0] + s[1] * y[1];
    const double theta = sy >= 0.2 * sws ? 1.0 : qdiv(0.8 * sws, sws - sy);
    const double r0 = theta * y[0] + (1.0 - theta) * ws0;
    const double r1 = theta * y[1] + (1.0 - theta) * ws1;
    const double sr = 0.0 + s[0] * r0 + s[1] * r1;
    if (!(smin(sws, sr) > kEpsMach)) return 0;
    q += qdiv(r0 * r0, sr) - qdiv(ws0 * ws0, sws);
    mm += qdiv(r1 * r0, sr) - qdiv(ws1 * ws0, sws);  // w(1,0) == w(0,1): same products, commuted
    r += qdiv(r1 * r1, sr) - qdiv(ws1 * ws1, sws);
    mm = 0.5 * (mm + mm);                  // symmetrize
    // cholesky_factor audit (linalg.cpp:69-103)
    if (q <= 0.0 || !dfinite(q)) return -1;
    const double l00 = sqrt(q);
    const double l10 = qdiv(mm, l00);
    const double d = r - l10 * l10;
    if (d <= 0.0 || !dfinite(d)) return -1;
    return 1;
}

struct SqpOut {
    bool converged;
    int status;  // ST_OK or ST_DOMAIN (propagating)
};

/// Merit update, line search, acceptance and BFGS of one SQP iteration
/// (sqp.cpp:312-406). Returns 0 = continue, 1 = break (exhausted with no
/// finite trial), ST_DOMAIN << 4 = DomainError escaped.
template <int ST>
__device__ __noinline__ int sqp_step(const Ocp& o, const nmpcmc_sqp_options& opt, double* f, bool first_merit,
                                     Cnt* cnt) {
    const int lane = threadIdx.x & 31;
    const int N = o.N;
    double* U = GA(G_U);
    double* X = GA(G_X);
    double* tU = GA(G_TU);
    double* tX = GA(G_TX);
    double* lam = GA(G_LAM);
    double* pil = GA(G_PIL);
    double* piu = GA(G_PIU);
    double* gX = GA(G_GX);
    double* g = GA(G_G);
    double* tgX = GA(G_TGX);
    double* tg = GA(G_TG);
    double* tJx = GA(G_TJX);
    double* tJu = GA(G_TJU);
    double* Jx = SA(S_JX);
    double* Ju = SA(S_JU);
    double* sig = GA(G_SIG);
    double* tmp = SA(S_TMP);
    const double* dU = IA(I_DU);
    const double* dX = IA(I_DX);
    const double* mu = IA(I_MU);
    const double* nl = IA(I_NL);
    const double* nu = IA(I_NU);
    // merit_weights_update (sqp.cpp:12-20) + line_search terms (sqp.cpp:28-31)
    bool du_bad = false;
#pragma unroll 1
    for (int k = lane; k < N; k += 32) {
        const double am = fabs(mu[k]);
        const double sg = first_merit ? am : smax(am, 0.5 * (sig[k] + am));
        sig[k] = sg;
        tmp[k] = sg * fabs(g[k]);
        tmp[ST + k] = gX[k] * dX[k];
        du_bad |= !dfinite(dU[k]);
    }
    du_bad = warp_any(du_bad);
    __syncwarp();
    double penalty0, dd;
    {
        // two serial chains (even/odd lanes): penalty0 and dot(grad f, dxi);
        // the u slots contribute 0 * du (exactly +-0) unless du is not finite
        double s0 = 0.0, s1 = 0.0;
#pragma unroll 1
        for (int k = 0; k < N; ++k) {
            s0 += tmp[k];
            s1 += tmp[ST + k];
        }
        penalty0 = s0;
        const double dot_gd = du_bad ? kNaN : s1;
        dd = dot_gd - penalty0;
        __syncwarp();
    }
    const double merit_before = *f + penalty0;
    double alpha = 1.0, merit = 0.0, f_trial = 0.0;
    bool ok = false;
#pragma unroll 1
    for (int bt = 0;; ++bt) {
#pragma unroll 1
        for (int k = lane; k < N; k += 32) {
            tU[k] = U[k] + alpha * dU[k];
            tX[k] = X[k] + alpha * dX[k];
        }
        __syncwarp();
        f_trial = eval_objective<ST>(o, tX, tgX);
        const int st = eval_constraints<ST>(o, tU, tX, tg, tJx, tJu, cnt);
        if (st == ST_DOMAIN) return ST_DOMAIN << 4;
        merit = HUGE_VAL;
        if (st == ST_OK) {
#pragma unroll 1
            for (int k = lane; k < N; k += 32) tmp[k] = sig[k] * fabs(tg[k]);
            __syncwarp();
            merit = f_trial;
#pragma unroll 1
            for (int k = 0; k < N; ++k) merit += tmp[k];
            __syncwarp();
        }
        cnt->ls += 1;
        ok = dfinite(merit) && merit <= merit_before + opt.c1 * alpha * dd;
        if (ok || bt >= opt.max_backtracks) break;
        alpha *= opt.backtrack_factor;
    }
    if (!ok && !dfinite(merit)) return 1;  // exhausted with no finite trial

    // accept: xi_new = xi + a dxi equals the last trial bitwise, and so do f,
    // grad f and the constraint blocks (sqp.cpp:331-352)
    const double a = alpha;
#pragma unroll 1
    for (int k = lane; k < N; k += 32) {
        U[k] = tU[k];
        X[k] = tX[k];
        lam[k] += a * (mu[k] - lam[k]);
        pil[k] += a * (nl[k] - pil[k]);
        piu[k] += a * (nu[k] - piu[k]);
    }
    __syncwarp();
    // damped block BFGS on (s, y) with y = h_new - h_old (sqp.cpp:362-400)
    bool lost = false;
    double* Wq = SA(S_WQ);
    double* Wm = SA(S_WM);
    double* Wr = SA(S_WR);
#pragma unroll 1
    for (int blk = lane; blk <= N; blk += 32) {
        double s[2], y[2];
        int n;
        bool uonly = false;
        if (blk == 0) {
            n = 1;
            uonly = true;
            s[0] = a * dU[0];
            y[0] = lag_u(tJu, lam, 0) - lag_u(Ju, lam, 0);
        } else if (blk < N) {
            n = 2;
            s[0] = a * dX[blk - 1];
            s[1] = a * dU[blk];
            y[0] = lag_x(tgX, tJx, lam, blk - 1, N) - lag_x(gX, Jx, lam, blk - 1, N);
            y[1] = lag_u(tJu, lam, blk) - lag_u(Ju, lam, blk);
        } else {
            n = 1;
            s[0] = a * dX[N - 1];
            y[0] = lag_x(tgX, tJx, lam, N - 1, N) - lag_x(gX, Jx, lam, N - 1, N);
        }
        double q = Wq[blk], mm = Wm[blk], r = Wr[blk];
        const int res = bfgs_block(q, mm, r, n, s, y, uonly);
        if (res < 0) lost = true;
        if (res > 0) {
            Wq[blk] = q;
            Wm[blk] = mm;
            Wr[blk] = r;
        }
    }
    lost = warp_any(lost);
    __syncwarp();
    if (lost) reset_blocks<ST>(N);
    // the trial evaluation becomes the current one
#pragma unroll 1
    for (int k = lane; k < N; k += 32) {
        gX[k] = tgX[k];
        g[k] = tg[k];
        Jx[k] = tJx[k];
        Ju[k] = tJu[k];
    }
    __syncwarp();
    *f = f_trial;
    cnt->sqp += 1;
    return 0;
}

/// sqp_solve (sqp.cpp:182-411) on the iterate in (U, X) with duals in
/// LAM/PIL/PIU (already warm-started).
template <int ST>
__device__ __noinline__ SqpOut sqp_solve(const Ocp& o, const nmpcmc_sqp_options& opt, Cnt* cnt) {
    const int lane = threadIdx.x & 31;
    const int N = o.N;
    SqpOut out{false, ST_OK};
    const int m = N + (dfinite(o.umin) ? N : 0) + (dfinite(o.umax) ? N : 0);
    reset_blocks<ST>(N);
    bool first_merit = true;

    // initial evaluation: NonFiniteState -> unconverged return (sqp.cpp:238-246)
    double f = eval_objective<ST>(o, GA(G_X), GA(G_GX));
    const int st = eval_constraints<ST>(o, GA(G_U), GA(G_X), GA(G_G), SA(S_JX), SA(S_JU), cnt);
    if (st == ST_DOMAIN) return SqpOut{false, ST_DOMAIN};
    if (st == ST_NONFINITE) return out;

#pragma unroll 1
    for (int iter = 0;; ++iter) {
        if (kkt_check<ST>(o, GA(G_LAM), GA(G_PIL), GA(G_PIU), m, opt.eps)) {
            out.converged = true;
            break;
        }
        if (iter >= opt.max_iter) break;
        cnt->sqp_stage += N;
        // QP, with one identity-reset salvage attempt (sqp.cpp:263-278)
        int qs = QP_FAILED;
#pragma unroll 1
        for (int attempt = 0; attempt < 2; ++attempt) {
            if (attempt == 1) reset_blocks<ST>(N);
            qs = solve_qp<ST>(o, opt.qp_tol, opt.qp_max_iter, cnt);
            cnt->qp += 1;
            if (qs != QP_FAILED) break;
        }
        if (qs == QP_DOMAIN) return SqpOut{false, ST_DOMAIN};
        if (qs == QP_FAILED) break;  // rep.qp_failed
        // KKT certificate with the fresh QP multipliers (sqp.cpp:285-310)
        if (kkt_check<ST>(o, IA(I_MU), IA(I_NL), IA(I_NU), m, opt.eps)) {
#pragma unroll 1
            for (int k = lane; k < N; k += 32) {
                GA(G_LAM)[k] = IA(I_MU)[k];
                GA(G_PIL)[k] = IA(I_NL)[k];
                GA(G_PIU)[k] = IA(I_NU)[k];
            }
            __syncwarp();
            out.converged = true;
            break;
        }
        const int r = sqp_step<ST>(o, opt, &f, first_merit, cnt);
        first_merit = false;
        if (r == (ST_DOMAIN << 4)) return SqpOut{false, ST_DOMAIN};
        if (r == 1) break;
    }
    return out;
}

// ------------------------------------------------------------ closed loop
/// Warm/cold start of the SQP iterate (controllers.cpp:147-186) into U, X and
/// the duals. Returns ST_DOMAIN if a DomainError escapes.
template <int ST>
__device__ __noinline__ int start_iterate(const Ocp& o, bool warm, Cnt* cnt) {
    const int lane = threadIdx.x & 31;
    const int N = o.N;
    double* U = GA(G_U);
    double* X = GA(G_X);
    double* nU = GA(G_TU);
    double* nX = GA(G_TX);
    double* tmp = SA(S_TMP);
    double* lam = GA(G_LAM);
    double* pil = GA(G_PIL);
    double* piu = GA(G_PIU);
    const bool fl = dfinite(o.umin), fh = dfinite(o.umax);
    const double u_nom = fl && fh ? 0.5 * (o.umin + o.umax) : smax(o.umin, smin(o.umax, 0.0));
    // u sequence: shifted_inputs (controllers.cpp:70-83) or nominal_input (:58-66)
#pragma unroll 1
    for (int k = lane; k < N; k += 32)
        nU[k] = warm ? smax(o.umin, smin(o.umax, U[min(k + 1, N - 1)])) : u_nom;
    __syncwarp();
    const int st = xi_from_inputs<ST>(o, nU, nX, cnt);
    if (st == ST_DOMAIN) return ST_DOMAIN;
    if (st == ST_OK) {
#pragma unroll 1
        for (int k = lane; k < N; k += 32) {
            U[k] = nU[k];
            X[k] = nX[k];
        }
    } else if (warm) {
        // shifted_warm_start (controllers.cpp:97-110)
#pragma unroll 1
        for (int k = lane; k < N; k += 32) nX[k] = X[min(k + 1, N - 1)];
        __syncwarp();
#pragma unroll 1
        for (int k = lane; k < N; k += 32) {
            U[k] = nU[k];
            X[k] = nX[k];
        }
    } else {
        // flat guess (controllers.cpp:173-185)
#pragma unroll 1
        for (int k = lane; k < N; k += 32) {
            U[k] = u_nom;
            X[k] = o.x0;
        }
    }
    __syncwarp();
    if (warm) {
        // shifted_multipliers (controllers.cpp:87-93); sqp_solve then projects
        // the warm bound multipliers onto >= 0 (sqp.cpp:219-222)
#pragma unroll 1
        for (int k = lane; k < N; k += 32) {
            const int src = N >= 2 ? min(k + 1, N - 1) : k;
            tmp[k] = lam[src];
            tmp[ST + k] = pil[src];
            tmp[2 * ST + k] = piu[src];
        }
        __syncwarp();
#pragma unroll 1
        for (int k = lane; k < N; k += 32) {
            lam[k] = tmp[k];
            pil[k] = smax(0.0, tmp[ST + k]);
            piu[k] = smax(0.0, tmp[2 * ST + k]);
        }
    } else {
#pragma unroll 1
        for (int k = lane; k < N; k += 32) {
            lam[k] = 0.0;
            pil[k] = 0.0;
            piu[k] = 0.0;
        }
    }
    __syncwarp();
    return ST_OK;
}

/// filter_update (ekf.cpp:59-96), one-state, with nmpc_step's jitter retry
/// (controllers.cpp:123-132): posterior (xf, Pn) from the prediction (xhat,
/// Pf) and y; innov = y - c xhat. ST_NPD when the jittered innovation
/// covariance is still not positive definite.
__device__ __forceinline__ int filter_update1(const Ocp& o, double R_filter, double y, double xhat, double Pf,
                                              double& xf, double& Pn, double* innov = nullptr) {
    const double c = o.inv_V;
    const double e = y - xhat / o.p.V;
    if (innov) *innov = e;
    const double pc = epi0(dot1(Pf, c));
    double Rr = R_filter;
    double Re = epi1(dot1(c, pc), Rr);
    if (Re <= 0.0 || !dfinite(Re)) {
        Rr = Rr + 1e-10;
        Re = epi1(dot1(c, pc), Rr);
        if (Re <= 0.0 || !dfinite(Re)) return ST_NPD;
    }
    const double l = sqrt(Re);
    double K = pc / l;
    K = K / l;
    xf = epi1(dot1(K, e), xhat);
    const double ikc = epim1(dot1(K, c), 1.0);
    const double ikc_p = epi0(dot1(ikc, Pf));
    Pn = epi0(dot1(ikc_p, ikc));
    const double kr = epi0(dot1(K, Rr));
    Pn = epi1(dot1(kr, K), Pn);
    return ST_OK;
}

/// predict (ekf.cpp:26-57), one-state: np RK4 steps on (x, P) over
/// [t, t + Ts] under input u, in place.
__device__ __forceinline__ int predict1(const Ocp& o, double t, int np, double u, double& x, double& P) {
    const double t_next = t + o.Ts;
    const double h = (t_next - t) / np;
    int st = ST_OK;
#pragma unroll 1
    for (int s = 0; s < np && st == ST_OK; ++s) {
        // RK4 stages at (x, P) + c h k_{j-1}, c = 0, 1/2, 1/2, 1, with
        // 0.5 * h * k formed as (0.5 * h) * k (ekf.cpp:38-44); the
        // weighted sum accumulates left to right (ekf.cpp:46-50)
        double pkx = 0.0, pkp = 0.0, ax = 0.0, ap = 0.0;
#pragma unroll 1
        for (int j = 0; j < 4 && st == ST_OK; ++j) {
            double xs = x, ps = P;
            if (j == 1 || j == 2) {
                xs = x + 0.5 * h * pkx;
                ps = P + 0.5 * h * pkp;
            } else if (j == 3) {
                xs = x + h * pkx;
                ps = P + h * pkp;
            }
            double kx, kp;
            st = joint_rhs1(o.p, xs, ps, u, kx, kp);
            if (j == 0) {
                ax = kx;
                ap = kp;
            } else if (j < 3) {
                ax = ax + 2.0 * kx;
                ap = ap + 2.0 * kp;
            } else {
                ax = ax + kx;
                ap = ap + kp;
            }
            pkx = kx;
            pkp = kp;
        }
        if (st != ST_OK) break;
        x += (h / 6.0) * ax;
        P += (h / 6.0) * ap;
        if (!dfinite(x) || !dfinite(P)) st = ST_NONFINITE;
    }
    return st;
}

/// The NMPC branch of run_closed_loop (montecarlo.cpp:80-157) for one sample.
template <int NX, int ST>
__device__ __noinline__ void nmpc_closed_loop(const nmpcmc_scenario& sc, uint64_t sim_index, int nbar, double* gws,
                                              nmpcmc_sim_record* rec, nmpcmc_work_counters* cntp, double* traj) {
    const int lane = threadIdx.x & 31;
    const Cstr p = sample_truth(sc, sim_index);
    NormalStream rng;
    rng.init(sc.base_seed, sim_index);
    Plant<NX> pl;
#pragma unroll
    for (int i = 0; i < NX; ++i) pl.x[i] = sc.x0[i];
    const bool has_R = sc.has_noise_R != 0;
    const double lR = has_R ? chol_semidef_1x1(sc.noise_R) : 0.0;
    const int stride = sc.record_stride < 1 ? 1 : sc.record_stride;
    const bool record = traj != nullptr;

    Ocp o;
    o.p = load_cstr(sc.ctrl);
    o.N = sc.N;
    o.Nc = sc.Nc;
    o.Ts = sc.horizon_Ts;
    o.h = sc.horizon_Ts / sc.Nc;
    o.umin = sc.u_min;
    o.umax = sc.u_max;
    o.Qz = sc.Qz;
    o.inv_V = 1.0 / o.p.V;
    o.x0 = 0.0;
    o.gws = gws;
    const int N = o.N;
    Cnt cnt = {};

    // NmpcState (make_nmpc_state, controllers.cpp:25-48)
    double xhat = sc.x0_hat[0], Pf = sc.P0[0];
    bool have_last = false;  // last_xi empty -> cold start

    double t = sc.t0;
    double z = pl.x[NX - 1] / p.V;
    double zbar = setpoint_at(sc, t);
    double acc = 0.0;
    {
        const double r = z - zbar;
        acc += r * r;
    }
    int status = ST_OK;
    bool counts_lost = false;
    int ocp_solves = 0, ocp_failures = 0;
    int row = 0;

#pragma unroll 1
    for (int i = 0; i < nbar; ++i) {
        const double y = measure<NX>(p, pl, has_R, lR, rng);
        // ---- nmpc_step (controllers.cpp:114-212)
        if (!dfinite(y)) {
            status = ST_NONFINITE;
            break;
        }
#pragma unroll 1
        for (int k = lane; k < N; k += 32) GA(G_SP)[k] = setpoint_at(sc, t + (k + 1) * sc.Ts);
        // filter_update (ekf.cpp:59-96) with the jitter retry (controllers.cpp:123-132)
        double xf, Pn;
        if (filter_update1(o, sc.R_filter, y, xhat, Pf, xf, Pn) != ST_OK) {
            status = ST_NPD;
            counts_lost = true;
            break;
        }
        o.x0 = xf;
        __syncwarp();
        if (start_iterate<ST>(o, have_last, &cnt) == ST_DOMAIN) {
            status = ST_DOMAIN;
            break;
        }
        const SqpOut so = sqp_solve<ST>(o, sc.sqp, &cnt);
        if (so.status != ST_OK) {
            status = so.status;
            break;
        }
        const double u = smax(o.umin, smin(o.umax, GA(G_U)[0]));
        have_last = true;
        // predict (ekf.cpp:26-57), np RK4 steps on (x, P)
        {
            double x = xf, P = Pn;
            const int st = predict1(o, t, sc.np, u, x, P);
            if (st != ST_OK) {
                status = st;
                break;
            }
            xhat = x;
            Pf = P;
        }
        ++ocp_solves;
        if (!so.converged) ++ocp_failures;
        cnt.steps += 1;
        // ---- back in run_closed_loop
        if (record && i % stride == 0) {
            if (lane == 0) {
                double* rw = traj + (size_t)row * 5;
                rw[0] = t;
                rw[1] = z;
                rw[2] = zbar;
                rw[3] = u;
                rw[4] = y;
            }
            ++row;
        }
        status = simulate_interval<NX>(p, pl, t, t + sc.Ts, u, sc.Ns, rng);
        if (status != ST_OK) break;
        t = sc.t0 + (i + 1) * sc.Ts;
        z = pl.x[NX - 1] / p.V;
        zbar = setpoint_at(sc, t);
        const double r = z - zbar;
        acc += r * r;
        __syncwarp();
    }
    if (lane == 0) {
        if (status == ST_OK) {
            rec->phi = acc / (double)(nbar + 1);
            rec->failed = 0;
            if (record) {
                double* rw = traj + (size_t)row * 5;
                rw[0] = t;
                rw[1] = z;
                rw[2] = zbar;
                rw[3] = kNaN;
                rw[4] = kNaN;
            }
        } else {
            rec->phi = kNaN;
            rec->failed = 1;
        }
        // a NotPositiveDefinite escaping run_closed_loop is caught by
        // run_monte_carlo's catch(...) with a fresh record (montecarlo.cpp:228-236)
        rec->ocp_solves = counts_lost ? 0 : ocp_solves;
        rec->ocp_failures = counts_lost ? 0 : ocp_failures;
        rec->status = status;
        if (cntp != nullptr) {
            nmpcmc_work_counters c;
            c.control_steps = cnt.steps;
            c.shoot_full = cnt.shoot_full;
            c.shoot_fonly = cnt.shoot_fonly;
            c.ipm_stage_iters = cnt.ipm_stage;
            c.sqp_stage_iters = cnt.sqp_stage;
            c.qp_solves = cnt.qp;
            c.sqp_iterations = cnt.sqp;
            c.ls_evals = cnt.ls;
            *cntp = c;
        }
    }
    __syncwarp();
}

/// Persistent blocks (one warp, one sample at a time) pull sample indices
/// from a global atomic counter -- the device form of run_monte_carlo's worker
/// pool (montecarlo.cpp:218-238) -- so long and short samples balance.
// Resident one-warp blocks per SM the kernel is compiled for. 12 (168
// registers, 3 warps per SM sub-partition) beats 16 (128 registers) by 4 %,
// and 13 / 14 (152 / 144 registers), 11 (184) and 8 (236) are no better
// (profiles/r02/r02T_k3_minblocks_ab.txt): fewer spills per warp; the larger
// L1 that fewer blocks leave is not what pays (same file, TMP-alias run).
// At the short stride (N < 32: one round of every stage loop) 16 still wins
// by 8 % (r02b2_k3_minblocks_other_N.txt); N = 120 gains 6 % at 12.
#ifndef NMPCMC_MIN_BLOCKS
#define NMPCMC_MIN_BLOCKS 12
#endif
#ifndef NMPCMC_MIN_BLOCKS_SHORT
#define NMPCMC_MIN_BLOCKS_SHORT 16
#endif
__host__ __device__ constexpr int k3_min_blocks(int stride) {
    return stride <= 32 ? NMPCMC_MIN_BLOCKS_SHORT : NMPCMC_MIN_BLOCKS;
}
template <int NX, int ST>
#ifdef NMPCMC_K3_MAXNREG
__global__ void __maxnreg__(NMPCMC_K3_MAXNREG) nmpc_kernel(
#else
__global__ void __launch_bounds__(32, k3_min_blocks(ST)) nmpc_kernel(
#endif
const __grid_constant__ nmpcmc_scenario sc, uint64_t first_sim,
                                                  int64_t n_sims, int nbar, nmpcmc_sim_record* records,
                                                  nmpcmc_work_counters* counters, double* traj, int traj_rows,
                                                  double* gws_all, unsigned long long* next) {
    double* gws = gws_all + (size_t)blockIdx.x * glob_arrays(ST) * ST;
#pragma unroll 1
    for (;;) {
        unsigned long long i = 0;
        if ((threadIdx.x & 31) == 0) i = atomicAdd(next, 1ULL);
        i = __shfl_sync(FULLMASK, i, 0);
        if (i >= (unsigned long long)n_sims) break;
        nmpc_closed_loop<NX, ST>(sc, first_sim + i, nbar, gws, records + i, counters ? counters + i : nullptr,
                                 traj ? traj + (size_t)i * traj_rows * 5 : nullptr);
    }
}

/// Resident blocks per SM for the K3 kernel of stride ST (occupancy query).
template <int NX, int ST>
inline int nmpc_blocks_per_sm() {
    const size_t smem = ws_bytes_for(ST);
    cudaFuncSetAttribute(nmpc_kernel<NX, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, nmpc_kernel<NX, ST>, 32, smem);
    return b < 1 ? 1 : b;
}

template <int NX, int ST>
inline int launch_nmpc_t(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
                         nmpcmc_work_counters* d_cnt, double* d_traj, int rows, int sm_count, double* gws,
                         int64_t gws_blocks, unsigned long long* counter, cudaStream_t stream) {
    const size_t smem = ws_bytes_for(ST);
    int64_t grid = (int64_t)sm_count * nmpc_blocks_per_sm<NX, ST>();
    if (grid > n) grid = n;
    if (grid > gws_blocks) return NMPCMC_INVALID_ARGUMENT;
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
    nmpc_kernel<NX, ST><<<(unsigned)grid, 32, smem, stream>>>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, gws,
                                                              counter);
    return NMPCMC_OK;
}

/// Global workspace bytes and block count K3 needs on this device.
inline void nmpc_gws_need(const nmpcmc_scenario& sc, int sm_count, int64_t n, size_t* bytes, int64_t* blocks) {
    const int ST = ws_stride_for(sc.N);
    const bool three = sc.truth_variant == NMPCMC_THREE_STATE;
    int per = 1;
    switch (ST) {
        case 32: per = three ? nmpc_blocks_per_sm<3, 32>() : nmpc_blocks_per_sm<1, 32>(); break;
        case 64: per = three ? nmpc_blocks_per_sm<3, 64>() : nmpc_blocks_per_sm<1, 64>(); break;
        case 128: per = three ? nmpc_blocks_per_sm<3, 128>() : nmpc_blocks_per_sm<1, 128>(); break;
        default: per = three ? nmpc_blocks_per_sm<3, 256>() : nmpc_blocks_per_sm<1, 256>(); break;
    }
    int64_t b = (int64_t)sm_count * per;
    if (b > n) b = n;
    if (b < 1) b = 1;
    *blocks = b;
    *bytes = (size_t)b * gws_bytes_for(ST);
}

inline int launch_nmpc(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
                       nmpcmc_work_counters* d_cnt, double* d_traj, int rows, int sm_count, double* gws,
                       int64_t gws_blocks, unsigned long long* counter, cudaStream_t stream) {
    if (sc.ctrl_variant != NMPCMC_ONE_STATE) return NMPCMC_UNSUPPORTED;
    if (sc.N < 1 || sc.N > 255) return NMPCMC_UNSUPPORTED;
    const int ST = ws_stride_for(sc.N);
    const bool three = sc.truth_variant == NMPCMC_THREE_STATE;
#define NMPCMC_K3_CASE(S)                                                                                      \
    if (ST == S)                                                                                              \
        return three ? launch_nmpc_t<3, S>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, sm_count, gws,       \
                                           gws_blocks, counter, stream)                                       \
                     : launch_nmpc_t<1, S>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, sm_count, gws,       \
                                           gws_blocks, counter, stream);
    NMPCMC_K3_CASE(32)
    NMPCMC_K3_CASE(64)
    NMPCMC_K3_CASE(128)
    NMPCMC_K3_CASE(256)
#undef NMPCMC_K3_CASE
    return NMPCMC_UNSUPPORTED;
}

/// Batched OCP service on K3's phases (one-state controller model, N <= 255):
/// for instance b, sqp_solve on the regulator OCP from x0[b] at t0[b], cold
/// start as nmpc_step (start_iterate) or the given xi0 with zero duals. The
/// iterate is scattered back to the interleaved xi layout (u_k, x_{k+1}).
// The OCP service keeps the round-1 residency (16 warps per SM, 128 registers):
// at 20,000 instances 12 and 16 measure the same within the run-to-run spread
// of the service benchmark (257k-284k OCPs/s, profiles/r02/r02N, r02Y, r02a2).
#ifndef NMPCMC_OCP1_MIN_BLOCKS
#define NMPCMC_OCP1_MIN_BLOCKS 16
#endif
template <int ST>
__global__ void __launch_bounds__(32, NMPCMC_OCP1_MIN_BLOCKS)
    ocp1_kernel(const __grid_constant__ nmpcmc_scenario sc, int64_t batch, const double* x0, const double* t0,
                const double* xi0, double* xi_out, double* lam_out, double* pil_out, double* piu_out,
                int32_t* conv_out, int32_t* status_out, double* gws_all, unsigned long long* next) {
    double* gws = gws_all + (size_t)blockIdx.x * glob_arrays(ST) * ST;
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (;;) {
        unsigned long long bi = 0;
        if (lane == 0) bi = atomicAdd(next, 1ULL);
        bi = __shfl_sync(FULLMASK, bi, 0);
        if (bi >= (unsigned long long)batch) break;
        const int64_t b = (int64_t)bi;
        Ocp o;
        o.p = load_cstr(sc.ctrl);
        o.N = sc.N;
        o.Nc = sc.Nc;
        o.Ts = sc.horizon_Ts;
        o.h = sc.horizon_Ts / sc.Nc;
        o.umin = sc.u_min;
        o.umax = sc.u_max;
        o.Qz = sc.Qz;
        o.inv_V = 1.0 / o.p.V;
        o.x0 = x0[b];
        o.gws = gws;
        const int N = o.N;
        Cnt cnt = {};
#pragma unroll 1
        for (int k = lane; k < N; k += 32) GA(G_SP)[k] = setpoint_at(sc, t0[b] + (k + 1) * sc.Ts);
        __syncwarp();
        int st = ST_OK;
        if (xi0 != nullptr) {
#pragma unroll 1
            for (int k = lane; k < N; k += 32) {
                GA(G_U)[k] = xi0[b * 2 * N + 2 * k];
                GA(G_X)[k] = xi0[b * 2 * N + 2 * k + 1];
                GA(G_LAM)[k] = 0.0;
                GA(G_PIL)[k] = 0.0;
                GA(G_PIU)[k] = 0.0;
            }
            __syncwarp();
        } else {
            st = start_iterate<ST>(o, false, &cnt);
        }
        SqpOut so{false, st};
        if (st == ST_OK) so = sqp_solve<ST>(o, sc.sqp, &cnt);
        const bool ok = so.status == ST_OK;
#pragma unroll 1
        for (int k = lane; k < N; k += 32) {
            xi_out[b * 2 * N + 2 * k] = ok ? GA(G_U)[k] : 0.0;
            xi_out[b * 2 * N + 2 * k + 1] = ok ? GA(G_X)[k] : 0.0;
            lam_out[b * N + k] = ok ? GA(G_LAM)[k] : 0.0;
            pil_out[b * N + k] = ok ? GA(G_PIL)[k] : 0.0;
            piu_out[b * N + k] = ok ? GA(G_PIU)[k] : 0.0;
        }
        if (lane == 0) {
            conv_out[b] = ok && so.converged ? 1 : 0;
            status_out[b] = ok ? 0 : so.status;
        }
        __syncwarp();
    }
}

template <int ST>
inline int launch_ocp1_t(const nmpcmc_scenario& sc, int64_t batch, const double* x0, const double* t0,
                         const double* xi0, double* xi, double* lam, double* pil, double* piu, int32_t* conv,
                         int32_t* status, int sm_count, double* gws, int64_t gws_blocks, unsigned long long* counter,
                         cudaStream_t stream) {
    const size_t smem = ws_bytes_for(ST);
    cudaFuncSetAttribute(ocp1_kernel<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ocp1_kernel<ST>, 32, smem);
    int64_t grid = (int64_t)sm_count * (per < 1 ? 1 : per);
    if (grid > batch) grid = batch;
    if (grid > gws_blocks) grid = gws_blocks;
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
    ocp1_kernel<ST><<<(unsigned)grid, 32, smem, stream>>>(sc, batch, x0, t0, xi0, xi, lam, pil, piu, conv, status,
                                                          gws, counter);
    return NMPCMC_OK;
}
/// One-state OCP batches on K3's phases; returns NMPCMC_UNSUPPORTED otherwise.
inline int launch_ocp1(const nmpcmc_scenario& sc, int64_t batch, const double* x0, const double* t0,
                       const double* xi0, double* xi, double* lam, double* pil, double* piu, int32_t* conv,
                       int32_t* status, int sm_count, double* gws, int64_t gws_blocks, unsigned long long* counter,
                       cudaStream_t stream) {
    if (sc.ctrl_variant != NMPCMC_ONE_STATE || sc.N < 1 || sc.N > 255) return NMPCMC_UNSUPPORTED;
    switch (ws_stride_for(sc.N)) {
        case 32: return launch_ocp1_t<32>(sc, batch, x0, t0, xi0, xi, lam, pil, piu, conv, status, sm_count, gws,
                                          gws_blocks, counter, stream);
        case 64: return launch_ocp1_t<64>(sc, batch, x0, t0, xi0, xi, lam, pil, piu, conv, status, sm_count, gws,
                                          gws_blocks, counter, stream);
        case 128: return launch_ocp1_t<128>(sc, batch, x0, t0, xi0, xi, lam, pil, piu, conv, status, sm_count, gws,
                                            gws_blocks, counter, stream);
        default: return launch_ocp1_t<256>(sc, batch, x0, t0, xi0, xi, lam, pil, piu, conv, status, sm_count, gws,
                                           gws_blocks, counter, stream);
    }
}

#undef SA
#undef GA
#undef CA
#undef IA

}  // namespace nmpcmc_dev
