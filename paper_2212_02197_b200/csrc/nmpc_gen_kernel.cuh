// nmpc_gen_kernel.cuh -- K3g / K3w: NMPC closed loop for a controller model
// of any state dimension NX (compile time). W = lanes per sample: W = 1 is
// K3g (one thread per sample), W = 32 is K3w (one warp per sample: stage
// loops across lanes, Riccati sweeps and ordered sums serial on every lane).
//
// K3 (nmpc_kernel.cuh) is the one-state fast path. K3g covers the
// three-state controller model: the literal "CD-EKF on the 3-state model"
// reading of BASELINE config 2, and SURVEY.md §8(f) row 3. It restates the
// reference's NMPC branch for general n_x with n_u = n_y = n_z = 1:
//   run_closed_loop      montecarlo.cpp:80-157
//   nmpc_step            controllers.cpp:114-212
//   filter_update        ekf.cpp:59-96      predict / joint_rhs  ekf.cpp:12-57
//   drift / jacobians    cstr.cpp:36-53, :99-127
//   shoot                ocp.cpp:9-74       eval_objective / eval_constraints  ocp.cpp:76-135
//   xi_from_inputs       ocp.cpp:137-154
//   sqp_solve            sqp.cpp:12-411     solve_qp  qp.cpp:66-423
//   gemm/gemv/cholesky   linalg.cpp:69-235 (loop orders and epilogues)
// keeping every floating-point operation in the reference's order, so the
// records are bitwise those of the exact-libm reference (tests/test_gpu_gen.py).
//
// Layout: a per-sample workspace of ~9k doubles (N = 60, NX = 3) in global
// memory. K3g: element e of slot t at ws[e * T + t] (T = resident slots), so
// the 32 lanes of a warp touch 32 consecutive doubles. K3w: one contiguous
// slab per warp (T = 1), lanes touching consecutive stages. Small matrices
// (NX x NX) live in registers. Reference exceptions become status codes
// returned to exactly the callers that catch them. In K3w every serial
// section runs redundantly on all lanes and only ever stores (no
// read-modify-write of a shared slot); order-independent reductions (inf
// norms, step minima, counts) combine per-lane partials with std::max/min
// semantics; ordered sums stay serial.
#pragma once

#include "certified_math.cuh"
#include "device_common.cuh"

namespace nmpcmc_dev {
namespace gen {

enum : int { G_OK = 0, G_NPD = ST_NPD, G_NONFINITE = ST_NONFINITE, G_DOMAIN = ST_DOMAIN };

/// View of one sample's workspace. K3g (W = 1): SoA across slots, element e
/// at p[e * T]; K3w (W = 32): one contiguous slab, element e at p[e] -- the
/// stride is a compile-time 1 and offsets are 32-bit, so an access is one
/// integer add instead of a 64-bit multiply chain.
template <int W>
struct WsT {
    double* p;
    int64_t T;
    __device__ __forceinline__ double& operator[](int64_t e) const {
        if (W == 1) return p[e * T];
        return p[(int)e];
    }
};
using Ws = WsT<1>;

/// The Riccati sweep arrays (value matrices, pivots and their reciprocal
/// seeds, gains, G, value gradients, feedforward steps) are private to
/// rfactor_t / rsolve_t. K3w keeps them in the block's shared memory (one warp
/// per block): 32-bit LDS/STS addressing and LDS latency on the serial
/// recursions. K3g keeps them in its global slab.
extern __shared__ __align__(16) double gen_smem[];
/// JX / JU: K3w's shared-memory copies of the current QP's constraint
/// jacobians (FX[s], FU[s], constant during one solve_qp), staged once per QP
/// so the serial sweeps read them with LDS latency instead of L1/L2 misses
/// on the dependency chain (r02j profile: 14 % of K3w's stall samples).
/// RS / RD / RH: the IPM residuals the vector sweep reads (K3w keeps them in
/// shared memory; K3g in its slab at Layout's offsets). TG: the products of
/// the complementarity gap's ordered sums, formed lane-parallel. LB / UB /
/// RR / QQ: the QP's input bounds and the R and Q parts of the Hessian
/// blocks, staged once per QP (constant during solve_qp) for the lane loops
/// and the factor sweep. At N = 60, NX = 3 the layout is 26.4 KB, so 8
/// one-warp blocks (the register limit) still fit an SM.
// NMPCMC_K3W_NOQQ = 1 (default): the Hessian blocks Q, R are not staged in
// shared memory; the lane-split factor sweep reads them from the slab one
// stage ahead. Frees 4.8 KB per warp at N = 60, NX = 3, which the SM gives to
// L1 (measured +5 %, profiles/r02/r02J_k3w_noqq_ab.txt).
#ifndef NMPCMC_K3W_NOQQ
#define NMPCMC_K3W_NOQQ 1
#endif
// NMPCMC_K3W_NOJX = 1: likewise for the constraint jacobians Jx, Ju (6.7 KB);
// measured 5 % slower (r02K_k3w_nojx_ab.txt), so they stay staged.
#ifndef NMPCMC_K3W_NOJX
#define NMPCMC_K3W_NOJX 0
#endif
#ifndef NMPCMC_K3W_MIN_BLOCKS
#define NMPCMC_K3W_MIN_BLOCKS 1
#endif
template <int NX>
struct SweepLay {
    int FP, FLL, FLY, FK, FG, PV, DFF, JX, JU, RS, RD, RH, TG, LB, UB, RR, QQ, total;
    __host__ __device__ explicit SweepLay(int N) {
        FP = 0;
        FLL = FP + (N + 1) * NX * NX;
        FLY = FLL + N;
        FK = FLY + N;
        FG = FK + N * NX;
        PV = FG + N * NX;
        DFF = PV + (N + 1) * NX;
        JX = DFF + N;
        JU = JX + (NMPCMC_K3W_NOJX ? 0 : N * NX * NX);
        RS = JU + (NMPCMC_K3W_NOJX ? 0 : N * NX);
        RD = RS + N * (1 + NX);
        RH = RD + N * NX;
        TG = RH + N;
        LB = TG + 2 * N;
        UB = LB + N;
        RR = UB + N;
        QQ = RR + (NMPCMC_K3W_NOQQ ? 0 : N + 1);
        total = QQ + (NMPCMC_K3W_NOQQ ? 0 : (N + 1) * NX * NX);
    }
};
/// Bytes of shared memory K3w needs per block; K3w runs only if it fits.
template <int NX>
__host__ __device__ inline size_t sweep_smem_bytes(int N) {
    return (size_t)SweepLay<NX>(N).total * sizeof(double);
}
constexpr size_t kSweepSmemMax = 200u << 10;
/// Pointer view of one sweep array (pre-offset; K3g strided by T).
template <int W>
struct ArrT {
    double* p;
    int64_t T;
    __device__ __forceinline__ double& operator[](int i) const {
        if (W == 1) return p[(int64_t)i * T];
        return p[i];
    }
};
template <int W>
__device__ __forceinline__ ArrT<W> sweep_arr(const WsT<W>& w, int goff, int soff) {
    if (W == 1) return ArrT<W>{w.p + (int64_t)goff * w.T, w.T};
    return ArrT<W>{gen_smem + soff, 1};
}

/// The constraint jacobians for the sweeps: the staged copy, or the slab.
template <int W>
__device__ __forceinline__ ArrT<W> jac_arr(const WsT<W>& w, int goff, int soff) {
    if (W > 1 && NMPCMC_K3W_NOJX) return ArrT<W>{w.p + goff, 1};
    return sweep_arr<W>(w, goff, soff);
}

/// Ordered sum s = init + t(0) + t(1) + ... + t(n-1), left to right, the
/// reference's serial reduction order. K3w forms the terms lane-parallel into
/// the shared-memory scratch (n <= cap doubles) and then adds them serially on
/// every lane, so the serial chain reads LDS instead of slab loads; K3g (or a
/// missing scratch) adds them directly. Bitwise the same either way: every
/// term is the same IEEE expression and the additions happen in index order.
template <int W, class T>
__device__ __forceinline__ double ordered_sum(double init, int n, double* scratch, int cap, const T& term) {
    double acc = init;
    if (W > 1 && scratch != nullptr && n <= cap) {
        for (int e = (int)(threadIdx.x & 31); e < n; e += W) scratch[e] = term(e);
        __syncwarp();
#pragma unroll 4
        for (int e = 0; e < n; ++e) acc += scratch[e];
        __syncwarp();
    } else {
        for (int e = 0; e < n; ++e) acc += term(e);
    }
    return acc;
}

/// Lane helpers: W = 1 (thread per sample) or 32 (warp per sample).
constexpr unsigned kMask = 0xffffffffu;
template <int W>
struct Lanes {
    __device__ static int lane() { return W == 1 ? 0 : (int)(threadIdx.x & 31); }
    __device__ static void sync() {
        if (W > 1) __syncwarp();
    }
    __device__ static bool any(bool p) { return W == 1 ? p : __any_sync(kMask, p); }
    __device__ static int sum(int v) { return W == 1 ? v : __reduce_add_sync(kMask, v); }
    __device__ static int imin(int v) { return W == 1 ? v : __reduce_min_sync(kMask, v); }
    __device__ static int bcast(int v, int src) { return W == 1 ? v : __shfl_sync(kMask, v, src); }
    /// std::max fold of per-lane partials (NaN-free, no -0).
    __device__ static double max_fold(double m) {
        if (W > 1)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double v = __shfl_xor_sync(kMask, m, o);
                m = (m < v) ? v : m;
            }
        return m;
    }
    /// std::min fold of per-lane partials (NaN-free, no -0).
    __device__ static double min_fold(double m) {
        if (W > 1)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double v = __shfl_xor_sync(kMask, m, o);
                m = (v < m) ? v : m;
            }
        return m;
    }
};

/// Element offsets of the per-sample arrays for horizon N (NX compile time).
/// Two evaluation sets (iterate / trial) are swapped by index, not copied.
template <int NX>
struct Layout {
    static constexpr int W = 1 + NX;  // stride of xi (n_u + n_x)
    static constexpr int B = (NX + 1) * (NX + 1);
    int N, L, NN;
    int XI[2], GF[2], G[2], FX[2], FU[2], BB[2];
    int LAM, PL, PU, QDXI, QMU, QNL, QNU, SL, SU, RS, RD, RL, RU, CL, CU, DSL, DSU, DNL, DNU, BAR, DXI,
        DMU, RH, FP, FLL, FLY, FK, FG, PV, DFF, WB, SIG, HO, HN, LXI, LLAM, LPL, LPU, SP, US, total;
    __host__ __device__ explicit Layout(int n) : N(n), L(n * W), NN(n * NX) {
        int o = 0;
        auto take = [&](int len) {
            const int at = o;
            o += len;
            return at;
        };
        for (int s = 0; s < 2; ++s) {
            XI[s] = take(L);
            GF[s] = take(L);
            G[s] = take(NN);
            FX[s] = take(NN * NX);
            FU[s] = take(NN);
            BB[s] = take(NN);
        }
        LAM = take(NN), PL = take(N), PU = take(N);
        QDXI = take(L), QMU = take(NN), QNL = take(N), QNU = take(N);
        SL = take(N), SU = take(N), RS = take(L), RD = take(NN), RL = take(N), RU = take(N);
        CL = take(N), CU = take(N), DSL = take(N), DSU = take(N), DNL = take(N), DNU = take(N);
        BAR = take(N), DXI = take(L), DMU = take(NN), RH = take(N);
        FP = take((N + 1) * NX * NX), FLL = take(N), FLY = take(N), FK = take(NN), FG = take(NN);
        PV = take((N + 1) * NX), DFF = take(N);
        WB = take((N + 1) * B);
        SIG = take(NN), HO = take(L), HN = take(L);
        LXI = take(L), LLAM = take(NN), LPL = take(N), LPU = take(N);
        SP = take(N), US = take(N);
        total = o;
    }
    __host__ __device__ int uo(int k) const { return k * W; }            // u slot of stage k
    __host__ __device__ int xo(int k) const { return (k - 1) * W + 1; }  // x_k, k >= 1
};

/// Work counters (K3's units: stage intervals shot, IPM stage-iterations,
/// completed SQP steps, ...), for the roofline.
struct Cnt {
    int64_t steps, shoot_full, shoot_fonly, ipm_stage, sqp_stage, qp, sqp, ls;
};

// ------------------------------------------------------------------ model
/// One CSTR variant (cstr.cpp:21-34 stoichiometry, cstr.hpp:21-34 params).
template <int NX>
struct Model {
    Cstr p;
    double S[NX], Cin[NX], sb[NX];
    /// 1: the model carries no analytic jacobians, so drift_jacobian_x /
    /// _u, measurement_jacobian_x and output_jacobian_x take the reference's
    /// central finite differences (model.cpp:54-124); NMPCMC_OPT_CTRL_JACOBIANS.
    int fd = 0;
};
template <int NX>
__device__ Model<NX> make_model(const nmpcmc_cstr_params& q) {
    Model<NX> m;
    m.p = load_cstr(q);
    if (NX == 3) {
        m.S[0] = -1.0, m.S[1] = -2.0, m.S[NX - 1] = q.beta;
        m.Cin[0] = q.cA_in, m.Cin[1] = q.cB_in, m.Cin[NX - 1] = q.cT_in;
        m.sb[0] = q.sigmaA, m.sb[1] = q.sigmaB, m.sb[NX - 1] = q.sigmaT;
    } else {
        m.S[0] = q.beta;
        m.Cin[0] = q.cT_in;
        m.sb[0] = q.sigmaT;
    }
    return m;
}

/// fd_step (model.cpp:9): max(1e-6, 1e-6 |v|) with std::max semantics.
__device__ __forceinline__ double fd_step(double v) { return smax(1e-6, 1e-6 * fabs(v)); }

template <int NX>
__device__ __forceinline__ int drift_jac(const Model<NX>& m, const double* x, double u, double* d, double* J);

/// drift_jacobian_x by central differences (model.cpp:54-71): column j from
/// drift at x +- h e_j, h = fd_step(x_j), (f+ - f-) / (2 h). A DomainError of
/// either evaluation escapes, as in the reference.
template <int NX>
__device__ __noinline__ int fd_jac_x(const Model<NX>& m, const double* x, double u, double* J) {
    double xp[NX], xm[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) xp[i] = x[i], xm[i] = x[i];
#pragma unroll 1
    for (int j = 0; j < NX; ++j) {
        const double h = fd_step(x[j]);
        xp[j] = x[j] + h;
        xm[j] = x[j] - h;
        double fp[NX], fm[NX];
        int st = drift_jac<NX>(m, xp, u, fp, nullptr);
        if (st) return st;
        st = drift_jac<NX>(m, xm, u, fm, nullptr);
        if (st) return st;
#pragma unroll
        for (int i = 0; i < NX; ++i) J[j * NX + i] = (fp[i] - fm[i]) / (2.0 * h);
        xp[j] = x[j];
        xm[j] = x[j];
    }
    return G_OK;
}

/// drift_jacobian_u by central differences (model.cpp:73-89), n_u = 1.
template <int NX>
__device__ __noinline__ int fd_jac_u(const Model<NX>& m, const double* x, double u, double* B) {
    const double h = fd_step(u);
    double fp[NX], fm[NX];
    int st = drift_jac<NX>(m, x, u + h, fp, nullptr);
    if (st) return st;
    st = drift_jac<NX>(m, x, u - h, fm, nullptr);
    if (st) return st;
#pragma unroll
    for (int i = 0; i < NX; ++i) B[i] = (fp[i] - fm[i]) / (2.0 * h);
    return G_OK;
}

/// d g / d x_{NX-1} of g(x) = x_{NX-1} / V (measurement = output,
/// cstr.cpp:86-95): 1/V analytically, or the central difference of
/// state_fn_jacobian (model.cpp:93-113); the other entries are +0 either way
/// ((g(x) - g(x)) / (2 h) = +0).
template <int NX>
__device__ __forceinline__ double meas_jac_T(const Model<NX>& m, double xT) {
    if (!m.fd) return 1.0 / m.p.V;
    const double h = fd_step(xT);
    const double gp = (xT + h) / m.p.V, gm = (xT - h) / m.p.V;
    return (gp - gm) / (2.0 * h);
}

/// drift (cstr.cpp:42-53) and, when J != nullptr, drift_jacobian_x
/// (cstr.cpp:99-119); both evaluate exp(-EaR/cT) of the same argument, so it
/// is computed once. Returns G_DOMAIN when c_T <= 0 (cstr.cpp:38).
template <int NX>
__device__ __forceinline__ int drift_jac(const Model<NX>& m, const double* x, double u, double* d, double* J) {
    const double f = u * kMlMinToLs;
    double c[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) c[i] = x[i] / m.p.V;
    double cA, cB, cT;
    if (NX == 3) {
        cA = c[0], cB = c[1], cT = c[NX - 1];
    } else {
        cT = c[0];
        cA = m.p.cA_in - (cT - m.p.cT_in) / m.p.beta;
        cB = m.p.cB_in - 2.0 * (cT - m.p.cT_in) / m.p.beta;
    }
    if (cT <= 0.0) return G_DOMAIN;
    const double k = m.p.k0 * xlibm_exp(-m.p.EaR / cT);
    const double r = k * cA * cB;
#pragma unroll
    for (int i = 0; i < NX; ++i) d[i] = m.Cin[i] * f - c[i] * f + m.S[i] * r * m.p.V;
    if (J != nullptr && m.fd) return fd_jac_x<NX>(m, x, u, J);
    if (J != nullptr) {
        if (NX == 3) {
            const double g[3] = {k * cB, k * cA, k * (m.p.EaR / (cT * cT)) * cA * cB};
            const double dg = -f / m.p.V;
#pragma unroll
            for (int j = 0; j < NX; ++j)
#pragma unroll
                for (int i = 0; i < NX; ++i) J[j * NX + i] = (i == j ? dg : 0.0) + m.S[i] * g[j];
        } else {
            const double g = k * (m.p.EaR / (cT * cT)) * cA * cB + k * (-cB / m.p.beta - 2.0 * cA / m.p.beta);
            J[0] = -f / m.p.V + m.p.beta * g;
        }
    }
    return G_OK;
}
/// drift_jacobian_u (cstr.cpp:120-127), or its central difference.
template <int NX>
__device__ __forceinline__ int jac_u(const Model<NX>& m, const double* x, double u, double* B) {
    if (m.fd) return fd_jac_u<NX>(m, x, u, B);
#pragma unroll
    for (int i = 0; i < NX; ++i) B[i] = (m.Cin[i] - x[i] / m.p.V) * kMlMinToLs;
    return G_OK;
}

// ------------------------------------------------------------------ shoot
#ifndef NMPCMC_SHOOT_MODEL_COPY
#define NMPCMC_SHOOT_MODEL_COPY 1  // measured +3.5 % three-state (profiles/r02/r02s_k3w_model_ab.txt)
#endif
/// shoot (ocp.cpp:9-74): Nc RK4 steps of (F, Fx, Fu). Column-major Fx.
/// The RK4 weighted sum a + 2b + 2c + d accumulates left to right.
template <int NX, bool SENS>
__device__ __noinline__ int shoot(const Model<NX>& m_in, const double* x, double u, double h, int nc,
                                  double* F_out, double* Fx_out, double* Fu_out) {
#if NMPCMC_SHOOT_MODEL_COPY
    // a private copy: the stores to F / Fx / Fu may alias the caller's model
    // (both live in local memory), which would force a reload of every model
    // field after each store inside the RK4 loop
    const Model<NX> m = m_in;
#else
    const Model<NX>& m = m_in;
#endif
    // the running (F, Fx, Fu) live in registers; the caller's arrays (local
    // memory) are written once on the way out, with the values the reference's
    // in-place update would hold at that point
    double F[NX], Fx[NX * NX], Fu[NX];
    auto put = [&](int st) {
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            F_out[i] = F[i];
            if (SENS) {
                Fu_out[i] = Fu[i];
#pragma unroll
                for (int l = 0; l < NX; ++l) Fx_out[l * NX + i] = Fx[l * NX + i];
            }
        }
        return st;
    };
#pragma unroll
    for (int i = 0; i < NX; ++i) {
        F[i] = x[i];
        if (SENS) {
            Fu[i] = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) Fx[j * NX + i] = (i == j) ? 1.0 : 0.0;
        }
    }
#pragma unroll 1
    for (int step = 0; step < nc; ++step) {
        double pk[NX], pkx[NX * NX], pku[NX], ak[NX], akx[NX * NX], aku[NX];
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
            double xs[NX], sx[NX * NX], su[NX];
            const double c = (j == 3) ? 1.0 : 0.5;
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                xs[i] = j == 0 ? F[i] : F[i] + c * h * pk[i];
                if (SENS) {
                    su[i] = j == 0 ? Fu[i] : Fu[i] + c * h * pku[i];
#pragma unroll
                    for (int l = 0; l < NX; ++l)
                        sx[l * NX + i] = j == 0 ? Fx[l * NX + i] : Fx[l * NX + i] + c * h * pkx[l * NX + i];
                }
            }
            double k[NX], A[NX * NX], B[NX];
            const int st = drift_jac<NX>(m, xs, u, k, SENS ? A : nullptr);
            if (st) return put(st);
            double kx[NX * NX], ku[NX];
            if (SENS) {
                const int su_st = jac_u<NX>(m, xs, u, B);
                if (su_st) return put(su_st);
#pragma unroll
                for (int jj = 0; jj < NX; ++jj)  // kx = A sx (gemm, beta 0)
#pragma unroll
                    for (int i = 0; i < NX; ++i) {
                        double s = 0.0;
#pragma unroll
                        for (int l = 0; l < NX; ++l) s += A[l * NX + i] * sx[jj * NX + l];
                        kx[jj * NX + i] = 1.0 * s + 0.0;
                    }
#pragma unroll
                for (int i = 0; i < NX; ++i) {  // ku = B; gemm(1, A, su, 1, ku)
                    double s = 0.0;
#pragma unroll
                    for (int l = 0; l < NX; ++l) s += A[l * NX + i] * su[l];
                    ku[i] = 1.0 * s + 1.0 * B[i];
                }
            }
            const double w = (j == 1 || j == 2) ? 2.0 : 1.0;
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                ak[i] = j == 0 ? k[i] : (j < 3 ? ak[i] + w * k[i] : ak[i] + k[i]);
                pk[i] = k[i];
                if (SENS) {
                    aku[i] = j == 0 ? ku[i] : (j < 3 ? aku[i] + w * ku[i] : aku[i] + ku[i]);
                    pku[i] = ku[i];
#pragma unroll
                    for (int l = 0; l < NX; ++l) {
                        const int e = l * NX + i;
                        akx[e] = j == 0 ? kx[e] : (j < 3 ? akx[e] + w * kx[e] : akx[e] + kx[e]);
                        pkx[e] = kx[e];
                    }
                }
            }
        }
        const double h6 = h / 6.0;
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            F[i] += h6 * ak[i];
            if (SENS) {
                Fu[i] += h6 * aku[i];
#pragma unroll
                for (int l = 0; l < NX; ++l) Fx[l * NX + i] += h6 * akx[l * NX + i];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NX; ++i)
        if (!dfinite(F[i])) return put(G_NONFINITE);
    return put(G_OK);
}

// -------------------------------------------------------------------- OCP
template <int NX, int W>
struct Ocp {
    Model<NX> m;
    Layout<NX> lay;
    WsT<W> ws;
    int N, Nc;
    double Ts, h, umin, umax, Qz, invV;
    double x0[NX];
    Cnt* cnt;
    /// Problem kind of the SqpProblem interface (sqp.hpp:15-25) sqp_solve runs
    /// on: nullptr = the CSTR regulator OcpProblem (sqp.hpp:28-48); else the
    /// packed data of one stagewise quadratic NLP (QNLP below). A new kind is
    /// added by giving objective() and constraints() one more branch.
    const double* prob = nullptr;
    /// SqpReport::trace (sqp.hpp:64-90) of the next sqp_solve: up to
    /// trace_cap SqpIterationLog records (null: no trace), count in *trace_len.
    nmpcmc_sqp_iter_log* trace = nullptr;
    int trace_cap = 0;
    int32_t* trace_len = nullptr;
};

// --------------------------------------------- quadratic stagewise NLP kind
/// Stagewise quadratic NLP with affine dynamics (the problems the reference's
/// SQP tests pose through SqpProblem): decision xi = (u_0, x_1, ..., u_{N-1},
/// x_N), n_u = 1, x_0 given,
///   f(xi) = sum_k [ 1/2 R_k u_k^2 + r_k u_k + 1/2 x_{k+1}' Q_k x_{k+1} + q_k' x_{k+1} ]
///   F_k(x_k, u_k) = A_k x_k + B_k u_k + c_k,  g_k = x_{k+1} - F_k,
/// u_min <= u_k <= u_max. Per stage k the packed data hold
/// R r Q[NX*NX] q[NX] A[NX*NX] B[NX] c[NX] (matrices column-major); the
/// evaluation order below is the one of oracle/ref_driver.cpp's QnlpProblem
/// (the host SqpProblem the parity tests hand to the reference's sqp_solve).
template <int NX>
struct Qnlp {
    static constexpr int kStage = 2 + 2 * NX * NX + 3 * NX;
    __host__ __device__ static constexpr int R() { return 0; }
    __host__ __device__ static constexpr int r() { return 1; }
    __host__ __device__ static constexpr int Q() { return 2; }
    __host__ __device__ static constexpr int q() { return 2 + NX * NX; }
    __host__ __device__ static constexpr int A() { return 2 + NX * NX + NX; }
    __host__ __device__ static constexpr int B() { return 2 + 2 * NX * NX + NX; }
    __host__ __device__ static constexpr int c() { return 2 + 2 * NX * NX + 2 * NX; }
};

/// objective() of the quadratic kind: phi in stage order (serial on every
/// lane), gradient R u + r / Q x + q lane-parallel.
template <int NX, int W>
__device__ __noinline__ double qnlp_objective(const Ocp<NX, W>& o, int s, bool grad) {
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    using D = Qnlp<NX>;
    double phi = 0.0;
#pragma unroll 1
    for (int k = 0; k < o.N; ++k) {
        const double* P = o.prob + (int64_t)k * D::kStage;
        const double u = w[L.XI[s] + L.uo(k)];
        const double su = __ldg(P + D::R()) * u;
        phi = phi + (0.5 * (u * su) + __ldg(P + D::r()) * u);
        double xQx = 0.0, qx = 0.0;
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            double qxi = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) qxi += __ldg(P + D::Q() + j * NX + i) * w[L.XI[s] + L.xo(k + 1) + j];
            const double xi_ = w[L.XI[s] + L.xo(k + 1) + i];
            xQx += xi_ * qxi;
            qx += __ldg(P + D::q() + i) * xi_;
        }
        phi = phi + (0.5 * xQx + qx);
    }
    if (grad) {
#pragma unroll 1
        for (int k = Lanes<W>::lane(); k < o.N; k += W) {
            const double* P = o.prob + (int64_t)k * D::kStage;
            const double u = w[L.XI[s] + L.uo(k)];
            w[L.GF[s] + L.uo(k)] = __ldg(P + D::R()) * u + __ldg(P + D::r());
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                double qxi = 0.0;
#pragma unroll
                for (int j = 0; j < NX; ++j) qxi += __ldg(P + D::Q() + j * NX + i) * w[L.XI[s] + L.xo(k + 1) + j];
                w[L.GF[s] + L.xo(k + 1) + i] = qxi + __ldg(P + D::q() + i);
            }
        }
    }
    Lanes<W>::sync();
    return phi;
}

/// constraints() of the quadratic kind: F_k = (A_k x_k + B_k u_k) + c_k per
/// stage, lane-parallel; never fails.
template <int NX, int W>
__device__ __noinline__ int qnlp_constraints(const Ocp<NX, W>& o, int s) {
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    using D = Qnlp<NX>;
#pragma unroll 1
    for (int k = Lanes<W>::lane(); k < o.N; k += W) {
        const double* P = o.prob + (int64_t)k * D::kStage;
        double xk[NX];
#pragma unroll
        for (int i = 0; i < NX; ++i) xk[i] = k == 0 ? o.x0[i] : w[L.XI[s] + L.xo(k) + i];
        const double u = w[L.XI[s] + L.uo(k)];
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            double F = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) F += __ldg(P + D::A() + j * NX + i) * xk[j];
            F = F + __ldg(P + D::B() + i) * u;
            F = F + __ldg(P + D::c() + i);
            const double nx = w[L.XI[s] + L.xo(k + 1) + i];
            w[L.BB[s] + k * NX + i] = F - nx;
            w[L.G[s] + k * NX + i] = nx - F;
            w[L.FU[s] + k * NX + i] = __ldg(P + D::B() + i);
#pragma unroll
            for (int j = 0; j < NX; ++j) w[L.FX[s] + (k * NX + j) * NX + i] = __ldg(P + D::A() + j * NX + i);
        }
    }
    Lanes<W>::sync();
    return G_OK;
}

/// eval_objective (ocp.cpp:76-99) of xi set s; gradient into GF[s] if grad.
template <int NX, int W>
__device__ __noinline__ double objective(const Ocp<NX, W>& o, int s, bool grad) {
    if (o.prob != nullptr) return qnlp_objective<NX, W>(o, s, grad);
    // serial on every lane (phi is an ordered sum); the gradient is stored,
    // not accumulated: each slot is 0.0 + 2 Ts g once (ocp.cpp:80-97)
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    // scalars hoisted: the stores below may alias the Ocp (local memory)
    const double V = o.m.p.V, Qz = o.Qz, Ts = o.Ts, invV = o.invV;
    const int N = o.N;
    double phi = 0.0;
#pragma unroll 1
    for (int k = 1; k <= N; ++k) {
        const double res = w[L.XI[s] + L.xo(k) + NX - 1] / V - w[L.SP + k - 1];
        const double qres = 1.0 * (0.0 + Qz * res) + 0.0;
        phi += Ts * (0.0 + res * qres);
        if (grad) {
            w[L.GF[s] + L.uo(k - 1)] = 0.0;
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                const double hi = (i == NX - 1) ? (o.m.fd ? meas_jac_T<NX>(o.m, w[L.XI[s] + L.xo(k) + NX - 1])
                                                          : invV)
                                                : 0.0;
                const double g = 1.0 * (0.0 + hi * qres) + 0.0;
                w[L.GF[s] + L.xo(k) + i] = 0.0 + 2.0 * Ts * g;
            }
        }
    }
    Lanes<W>::sync();
    return phi;
}

/// eval_constraints (ocp.cpp:101-135) of xi set s into G/FX/FU/BB[s].
template <int NX, int W>
__device__ __noinline__ int constraints(const Ocp<NX, W>& o, int s) {
    if (o.prob != nullptr) return qnlp_constraints<NX, W>(o, s);
    // stages are independent (multiple shooting): lane-parallel; the status
    // is the one of the lowest failing stage, as the sequential loop returns
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    int bad_k = 0x7fffffff, bad_st = G_OK, shot = 0;
#pragma unroll 1
    for (int k = Lanes<W>::lane(); k < o.N; k += W) {
        double xk[NX];
#pragma unroll
        for (int i = 0; i < NX; ++i) xk[i] = k == 0 ? o.x0[i] : w[L.XI[s] + L.xo(k) + i];
        double F[NX], Fx[NX * NX], Fu[NX];
        const int st = shoot<NX, true>(o.m, xk, w[L.XI[s] + L.uo(k)], o.h, o.Nc, F, Fx, Fu);
        ++shot;  // one stage interval (workmodel.SHOOT_FULL)
        if (st) {
            bad_k = k;
            bad_st = st;
            break;
        }
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            const double nx = w[L.XI[s] + L.xo(k + 1) + i];
            w[L.BB[s] + k * NX + i] = F[i] - nx;
            w[L.G[s] + k * NX + i] = nx - F[i];
            w[L.FU[s] + k * NX + i] = Fu[i];
#pragma unroll
            for (int j = 0; j < NX; ++j) w[L.FX[s] + (k * NX + j) * NX + i] = Fx[j * NX + i];
        }
    }
    o.cnt->shoot_full += Lanes<W>::sum(shot);
    const int kmin = Lanes<W>::imin(bad_k);
    Lanes<W>::sync();
    if (kmin == 0x7fffffff) return G_OK;
    return Lanes<W>::bcast(bad_st, kmin % W);
}

/// xi_from_inputs (ocp.cpp:137-154): u from US, result into XI[s].
template <int NX, int W>
__device__ __noinline__ int xi_from_u(const Ocp<NX, W>& o, int s) {
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    double xk[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) xk[i] = o.x0[i];
#pragma unroll 1
    for (int k = 0; k < o.N; ++k) {
        const double u = w[L.US + k];
        w[L.XI[s] + L.uo(k)] = u;
        double F[NX];
        const int st = shoot<NX, false>(o.m, xk, u, o.h, o.Nc, F, nullptr, nullptr);
        o.cnt->shoot_fonly += 1;
        if (st) {
            Lanes<W>::sync();
            return st;
        }
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            w[L.XI[s] + L.xo(k + 1) + i] = F[i];
            xk[i] = F[i];
        }
    }
    Lanes<W>::sync();
    return G_OK;
}

// --------------------------------------------------------------------- QP
// Stage data (build_stages, sqp.cpp:130-171) is read in place: R_0 = W_0;
// for k >= 1, Q = W_k[0:nx,0:nx], M = W_k[0:nx,nx], R = W_k[nx,nx],
// q = gf(x_k); r = gf(u_k); Jx/Ju/b = the constraint blocks of set s;
// terminal Q = W_N, q = gf(x_N); lb/ub = umin/umax - u_k.
template <int NX, int W>
struct QpView {
    const Ocp<NX, W>* o;
    int s;  // evaluation set of the current iterate
    // cached by value, so the accessors need no reload through *o after stores
    WsT<W> w;
    int N, WB, GFs, FXs, FUs, BBs, XIs, sLB, sUB;
    double umin, umax;
    __device__ QpView(const Ocp<NX, W>* op, int set)
        : o(op), s(set), w(op->ws), N(op->N), WB(op->lay.WB), GFs(op->lay.GF[set]), FXs(op->lay.FX[set]),
          FUs(op->lay.FU[set]), BBs(op->lay.BB[set]), XIs(op->lay.XI[set]), sLB(SweepLay<NX>(op->N).LB),
          sUB(SweepLay<NX>(op->N).UB), umin(op->umin), umax(op->umax) {}
    __device__ double Wb(int k, int i, int j) const {
        const int ld = k == 0 ? 1 : (k < N ? NX + 1 : NX);
        return w[WB + k * Layout<NX>::B + j * ld + i];
    }
    __device__ double R(int k) const { return k == 0 ? Wb(0, 0, 0) : Wb(k, NX, NX); }
    __device__ double Q(int k, int i, int j) const { return Wb(k, i, j); }
    __device__ double M(int k, int i) const { return Wb(k, i, NX); }
    __device__ double q(int k, int i) const { return w[GFs + Layout<NX>::W * (k - 1) + 1 + i]; }
    __device__ double r(int k) const { return w[GFs + Layout<NX>::W * k]; }
    __device__ double Jx(int k, int i, int j) const { return w[FXs + (k * NX + j) * NX + i]; }
    __device__ double Ju(int k, int i) const { return w[FUs + k * NX + i]; }
    __device__ double b(int k, int i) const { return w[BBs + k * NX + i]; }
    __device__ double u(int k) const { return w[XIs + Layout<NX>::W * k]; }
    // K3w reads the copies solve_qp staged (SweepLay LB / UB)
    __device__ double lb(int k) const { return W > 1 ? gen_smem[sLB + k] : umin - u(k); }
    __device__ double ub(int k) const { return W > 1 ? gen_smem[sUB + k] : umax - u(k); }
    __device__ double lb_src(int k) const { return umin - u(k); }
    __device__ double ub_src(int k) const { return umax - u(k); }
};

/// riccati_factor (qp.cpp:73-110) with barrier diagonal BAR. Returns true on
/// NotPositiveDefinite.
template <int NX, int W, bool FAST>
__device__ __noinline__ bool rfactor_t(const QpView<NX, W> v, bool* cert) {
    const Ocp<NX, W>& o = *v.o;
    const WsT<W> w = o.ws;  // by value: base/stride and the offsets below live in registers
    const Layout<NX> L = o.lay;
    const int oBAR = L.BAR, oFG = L.FG, oFK = L.FK, oFLL = L.FLL, oFLY = L.FLY, oFP = L.FP;
    const SweepLay<NX> SL(o.N);
    const ArrT<W> aFP = sweep_arr<W>(w, oFP, SL.FP);
    const ArrT<W> aFLL = sweep_arr<W>(w, oFLL, SL.FLL);
    const ArrT<W> aFLY = sweep_arr<W>(w, oFLY, SL.FLY);
    const ArrT<W> aFK = sweep_arr<W>(w, oFK, SL.FK);
    const ArrT<W> aFG = sweep_arr<W>(w, oFG, SL.FG);
    const int oFXs = L.FX[v.s], oFUs = L.FU[v.s], oWB = L.WB, oXIs = L.XI[v.s], oGFs = L.GF[v.s];
    // K3w: the shared-memory copies staged by solve_qp; K3g: the set in place
    const ArrT<W> aJX = jac_arr<W>(w, oFXs, SL.JX);
    const ArrT<W> aJU = jac_arr<W>(w, oFUs, SL.JU);
    auto Jx_ = [&](int k, int i, int j) -> double { return aJX[(k * NX + j) * NX + i]; };
    auto Ju_ = [&](int k, int i) -> double { return aJU[k * NX + i]; };
    const int nN = o.N;
    auto Wb_ = [&](int k, int i, int j) -> double {
        const int ld = k == 0 ? 1 : (k < nN ? NX + 1 : NX);
        return w[oWB + k * Layout<NX>::B + j * ld + i];
    };
    // K3w: R and Q from the copies solve_qp staged (SweepLay RR / QQ)
    auto R_ = [&](int k) -> double {
        if (W > 1 && !NMPCMC_K3W_NOQQ) return gen_smem[SL.RR + k];
        return k == 0 ? Wb_(0, 0, 0) : Wb_(k, NX, NX);
    };
    auto Q_ = [&](int k, int i, int j) -> double {
        if (W > 1 && !NMPCMC_K3W_NOQQ) return gen_smem[SL.QQ + (k * NX + j) * NX + i];
        return Wb_(k, i, j);
    };
    auto M_ = [&](int k, int i) -> double { return Wb_(k, i, NX); };
    (void)oXIs, (void)oGFs;

    const int N = o.N;
    auto P = [&](int k, int i, int j) -> double& { return aFP[(k * NX + j) * NX + i]; };
    // P_{k+1} is carried in registers from one stage to the next: reloading
    // what the previous stage just stored would put a store-to-load round trip
    // through the cache hierarchy on the recursion's critical path
    double Pn[NX * NX];
#pragma unroll
    for (int j = 0; j < NX; ++j)
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            Pn[j * NX + i] = Q_(N, i, j);
            P(N, i, j) = Pn[j * NX + i];
        }
#pragma unroll 1
    for (int k = N - 1; k >= 0; --k) {
        double ju[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) ju[j] = Ju_(k, j);
        double PJu[NX];
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < NX; ++l) s += Pn[l * NX + i] * ju[l];
            PJu[i] = 1.0 * s + 0.0;
        }
        double H;
        {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < NX; ++l) s += ju[l] * PJu[l];
            H = 1.0 * s + 0.0;
        }
        H += R_(k);
        H += w[oBAR + k];
        if (H <= 0.0 || !dfinite(H)) return true;  // cholesky_factor (linalg.cpp:69-103)
        double l, y;
        if (FAST) {
            fast_sqrt(H, l, y);
            *cert &= cert_sqrt_bf(H, l);
        } else {
            l = sqrt(H);
            y = 1.0 / l;  // seed of rsolve's certified division
        }
        aFLL[k] = l;
        aFLY[k] = y;
        if (k >= 1) {
            double PJx[NX * NX], G[NX], K[NX];
#pragma unroll
            for (int j = 0; j < NX; ++j)
#pragma unroll
                for (int i = 0; i < NX; ++i) {
                    double s = 0.0;
#pragma unroll
                    for (int m = 0; m < NX; ++m) s += Pn[m * NX + i] * Jx_(k, m, j);
                    PJx[j * NX + i] = 1.0 * s + 0.0;
                }
#pragma unroll
            for (int j = 0; j < NX; ++j) {
                double s = 0.0;
#pragma unroll
                for (int m = 0; m < NX; ++m) s += ju[m] * PJx[j * NX + m];
                G[j] = 1.0 * s + 0.0;
            }
#pragma unroll
            for (int j = 0; j < NX; ++j) G[j] += M_(k, j);
#pragma unroll
            for (int j = 0; j < NX; ++j) {  // cholesky_solve of the 1x1 factor, then negate
                double t;
                if (FAST) {
                    t = cdiv_seed(G[j], l, y, *cert);
                    t = cdiv_seed(t, l, y, *cert);
                } else {
                    t = G[j] / l;
                    t = t / l;
                }
                K[j] = -t;
            }
            double Pk[NX * NX];
#pragma unroll
            for (int j = 0; j < NX; ++j)
#pragma unroll
                for (int i = 0; i < NX; ++i) {
                    double s = 0.0;
#pragma unroll
                    for (int m = 0; m < NX; ++m) s += Jx_(k, m, i) * PJx[j * NX + m];
                    Pk[j * NX + i] = 1.0 * s + 0.0;
                }
#pragma unroll
            for (int j = 0; j < NX; ++j)
#pragma unroll
                for (int i = 0; i < NX; ++i) Pk[j * NX + i] += Q_(k, i, j);
#pragma unroll
            for (int j = 0; j < NX; ++j)
#pragma unroll
                for (int i = 0; i < NX; ++i) Pk[j * NX + i] = 1.0 * (0.0 + G[i] * K[j]) + 1.0 * Pk[j * NX + i];
#pragma unroll
            for (int j = 0; j < NX; ++j)  // symmetrize (linalg.cpp:227-235)
#pragma unroll
                for (int i = j + 1; i < NX; ++i) {
                    const double mm = 0.5 * (Pk[j * NX + i] + Pk[i * NX + j]);
                    Pk[j * NX + i] = mm;
                    Pk[i * NX + j] = mm;
                }
#pragma unroll
            for (int j = 0; j < NX; ++j) {
                aFK[k * NX + j] = K[j];
                aFG[k * NX + j] = G[j];
#pragma unroll
                for (int i = 0; i < NX; ++i) {
                    P(k, i, j) = Pk[j * NX + i];
                    Pn[j * NX + i] = Pk[j * NX + i];
                }
            }
        }
    }
    return false;
}

// ------------------------------------------------ lane-split sweeps (K3w)
// In the serial sweeps above a warp does the same NX x NX block arithmetic on
// all 32 lanes. The elements of each block product are independent dot
// products, so K3w gives lane (lane % NX^2) ONE element (row i, column j) of
// every NX x NX product and lane (lane % NX) one component of every NX-vector,
// and passes operands between lanes with shuffles. Each element is still the
// same left-to-right sum over the same operands (s = 0.0; s += a*b ...; the
// gemm epilogue), so results are bitwise those of rfactor_t / rsolve_t; the
// warp issues ~3x fewer FP64 instructions per stage.
#ifndef NMPCMC_SPLIT_SWEEPS
#define NMPCMC_SPLIT_SWEEPS 1
#endif

/// a / b from y ~ 1/b as cdiv_seed computes it, without the certificate (the
/// split sweeps stash the operands and certify them lane-parallel afterwards).
__device__ __forceinline__ double div_seed(double a, double b, double y) {
    const double q0 = a * y;
    const double q = __fma_rn(__fma_rn(-b, q0, a), y, q0);
    return a == 0.0 ? q0 : q;
}
/// cdiv_seed's certificate of q = a / b.
__device__ __forceinline__ bool div_seed_ok(double a, double b, double q) {
    return (a == 0.0) | cert_div_bf(a, b, q);
}

/// riccati_factor (qp.cpp:73-110), fast forms, one block element per lane.
/// Returns true on NotPositiveDefinite; *cert is false if any fast
/// sqrt/division was not certified (the caller replays rfactor_t<FAST=false>).
/// The operands of stage k-1 are loaded while stage k computes, so neither
/// shared-memory nor slab (BAR, M) latency sits on the recursion.
template <int NX>
__device__ __noinline__ bool rfactor_split(const QpView<NX, 32> v, bool* cert_out) {
    constexpr int W = 32;
    constexpr unsigned kFull = 0xffffffffu;
    const Ocp<NX, W>& o = *v.o;
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    const int oBAR = L.BAR, oWB = L.WB;
    const SweepLay<NX> SL(o.N);
    double* const aFP = gen_smem + SL.FP;
    double* const aFLL = gen_smem + SL.FLL;
    double* const aFLY = gen_smem + SL.FLY;
    double* const aFK = gen_smem + SL.FK;
    double* const aFG = gen_smem + SL.FG;
    const double* const aJX = NMPCMC_K3W_NOJX ? w.p + L.FX[v.s] : gen_smem + SL.JX;
    const double* const aJU = NMPCMC_K3W_NOJX ? w.p + L.FU[v.s] : gen_smem + SL.JU;
    // this lane's element: row i, column j
    auto i_of = [] { return ((int)(threadIdx.x & 31) % (NX * NX)) % NX; };
    auto j_of = [] { return ((int)(threadIdx.x & 31) % (NX * NX)) / NX; };
    // Q(k, i, j) and R(k): the staged copies, or the W blocks in the slab
    auto Qk = [&](int k) -> double {
        if (!NMPCMC_K3W_NOQQ) return gen_smem[SL.QQ + (k * NX + j_of()) * NX + i_of()];
        const int ld = k < o.N ? NX + 1 : NX;  // k >= 1
        return w[oWB + k * Layout<NX>::B + j_of() * ld + i_of()];
    };
    auto Rk = [&](int k) -> double {
        if (!NMPCMC_K3W_NOQQ) return gen_smem[SL.RR + k];
        return k == 0 ? w[oWB] : w[oWB + k * Layout<NX>::B + NX * (NX + 1) + NX];
    };
    // certificate inputs, checked lane-parallel after the sweep: the pivots'
    // radicands in DFF and the first quotients G / l in RH..TG (3 N doubles,
    // contiguous); all three are dead between qp_resid's sums and qp_csolve
    double* const cH = gen_smem + SL.DFF;
    double* const cQ1 = gen_smem + SL.RH;
    static_assert(NX <= 3, "the RH..TG scratch holds NX <= 3 quotients per stage");
    const int N = o.N;
    const int i = i_of(), j = j_of();
    double Pn = Qk(N);  // P_{k+1}(i, j)
    aFP[(N * NX + j) * NX + i] = Pn;
    // stage operands: Ju, columns j and i of Jx, Q(i, j), R, BAR, M(j)
    struct Ops {
        double ju[NX], jxj[NX], jxi[NX], qq, rr, bar, mj;
    };
    auto load_ops = [&](int k) {
        Ops n;
#pragma unroll
        for (int l = 0; l < NX; ++l) {
            n.ju[l] = aJU[k * NX + l];
            n.jxj[l] = aJX[(k * NX + j) * NX + l];
            n.jxi[l] = aJX[(k * NX + i) * NX + l];
        }
        n.qq = Qk(k > 0 ? k : 1);  // unused at k = 0
        n.rr = Rk(k);
        n.bar = w[oBAR + k];
        n.mj = w[oWB + k * Layout<NX>::B + NX * (NX + 1) + j];  // M(k, j), 1 <= k < N (unused at k = 0)
        return n;
    };
    Ops c = load_ops(N - 1);
#pragma unroll 1
    for (int k = N - 1; k >= 0; --k) {
        const Ops nx = load_ops(k > 0 ? k - 1 : 0);
        double row[NX];
#pragma unroll
        for (int l = 0; l < NX; ++l) row[l] = __shfl_sync(kFull, Pn, i + NX * l);  // P_{k+1}(i, l)
        double pju;  // (P Ju)(i)
        {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < NX; ++l) s += row[l] * c.ju[l];
            pju = 1.0 * s + 0.0;
        }
        double H;
        {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < NX; ++l) s += c.ju[l] * __shfl_sync(kFull, pju, l);  // lane l holds row l
            H = 1.0 * s + 0.0;
        }
        H += c.rr;
        H += c.bar;
        if (H <= 0.0 || !dfinite(H)) {  // cholesky_factor (linalg.cpp:69-103); H is lane-uniform
            __syncwarp();
            return true;
        }
        double l, y;
        fast_sqrt(H, l, y);
        cH[k] = H;
        aFLL[k] = l;
        aFLY[k] = y;
        if (k >= 1) {
            double pjx;  // (P Jx)(i, j)
            {
                double s = 0.0;
#pragma unroll
                for (int m = 0; m < NX; ++m) s += row[m] * c.jxj[m];
                pjx = 1.0 * s + 0.0;
            }
            double col[NX];  // (P Jx)(m, j)
#pragma unroll
            for (int m = 0; m < NX; ++m) col[m] = __shfl_sync(kFull, pjx, m + NX * j);
            double G;  // G(j)
            {
                double s = 0.0;
#pragma unroll
                for (int m = 0; m < NX; ++m) s += c.ju[m] * col[m];
                G = 1.0 * s + 0.0;
            }
            G += c.mj;
            double t = div_seed(G, l, y);  // cholesky_solve of the 1x1 factor, then negate
            cQ1[k * NX + j] = t;
            t = div_seed(t, l, y);
            const double K = -t;
            double pk;  // (Jx' P Jx)(i, j)
            {
                double s = 0.0;
#pragma unroll
                for (int m = 0; m < NX; ++m) s += c.jxi[m] * col[m];
                pk = 1.0 * s + 0.0;
            }
            pk += c.qq;
            const double Gi = __shfl_sync(kFull, G, NX * i);  // lane (0, i) holds G(i)
            pk = 1.0 * (0.0 + Gi * K) + 1.0 * pk;
            // symmetrize (linalg.cpp:227-235): 0.5 * (lower + upper)
            const double pt = __shfl_sync(kFull, pk, j + NX * i);  // element (j, i)
            if (i > j) pk = 0.5 * (pk + pt);
            if (i < j) pk = 0.5 * (pt + pk);
            aFK[k * NX + j] = K;
            aFG[k * NX + j] = G;
            aFP[(k * NX + j) * NX + i] = pk;
            Pn = pk;
        }
        c = nx;
    }
    __syncwarp();
    // certificates (cert_sqrt_bf / cdiv_seed's), one stage entry per lane
    bool cert = true;
#pragma unroll 1
    for (int k = (int)(threadIdx.x & 31); k < N; k += W) cert &= cert_sqrt_bf(cH[k], aFLL[k]);
#pragma unroll 1
    for (int q = NX + (int)(threadIdx.x & 31); q < N * NX; q += W) {
        const double pl = aFLL[q / NX], q1 = cQ1[q];
        cert &= div_seed_ok(aFG[q], pl, q1) & div_seed_ok(q1, pl, -aFK[q]);
    }
    *cert_out = __all_sync(kFull, cert);
    __syncwarp();
    return false;
}

/// riccati_factor with the certified fast sqrt/division; any uncertified
/// stage (or a fast NotPositiveDefinite) replays the sweep with IEEE ops.
template <int NX, int W>
__device__ __forceinline__ bool rfactor(const QpView<NX, W> v) {
    bool cert = true;
    bool npd;
    if constexpr (W == 32 && NX > 1 && NMPCMC_SPLIT_SWEEPS) {
        npd = rfactor_split<NX>(v, &cert);
    } else {
        npd = rfactor_t<NX, W, true>(v, &cert);
    }
    if (npd || !cert) npd = rfactor_t<NX, W, false>(v, nullptr);
    return npd;
}

/// riccati_solve_vectors (qp.cpp:116-155) for the condensed right-hand side
/// rh = RH, qhat_k = rs(x_k), bhat_k = -rd_k; step into DXI, DMU.
template <int NX, int W, bool FAST>
__device__ __noinline__ bool rsolve_t(const QpView<NX, W> v) {
    bool cert = true;
    const Ocp<NX, W>& o = *v.o;
    const WsT<W> w = o.ws;  // by value: base/stride and the offsets below live in registers
    const Layout<NX> L = o.lay;
    const int oDFF = L.DFF, oDMU = L.DMU, oDXI = L.DXI, oFG = L.FG, oFK = L.FK, oFLL = L.FLL, oFLY = L.FLY, oFP = L.FP, oPV = L.PV, oRD = L.RD, oRH = L.RH, oRS = L.RS;
    const SweepLay<NX> SL(o.N);
    const ArrT<W> aFP = sweep_arr<W>(w, oFP, SL.FP);
    const ArrT<W> aFLL = sweep_arr<W>(w, oFLL, SL.FLL);
    const ArrT<W> aFLY = sweep_arr<W>(w, oFLY, SL.FLY);
    const ArrT<W> aFK = sweep_arr<W>(w, oFK, SL.FK);
    const ArrT<W> aFG = sweep_arr<W>(w, oFG, SL.FG);
    const ArrT<W> aPV = sweep_arr<W>(w, oPV, SL.PV);
    const ArrT<W> aDFF = sweep_arr<W>(w, oDFF, SL.DFF);
    const int oFXs = L.FX[v.s], oFUs = L.FU[v.s], oWB = L.WB, oXIs = L.XI[v.s], oGFs = L.GF[v.s];
    // K3w: the shared-memory copies staged by solve_qp; K3g: the set in place
    const ArrT<W> aJX = jac_arr<W>(w, oFXs, SL.JX);
    const ArrT<W> aJU = jac_arr<W>(w, oFUs, SL.JU);
    auto Jx_ = [&](int k, int i, int j) -> double { return aJX[(k * NX + j) * NX + i]; };
    auto Ju_ = [&](int k, int i) -> double { return aJU[k * NX + i]; };
    const int nN = o.N;
    auto Wb_ = [&](int k, int i, int j) -> double {
        const int ld = k == 0 ? 1 : (k < nN ? NX + 1 : NX);
        return w[oWB + k * Layout<NX>::B + j * ld + i];
    };
    auto R_ = [&](int k) -> double { return k == 0 ? Wb_(0, 0, 0) : Wb_(k, NX, NX); };
    auto Q_ = [&](int k, int i, int j) -> double { return Wb_(k, i, j); };
    auto M_ = [&](int k, int i) -> double { return Wb_(k, i, NX); };
    (void)oXIs, (void)oGFs;

    const int N = o.N;
    auto P = [&](int k, int i, int j) -> double { return aFP[(k * NX + j) * NX + i]; };
    const ArrT<W> aRS = sweep_arr<W>(w, oRS, SL.RS);
    const ArrT<W> aRD = sweep_arr<W>(w, oRD, SL.RD);
    const ArrT<W> aRH = sweep_arr<W>(w, oRH, SL.RH);
    auto bh = [&](int k, int i) -> double { return -aRD[k * NX + i]; };
    double pvn[NX];  // p_{k+1}, carried in registers (see rfactor)
#pragma unroll
    for (int i = 0; i < NX; ++i) {
        pvn[i] = aRS[L.xo(N) + i];
        aPV[N * NX + i] = pvn[i];
    }
#pragma unroll 1
    for (int k = N - 1; k >= 0; --k) {
        double t[NX];
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += P(k + 1, i, j) * bh(k, j);
            t[i] = 1.0 * s + 1.0 * pvn[i];
        }
        double hv;
        {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += Ju_(k, j) * t[j];
            hv = 1.0 * s + 1.0 * aRH[k];
        }
        const double l = aFLL[k];
        if (FAST) {
            const double y = aFLY[k];
            hv = cdiv_seed(hv, l, y, cert);
            hv = cdiv_seed(hv, l, y, cert);
        } else {
            hv = hv / l;
            hv = hv / l;
        }
        const double dff = -hv;
        aDFF[k] = dff;
        if (k >= 1) {
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                double s = 0.0;
#pragma unroll
                for (int j = 0; j < NX; ++j) s += Jx_(k, j, i) * t[j];
                double p = 1.0 * s + 1.0 * aRS[L.xo(k) + i];
                p = 1.0 * (0.0 + aFG[k * NX + i] * dff) + 1.0 * p;
                aPV[k * NX + i] = p;
                pvn[i] = p;
            }
        }
    }
    double dx[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) dx[i] = 0.0;
#pragma unroll 1
    for (int k = 0; k < N; ++k) {
        double du = aDFF[k];
        if (k >= 1) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += aFK[k * NX + j] * dx[j];
            du = 1.0 * s + 1.0 * du;
        }
        w[oDXI + L.uo(k)] = du;
        double dn[NX];
#pragma unroll
        for (int i = 0; i < NX; ++i) dn[i] = bh(k, i);
        if (k >= 1) {
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                double s = 0.0;
#pragma unroll
                for (int j = 0; j < NX; ++j) s += Jx_(k, i, j) * dx[j];
                dn[i] = 1.0 * s + 1.0 * dn[i];
            }
        }
#pragma unroll
        for (int i = 0; i < NX; ++i) dn[i] = 1.0 * (0.0 + Ju_(k, i) * du) + 1.0 * dn[i];
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            dx[i] = dn[i];
            w[oDXI + L.uo(k) + 1 + i] = dx[i];
        }
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += P(k + 1, i, j) * dx[j];
            const double mv = 1.0 * s + 1.0 * aPV[(k + 1) * NX + i];
            w[oDMU + k * NX + i] = -mv;
        }
    }
    return cert;
}

/// riccati_solve_vectors (qp.cpp:116-155), fast forms, one vector component
/// per lane (see rfactor_split). Returns false if a fast division was not
/// certified (the caller replays rsolve_t<FAST=false>). Stage operands, and
/// the recursion-free product P_{k+1} bhat_k, are formed one stage ahead.
template <int NX>
__device__ __noinline__ bool rsolve_split(const QpView<NX, 32> v) {
    constexpr int W = 32;
    constexpr unsigned kFull = 0xffffffffu;
    const Ocp<NX, W>& o = *v.o;
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    const int oDMU = L.DMU, oDXI = L.DXI;
    const SweepLay<NX> SL(o.N);
    const double* const aFP = gen_smem + SL.FP;
    const double* const aFLL = gen_smem + SL.FLL;
    const double* const aFLY = gen_smem + SL.FLY;
    const double* const aFK = gen_smem + SL.FK;
    const double* const aFG = gen_smem + SL.FG;
    double* const aPV = gen_smem + SL.PV;
    double* const aDFF = gen_smem + SL.DFF;
    const double* const aJX = NMPCMC_K3W_NOJX ? w.p + L.FX[v.s] : gen_smem + SL.JX;
    const double* const aJU = NMPCMC_K3W_NOJX ? w.p + L.FU[v.s] : gen_smem + SL.JU;
    const double* const aRS = gen_smem + SL.RS;
    const double* const aRD = gen_smem + SL.RD;
    const double* const aRH = gen_smem + SL.RH;
    // certificate inputs of the two divisions per stage, checked lane-parallel
    // after the backward sweep (TG is free between the gap sums)
    double* const cA = gen_smem + SL.TG;
    const int N = o.N;
    double* const cQ1 = cA + N;
    const int i = (int)(threadIdx.x & 31) % NX;  // this lane's vector component
    double pvn = aRS[L.xo(N) + i];  // p_{k+1}(i)
    aPV[N * NX + i] = pvn;
    // backward: s = (P_{k+1} bhat_k)(i), Ju, rh, the pivot and its seed,
    // column i of Jx, qhat_k(i), G(i)
    struct Back {
        double s, ju[NX], rh, l, y, jx[NX], rs, fg;
    };
    auto load_back = [&](int k) {
        Back n;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NX; ++j) s += aFP[((k + 1) * NX + j) * NX + i] * -aRD[k * NX + j];
        n.s = s;
#pragma unroll
        for (int j = 0; j < NX; ++j) {
            n.ju[j] = aJU[k * NX + j];
            n.jx[j] = aJX[(k * NX + i) * NX + j];
        }
        n.rh = aRH[k];
        n.l = aFLL[k];
        n.y = aFLY[k];
        n.rs = aRS[L.xo(k > 0 ? k : 1) + i];  // unused at k = 0
        n.fg = aFG[k * NX + i];
        return n;
    };
    Back c = load_back(N - 1);
#pragma unroll 1
    for (int k = N - 1; k >= 0; --k) {
        const Back nx = load_back(k > 0 ? k - 1 : 0);
        const double t = 1.0 * c.s + 1.0 * pvn;
        double tj[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) tj[j] = __shfl_sync(kFull, t, j);
        double hv;
        {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += c.ju[j] * tj[j];
            hv = 1.0 * s + 1.0 * c.rh;
        }
        cA[k] = hv;
        hv = div_seed(hv, c.l, c.y);
        cQ1[k] = hv;
        hv = div_seed(hv, c.l, c.y);
        const double dff = -hv;
        aDFF[k] = dff;
        if (k >= 1) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += c.jx[j] * tj[j];
            double p = 1.0 * s + 1.0 * c.rs;
            p = 1.0 * (0.0 + c.fg * dff) + 1.0 * p;
            aPV[k * NX + i] = p;
            pvn = p;
        }
        c = nx;
    }
    bool cert = true;  // every lane stored the same (lane-uniform) certificate inputs
#pragma unroll 1
    for (int k = (int)(threadIdx.x & 31); k < N; k += W) {
        const double pl = aFLL[k], q1 = cQ1[k];
        cert &= div_seed_ok(cA[k], pl, q1) & div_seed_ok(q1, pl, -aDFF[k]);
    }
    if (!__all_sync(kFull, cert)) {
        __syncwarp();
        return false;
    }
    // forward: dff, K, bhat(i), row i of Jx, Ju(i), row i of P_{k+1}, p_{k+1}(i)
    struct Fwd {
        double dff, fk[NX], bh, jx[NX], ju, fp[NX], pv;
    };
    auto load_fwd = [&](int k) {
        Fwd n;
        n.dff = aDFF[k];
#pragma unroll
        for (int j = 0; j < NX; ++j) {
            n.fk[j] = aFK[k * NX + j];  // unused at k = 0
            n.jx[j] = aJX[(k * NX + j) * NX + i];
            n.fp[j] = aFP[((k + 1) * NX + j) * NX + i];
        }
        n.bh = -aRD[k * NX + i];
        n.ju = aJU[k * NX + i];
        n.pv = aPV[(k + 1) * NX + i];
        return n;
    };
    double dx[NX];  // the whole state step, on every lane
#pragma unroll
    for (int j = 0; j < NX; ++j) dx[j] = 0.0;
    Fwd f = load_fwd(0);
#pragma unroll 1
    for (int k = 0; k < N; ++k) {
        const Fwd nf = load_fwd(k + 1 < N ? k + 1 : k);
        double du = f.dff;
        if (k >= 1) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += f.fk[j] * dx[j];
            du = 1.0 * s + 1.0 * du;
        }
        double dn = f.bh;
        if (k >= 1) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += f.jx[j] * dx[j];
            dn = 1.0 * s + 1.0 * dn;
        }
        dn = 1.0 * (0.0 + f.ju * du) + 1.0 * dn;
#pragma unroll
        for (int j = 0; j < NX; ++j) dx[j] = __shfl_sync(kFull, dn, j);
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NX; ++j) s += f.fp[j] * dx[j];
        const double mv = 1.0 * s + 1.0 * f.pv;
        w[oDXI + L.uo(k)] = du;
        w[oDXI + L.uo(k) + 1 + i] = dn;
        w[oDMU + k * NX + i] = -mv;
        f = nf;
    }
    __syncwarp();
    return true;
}

/// riccati_solve_vectors with the certified fast division (replayed with
/// IEEE ops if any quotient is not certified).
template <int NX, int W>
__device__ __forceinline__ void rsolve(const QpView<NX, W> v) {
    bool ok;
    if constexpr (W == 32 && NX > 1 && NMPCMC_SPLIT_SWEEPS) {
        ok = rsolve_split<NX>(v);
    } else {
        ok = rsolve_t<NX, W, true>(v);
    }
    if (!ok) rsolve_t<NX, W, false>(v);
}

enum : int { QP_OPTIMAL = 0, QP_MAXITER = 1, QP_FAILED = 2, QP_DOMAIN = 3 };

/// residuals (qp.cpp:237-284) into RS, RD, RL, RU.
template <int NX, int W>
__device__ __noinline__ void qp_resid(const QpView<NX, W> v) {
    const Ocp<NX, W>& o = *v.o;
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    const int N = o.N;
    const SweepLay<NX> SL(N);
    const ArrT<W> aRS = sweep_arr<W>(w, L.RS, SL.RS);
    const ArrT<W> aRD = sweep_arr<W>(w, L.RD, SL.RD);
    auto dxi = [&](int e) -> double { return w[L.QDXI + e]; };
#pragma unroll 1
    for (int k = Lanes<W>::lane(); k < N; k += W) {
        const double vk = dxi(L.uo(k));
        double r = 1.0 * (0.0 + v.R(k) * vk) + 1.0 * v.r(k);
        if (k >= 1) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += v.M(k, j) * dxi(L.xo(k) + j);
            r = 1.0 * s + 1.0 * r;
        }
        {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += v.Ju(k, j) * w[L.QMU + k * NX + j];
            r = -1.0 * s + 1.0 * r;
        }
        r += w[L.QNU + k] - w[L.QNL + k];
        aRS[L.uo(k)] = r;
        double d[NX];
#pragma unroll
        for (int i = 0; i < NX; ++i) d[i] = dxi(L.xo(k + 1) + i) + -1.0 * v.b(k, i);
        if (k >= 1) {
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                double s = 0.0;
#pragma unroll
                for (int j = 0; j < NX; ++j) s += v.Jx(k, i, j) * dxi(L.xo(k) + j);
                d[i] = -1.0 * s + 1.0 * d[i];
            }
        }
#pragma unroll
        for (int i = 0; i < NX; ++i) aRD[k * NX + i] = -1.0 * (0.0 + v.Ju(k, i) * vk) + 1.0 * d[i];
    }
#pragma unroll 1
    for (int k = 1 + Lanes<W>::lane(); k <= N; k += W) {
        double x[NX];
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NX; ++j) s += v.Q(k, i, j) * dxi(L.xo(k) + j);
            x[i] = 1.0 * s + 1.0 * v.q(k, i);
        }
        if (k < N) {
            const double uk = dxi(L.uo(k));
#pragma unroll
            for (int i = 0; i < NX; ++i) x[i] = 1.0 * (0.0 + v.M(k, i) * uk) + 1.0 * x[i];
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                double s = 0.0;
#pragma unroll
                for (int j = 0; j < NX; ++j) s += v.Jx(k, j, i) * w[L.QMU + k * NX + j];
                x[i] = -1.0 * s + 1.0 * x[i];
            }
        }
#pragma unroll
        for (int i = 0; i < NX; ++i) aRS[L.xo(k) + i] = x[i] + w[L.QMU + (k - 1) * NX + i];
    }
#pragma unroll 1
    for (int k = Lanes<W>::lane(); k < N; k += W) {
        const double vk = dxi(L.uo(k));
        const double lb = v.lb(k), ub = v.ub(k);
        w[L.RL + k] = dfinite(lb) ? vk - w[L.SL + k] - lb : 0.0;
        w[L.RU + k] = dfinite(ub) ? ub - vk - w[L.SU + k] : 0.0;
    }
    Lanes<W>::sync();
}

/// Condensed right-hand side (qp.cpp:288-305) into RH, then the vector solve.
template <int NX, int W>
__device__ __forceinline__ void qp_csolve(const QpView<NX, W> v) {
    const Ocp<NX, W>& o = *v.o;
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    const SweepLay<NX> SL(o.N);
    const ArrT<W> aRS = sweep_arr<W>(w, L.RS, SL.RS);
    const ArrT<W> aRH = sweep_arr<W>(w, L.RH, SL.RH);
#pragma unroll 1
    for (int k = Lanes<W>::lane(); k < o.N; k += W) {
        double x = aRS[L.uo(k)];
        if (dfinite(v.lb(k))) x -= (w[L.CL + k] - w[L.QNL + k] * w[L.RL + k]) / w[L.SL + k];
        if (dfinite(v.ub(k))) x += (w[L.CU + k] - w[L.QNU + k] * w[L.RU + k]) / w[L.SU + k];
        aRH[k] = x;
    }
    Lanes<W>::sync();
    rsolve<NX, W>(v);
    Lanes<W>::sync();
}
/// expand (qp.cpp:308-317) of the step in DXI.
template <int NX, int W>
__device__ __forceinline__ void qp_expand(const QpView<NX, W> v) {
    const Ocp<NX, W>& o = *v.o;
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
#pragma unroll 1
    for (int k = Lanes<W>::lane(); k < o.N; k += W) {
        const double dv = w[L.DXI + L.uo(k)];
        const bool fl = dfinite(v.lb(k)), fu = dfinite(v.ub(k));
        const double dsl = fl ? dv + w[L.RL + k] : 0.0;
        const double dsu = fu ? w[L.RU + k] - dv : 0.0;
        w[L.DSL + k] = dsl;
        w[L.DSU + k] = dsu;
        w[L.DNL + k] = fl ? (w[L.CL + k] - w[L.QNL + k] * dsl) / w[L.SL + k] : 0.0;
        w[L.DNU + k] = fu ? (w[L.CU + k] - w[L.QNU + k] * dsu) / w[L.SU + k] : 0.0;
    }
    Lanes<W>::sync();
}
/// max_step (qp.cpp:321-337).
template <int NX, int W>
__device__ __forceinline__ double qp_step(const QpView<NX, W> v, double frac) {
    const Ocp<NX, W>& o = *v.o;
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    double a = 1.0;
    auto cap = [&](double val, double dir) {
        if (dir < 0.0) a = smin(a, -frac * val / dir);
    };
#pragma unroll 1
    for (int k = Lanes<W>::lane(); k < o.N; k += W) {
        if (dfinite(v.lb(k))) cap(w[L.SL + k], w[L.DSL + k]), cap(w[L.QNL + k], w[L.DNL + k]);
        if (dfinite(v.ub(k))) cap(w[L.SU + k], w[L.DSU + k]), cap(w[L.QNU + k], w[L.DNU + k]);
    }
    return Lanes<W>::min_fold(a);
}

__device__ __forceinline__ double inf_fold(double m, double x) { return smax(m, fabs(x)); }

/// solve_qp (qp.cpp:173-423): Mehrotra predictor-corrector interior point.
/// Result in QDXI, QMU, QNL, QNU.
template <int NX, int W>
__device__ __noinline__ int solve_qp(const QpView<NX, W> v, double tol, int max_iter, int* iters_out = nullptr) {
    const Ocp<NX, W>& o = *v.o;
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    const int N = o.N, lane = Lanes<W>::lane();
    const SweepLay<NX> SLq(N);
    const ArrT<W> aRSq = sweep_arr<W>(w, L.RS, SLq.RS);
    const ArrT<W> aRDq = sweep_arr<W>(w, L.RD, SLq.RD);
    if (W > 1) {  // stage the QP's constant operands (SweepLay JX JU LB UB RR QQ)
        if (!NMPCMC_K3W_NOJX) {
            for (int e = lane; e < N * NX * NX; e += W) gen_smem[SLq.JX + e] = w[L.FX[v.s] + e];
            for (int e = lane; e < N * NX; e += W) gen_smem[SLq.JU + e] = w[L.FU[v.s] + e];
        }
#pragma unroll 1
        for (int k = lane; k <= N; k += W) {
            if (k < N) {
                gen_smem[SLq.LB + k] = v.lb_src(k);
                gen_smem[SLq.UB + k] = v.ub_src(k);
                if (!NMPCMC_K3W_NOQQ) gen_smem[SLq.RR + k] = v.R(k);
            }
            if (!NMPCMC_K3W_NOQQ) {
#pragma unroll
                for (int j = 0; j < NX; ++j)
#pragma unroll
                    for (int i = 0; i < NX; ++i)
                        gen_smem[SLq.QQ + (k * NX + j) * NX + i] = k == 0 ? 0.0 : v.Q(k, i, j);
            }
        }
        Lanes<W>::sync();
    }
    int m = 0;
    double scale = 1.0;  // data_scale: an order-independent max (NaN ignored)
    bool domain = false;
#pragma unroll 1
    for (int k = lane; k < N; k += W) {
        const double lb = v.lb(k), ub = v.ub(k);
        if (lb > ub) domain = true;
        if (dfinite(lb)) ++m, scale = smax(scale, fabs(lb));
        if (dfinite(ub)) ++m, scale = smax(scale, fabs(ub));
        scale = smax(scale, inf_fold(0.0, v.r(k)));
        double nb = 0.0;
#pragma unroll
        for (int i = 0; i < NX; ++i) nb = inf_fold(nb, v.b(k, i));
        scale = smax(scale, nb);
    }
    if (Lanes<W>::any(domain)) return QP_DOMAIN;
#pragma unroll 1
    for (int k = 1 + lane; k <= N; k += W) {
        double nq = 0.0;
#pragma unroll
        for (int i = 0; i < NX; ++i) nq = inf_fold(nq, v.q(k, i));
        scale = smax(scale, nq);
    }
    m = Lanes<W>::sum(m);
    scale = Lanes<W>::max_fold(scale);
    const double eps = tol * scale;
    for (int e = lane; e < L.L; e += W) w[L.QDXI + e] = 0.0;
    for (int e = lane; e < L.NN; e += W) w[L.QMU + e] = 0.0;
#pragma unroll 1
    for (int k = lane; k < N; k += W) {
        const double lb = v.lb(k), ub = v.ub(k);
        const bool fl = dfinite(lb), fu = dfinite(ub);
        w[L.SL + k] = fl ? smax(1.0, fabs(lb)) : 0.0;
        w[L.QNL + k] = fl ? 1.0 : 0.0;
        w[L.SU + k] = fu ? smax(1.0, fabs(ub)) : 0.0;
        w[L.QNU + k] = fu ? 1.0 : 0.0;
        w[L.CL + k] = 0.0;
        w[L.CU + k] = 0.0;
    }
    Lanes<W>::sync();
    int status = QP_FAILED;
    int it = 0;  // completed iterations (QpSolution::iterations, qp.cpp:410)
#pragma unroll 1
    for (;; ++it) {
        qp_resid<NX, W>(v);
        double gap = 0.0;
        if (m > 0) {  // ordered sums: products lane-parallel, sums serial on every lane
            const ArrT<W> aTG = sweep_arr<W>(w, L.FLL, SLq.TG);
            double dl = 0.0, du = 0.0;
            if (W > 1) {
#pragma unroll 1
                for (int k = lane; k < N; k += W) {
                    aTG[k] = w[L.SL + k] * w[L.QNL + k];
                    aTG[N + k] = w[L.SU + k] * w[L.QNU + k];
                }
                Lanes<W>::sync();
#pragma unroll 1
                for (int k = 0; k < N; ++k) dl += aTG[k];
#pragma unroll 1
                for (int k = 0; k < N; ++k) du += aTG[N + k];
                Lanes<W>::sync();
            } else {
#pragma unroll 1
                for (int k = 0; k < N; ++k) dl += w[L.SL + k] * w[L.QNL + k];
#pragma unroll 1
                for (int k = 0; k < N; ++k) du += w[L.SU + k] * w[L.QNU + k];
            }
            gap = (dl + du) / m;
        }
        double ns = 0.0, nd = 0.0, nl = 0.0, nu = 0.0;
        for (int e = lane; e < L.L; e += W) ns = inf_fold(ns, aRSq[e]);
        for (int e = lane; e < L.NN; e += W) nd = inf_fold(nd, aRDq[e]);
#pragma unroll 1
        for (int k = lane; k < N; k += W) {
            nl = inf_fold(nl, w[L.RL + k]);
            nu = inf_fold(nu, w[L.RU + k]);
        }
        ns = Lanes<W>::max_fold(ns);
        nd = Lanes<W>::max_fold(nd);
        nl = Lanes<W>::max_fold(nl);
        nu = Lanes<W>::max_fold(nu);
        if (ns <= eps && nd <= eps && nl <= eps && nu <= eps && gap <= eps) {
            status = QP_OPTIMAL;
            break;
        }
        if (it >= max_iter) {
            status = QP_MAXITER;
            break;
        }
#pragma unroll 1
        for (int k = lane; k < N; k += W) {
            double b = 0.0;
            if (dfinite(v.lb(k))) b += w[L.QNL + k] / w[L.SL + k];
            if (dfinite(v.ub(k))) b += w[L.QNU + k] / w[L.SU + k];
            w[L.BAR + k] = b;
        }
        Lanes<W>::sync();
        const bool npd = rfactor<NX, W>(v);
        Lanes<W>::sync();
        if (npd) {
            status = QP_FAILED;
            break;
        }
#pragma unroll 1
        for (int k = lane; k < N; k += W) {
            w[L.CL + k] = dfinite(v.lb(k)) ? -w[L.SL + k] * w[L.QNL + k] : 0.0;
            w[L.CU + k] = dfinite(v.ub(k)) ? -w[L.SU + k] * w[L.QNU + k] : 0.0;
        }
        qp_csolve<NX, W>(v);
        qp_expand<NX, W>(v);
        double sig = 0.0;
        if (m > 0 && gap > 0.0) {
            const double aa = qp_step<NX, W>(v, 1.0);
            double ga = 0.0;
            if (W > 1) {
                // products lane-parallel, the ordered sum serial on every lane;
                // an absent bound contributes +0.0, which leaves ga unchanged
                // (ga starts at +0 and a sum from +0 is never -0)
#pragma unroll 1
                for (int k = lane; k < N; k += W) {
                    gen_smem[SLq.TG + 2 * k] =
                        dfinite(v.lb(k)) ? (w[L.SL + k] + aa * w[L.DSL + k]) * (w[L.QNL + k] + aa * w[L.DNL + k])
                                         : 0.0;
                    gen_smem[SLq.TG + 2 * k + 1] =
                        dfinite(v.ub(k)) ? (w[L.SU + k] + aa * w[L.DSU + k]) * (w[L.QNU + k] + aa * w[L.DNU + k])
                                         : 0.0;
                }
                Lanes<W>::sync();
#pragma unroll 1
                for (int e = 0; e < 2 * N; ++e) ga += gen_smem[SLq.TG + e];
                Lanes<W>::sync();
            } else {
#pragma unroll 1
                for (int k = 0; k < N; ++k) {
                    if (dfinite(v.lb(k)))
                        ga += (w[L.SL + k] + aa * w[L.DSL + k]) * (w[L.QNL + k] + aa * w[L.DNL + k]);
                    if (dfinite(v.ub(k)))
                        ga += (w[L.SU + k] + aa * w[L.DSU + k]) * (w[L.QNU + k] + aa * w[L.DNU + k]);
                }
            }
            ga /= m;
            const double ratio = smax(0.0, ga / gap);
            sig = smin(1.0, ratio * ratio * ratio);
        }
#pragma unroll 1
        for (int k = lane; k < N; k += W) {
            if (dfinite(v.lb(k)))
                w[L.CL + k] = sig * gap - w[L.SL + k] * w[L.QNL + k] - w[L.DSL + k] * w[L.DNL + k];
            if (dfinite(v.ub(k)))
                w[L.CU + k] = sig * gap - w[L.SU + k] * w[L.QNU + k] - w[L.DSU + k] * w[L.DNU + k];
        }
        qp_csolve<NX, W>(v);
        qp_expand<NX, W>(v);
        const double a = qp_step<NX, W>(v, 0.995);
        for (int e = lane; e < L.L; e += W) w[L.QDXI + e] += a * w[L.DXI + e];
        for (int e = lane; e < L.NN; e += W) w[L.QMU + e] += a * w[L.DMU + e];
#pragma unroll 1
        for (int k = lane; k < N; k += W) {
            if (dfinite(v.lb(k))) {
                w[L.SL + k] += a * w[L.DSL + k];
                w[L.QNL + k] += a * w[L.DNL + k];
            }
            if (dfinite(v.ub(k))) {
                w[L.SU + k] += a * w[L.DSU + k];
                w[L.QNU + k] += a * w[L.DNU + k];
            }
        }
        Lanes<W>::sync();
        o.cnt->ipm_stage += N;
    }
#pragma unroll 1
    for (int k = lane; k < N; k += W) {
        double& x = w[L.QDXI + L.uo(k)];
        x = smin(smax(x, v.lb(k)), v.ub(k));
    }
    Lanes<W>::sync();
    if (iters_out) *iters_out = it;
    return status;
}

// -------------------------------------------------------------------- SQP
/// h += J_g' lam (add_constraint_term, sqp.cpp:102-116) on the blocks of
/// set s; h at element offset H.
template <int NX, int W>
__device__ void add_jt(const Ocp<NX, W>& o, int s, int LAMo, int H) {
    // lane-parallel by slot ownership: unit k owns u_k and x_{k+1}; per slot
    // the reference's order is kept: x_{k+1} gets + lam_k (iteration k), then
    // - Fx_{k+1}' lam_{k+1} term by term (iteration k+1)
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
#pragma unroll 1
    for (int k = Lanes<W>::lane(); k < o.N; k += W) {
#pragma unroll
        for (int j = 0; j < NX; ++j) w[H + L.uo(k)] -= w[L.FU[s] + k * NX + j] * w[LAMo + k * NX + j];
        const int kn = k + 1;
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            double h = w[H + L.xo(kn) + i] + w[LAMo + k * NX + i];
            if (kn < o.N) {
#pragma unroll
                for (int j = 0; j < NX; ++j)
                    h -= w[L.FX[s] + (kn * NX + i) * NX + j] * w[LAMo + kn * NX + j];
            }
            w[H + L.xo(kn) + i] = h;
        }
    }
    Lanes<W>::sync();
}

/// lagrangian_gradient (sqp.cpp:118-128) into HO for duals (LAMo, PLo, PUo),
/// then check_convergence (sqp.cpp:86-96).
template <int NX, int W>
__device__ __noinline__ bool kkt_ok(const Ocp<NX, W>& o, int s, int LAMo, int PLo, int PUo, int m,
                                    double eps, double* gl_out = nullptr, double* gg_out = nullptr) {
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    const int lane = Lanes<W>::lane();
    for (int e = lane; e < L.L; e += W) w[L.HO + e] = w[L.GF[s] + e];
    Lanes<W>::sync();
    add_jt<NX, W>(o, s, LAMo, L.HO);
#pragma unroll 1
    for (int k = lane; k < o.N; k += W) w[L.HO + L.uo(k)] += w[PUo + k] - w[PLo + k];
    Lanes<W>::sync();
    double sd = 1.0;
    if (m > 0) {  // ordered one-norm sums (ordered_sum: terms lane-parallel on K3w)
        const SweepLay<NX> SL(o.N);
        // scratch outside solve_qp: its staged jacobians, or its residual arrays RS RD
        double* scr = W > 1 ? gen_smem + (NMPCMC_K3W_NOJX ? SL.RS : SL.JX) : nullptr;
        const int cap = NMPCMC_K3W_NOJX ? o.N * (2 * NX + 1) : o.N * NX * (NX + 1);
        const double a = ordered_sum<W>(0.0, L.NN, scr, cap, [&](int e) { return fabs(w[LAMo + e]); });
        const double b = ordered_sum<W>(0.0, o.N, scr, cap, [&](int k) { return fabs(w[PLo + k]); });
        const double c = ordered_sum<W>(0.0, o.N, scr, cap, [&](int k) { return fabs(w[PUo + k]); });
        sd = smax(100.0, (a + b + c) / m) / 100.0;
    }
    double gl = 0.0, gg = 0.0;
    for (int e = lane; e < L.L; e += W) gl = inf_fold(gl, w[L.HO + e]);
    for (int e = lane; e < L.NN; e += W) gg = inf_fold(gg, w[L.G[s] + e]);
    gl = Lanes<W>::max_fold(gl);
    gg = Lanes<W>::max_fold(gg);
    if (gl_out) *gl_out = gl;  // rep.grad_l_inf / rep.g_inf (sqp.cpp:249-250)
    if (gg_out) *gg_out = gg;
    return gl / sd <= eps && gg <= eps;
}

/// reset_blocks (sqp.cpp:173-178): identities of size 1, nx+1, ..., nx.
template <int NX, int W>
__device__ void identity_blocks(const Ocp<NX, W>& o) {
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
#pragma unroll 1
    for (int k = Lanes<W>::lane(); k <= o.N; k += W) {
        const int n = k == 0 ? 1 : (k < o.N ? NX + 1 : NX);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) w[L.WB + k * Layout<NX>::B + j * n + i] = (i == j) ? 1.0 : 0.0;
    }
    Lanes<W>::sync();
}

/// bfgs_block_update (sqp.cpp:61-84) of block k with s, y of length n.
/// Returns true on NotPositiveDefinite (the Cholesky audit).
template <int NX, int W>
__device__ bool bfgs_block(const Ocp<NX, W>& o, int k, int n, const double* s, const double* y) {
    const WsT<W> w = o.ws;
    const int base = o.lay.WB + k * Layout<NX>::B;
    auto Wm = [&](int i, int j) -> double& { return w[base + j * n + i]; };
    double Ws_[NX + 1];
    for (int i = 0; i < n; ++i) {
        double a = 0.0;
        for (int j = 0; j < n; ++j) a += Wm(i, j) * s[j];
        Ws_[i] = 1.0 * a + 0.0;
    }
    const double tiny = 0x1.0p-52;
    double sWs = 0.0;
    for (int i = 0; i < n; ++i) sWs += s[i] * Ws_[i];
    if (!(sWs > tiny)) return false;
    double sy = 0.0;
    for (int i = 0; i < n; ++i) sy += s[i] * y[i];
    const double th = sy >= 0.2 * sWs ? 1.0 : 0.8 * sWs / (sWs - sy);
    double r[NX + 1];
    for (int i = 0; i < n; ++i) r[i] = th * y[i] + (1.0 - th) * Ws_[i];
    double sr = 0.0;
    for (int i = 0; i < n; ++i) sr += s[i] * r[i];
    if (!(smin(sWs, sr) > tiny)) return false;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) Wm(i, j) += r[i] * r[j] / sr - Ws_[i] * Ws_[j] / sWs;
    for (int j = 0; j < n; ++j)
        for (int i = j + 1; i < n; ++i) {
            const double mm = 0.5 * (Wm(i, j) + Wm(j, i));
            Wm(i, j) = mm;
            Wm(j, i) = mm;
        }
    // cholesky_factor audit (linalg.cpp:69-103)
    double Lc[(NX + 1) * (NX + 1)];
    for (int e = 0; e < n * n; ++e) Lc[e] = 0.0;
    for (int j = 0; j < n; ++j) {
        double d = Wm(j, j);
        for (int q = 0; q < j; ++q) d -= Lc[q * n + j] * Lc[q * n + j];
        if (d <= 0.0 || !dfinite(d)) return true;
        const double p = sqrt(d);
        Lc[j * n + j] = p;
        for (int i = j + 1; i < n; ++i) {
            double a = Wm(i, j);
            for (int q = 0; q < j; ++q) a -= Lc[q * n + i] * Lc[q * n + j];
            Lc[j * n + i] = a / p;
        }
    }
    return false;
}

struct SqpOut {
    bool converged;
    int status;  // G_DOMAIN escapes sqp_solve
};

/// sqp_solve (sqp.cpp:182-411) from the iterate in XI[0] and duals LAM/PL/PU.
/// On return the iterate is in XI[*cur].
template <int NX, int W>
__device__ __noinline__ SqpOut sqp_solve(const Ocp<NX, W>& o, const nmpcmc_sqp_options& op, int* cur) {
    const WsT<W> w = o.ws;
    const Layout<NX> L = o.lay;
    const int N = o.N, lane = Lanes<W>::lane();
    const int m = N * NX + (dfinite(o.umin) ? N : 0) + (dfinite(o.umax) ? N : 0);
    int s = 0;
    *cur = 0;
    identity_blocks<NX, W>(o);
    double f = objective<NX, W>(o, s, true);
    {
        const int st = constraints<NX, W>(o, s);
        if (st == G_DOMAIN) return SqpOut{false, G_DOMAIN};
        if (st != G_OK) return SqpOut{false, G_OK};
    }
    bool first = true;
    // SqpIterationLog records (sqp.hpp:64-77) when a trace buffer is given;
    // pushed where sqp.cpp pushes them (:274, :327, :350, :406)
    int n_log = 0;
    nmpcmc_sqp_iter_log lg{};
    auto push_log = [&]() {
        if (o.trace != nullptr && n_log < o.trace_cap && lane == 0) o.trace[n_log] = lg;
        ++n_log;
    };
    auto finish_log = [&]() {
        if (o.trace_len != nullptr && lane == 0) *o.trace_len = n_log;
    };
#pragma unroll 1
    for (int it = 0;; ++it) {
        double gl0 = 0.0, gg0 = 0.0;
        if (kkt_ok<NX, W>(o, s, L.LAM, L.PL, L.PU, m, op.eps, &gl0, &gg0)) {
            finish_log();
            return SqpOut{true, G_OK};
        }
        if (it >= op.max_iter) break;
        lg = nmpcmc_sqp_iter_log{};
        lg.qp_status = QP_FAILED;
        lg.grad_l_inf = gl0;
        lg.g_inf = gg0;
        o.cnt->sqp_stage += N;
        const QpView<NX, W> v(&o, s);
        int qit = 0;
        int qs = solve_qp<NX, W>(v, op.qp_tol, op.qp_max_iter, &qit);
        o.cnt->qp += 1;
        if (qs == QP_DOMAIN) return SqpOut{false, G_DOMAIN};
        if (qs == QP_FAILED) {
            identity_blocks<NX, W>(o);
            lg.bfgs_reset = 1;
            qs = solve_qp<NX, W>(v, op.qp_tol, op.qp_max_iter, &qit);
            o.cnt->qp += 1;
            if (qs == QP_DOMAIN) return SqpOut{false, G_DOMAIN};
            if (qs == QP_FAILED) {
                push_log();
                break;
            }
        }
        lg.qp_iterations = qit;
        lg.qp_status = qs;
        if (kkt_ok<NX, W>(o, s, L.QMU, L.QNL, L.QNU, m, op.eps)) {
            for (int e = lane; e < L.NN; e += W) w[L.LAM + e] = w[L.QMU + e];
#pragma unroll 1
            for (int k = lane; k < N; k += W) {
                w[L.PL + k] = w[L.QNL + k];
                w[L.PU + k] = w[L.QNU + k];
            }
            Lanes<W>::sync();
            finish_log();
            return SqpOut{true, G_OK};
        }
        // merit_weights_update (sqp.cpp:12-20)
        for (int e = lane; e < L.NN; e += W) {
            const double am = fabs(w[L.QMU + e]);
            w[L.SIG + e] = first ? am : smax(am, 0.5 * (w[L.SIG + e] + am));
        }
        Lanes<W>::sync();
        first = false;
        // line_search (sqp.cpp:22-59); the trial of the accepted step is the
        // new iterate (identical by construction, sqp.cpp:331-352)
        const SweepLay<NX> SLs(N);
        // scratch outside solve_qp: its staged jacobians, or its residual arrays RS RD
        double* scr = W > 1 ? gen_smem + (NMPCMC_K3W_NOJX ? SLs.RS : SLs.JX) : nullptr;
        const int cap = NMPCMC_K3W_NOJX ? N * (2 * NX + 1) : N * NX * (NX + 1);
        const double pen =
            ordered_sum<W>(0.0, L.NN, scr, cap, [&](int e) { return w[L.SIG + e] * fabs(w[L.G[s] + e]); });
        const double m0 = f + pen;
        const double gd =
            ordered_sum<W>(0.0, L.L, scr, cap, [&](int e) { return w[L.GF[s] + e] * w[L.QDXI + e]; });
        const double dd = gd - pen;
        const int t = 1 - s;
        double a = 1.0, merit = 0.0, ft = 0.0;
        bool ok = false, tfin = false;
        int evals = 0;
#pragma unroll 1
        for (int bt = 0;; ++bt) {
            for (int e = lane; e < L.L; e += W) w[L.XI[t] + e] = w[L.XI[s] + e] + a * w[L.QDXI + e];
            Lanes<W>::sync();
            merit = __longlong_as_double(0x7ff0000000000000LL);
            ft = objective<NX, W>(o, t, true);
            const int st = constraints<NX, W>(o, t);
            if (st == G_DOMAIN) return SqpOut{false, G_DOMAIN};
            o.cnt->ls += 1;  // counted like K3: a trial that raises DomainError ends the solve uncounted
            ++evals;
            tfin = st == G_OK;
            if (tfin)
                merit = ordered_sum<W>(ft, L.NN, scr, cap, [&](int e) { return w[L.SIG + e] * fabs(w[L.G[t] + e]); });
            ok = dfinite(merit) && merit <= m0 + op.c1 * a * dd;
            if (ok || bt >= op.max_backtracks) break;
            a *= op.backtrack_factor;
        }
        lg.alpha = a;
        lg.merit_before = m0;
        lg.merit_after = merit;
        lg.directional_derivative = dd;
        lg.ls_evals = evals;
        lg.armijo_exhausted = ok ? 0 : 1;
        if (!ok && !dfinite(merit)) {
            push_log();
            break;
        }
        if (o.trace != nullptr) {  // step_inf = max |alpha dxi| (std::max: NaN ignored)
            double si = 0.0;
            for (int e = lane; e < L.L; e += W) si = inf_fold(si, a * w[L.QDXI + e]);
            lg.step_inf = Lanes<W>::max_fold(si);
        }
        if (!tfin) {  // the re-evaluation at xn would throw NonFiniteState
            push_log();
            break;
        }
        // duals (sqp.cpp:355-364)
        for (int e = lane; e < L.NN; e += W) w[L.LAM + e] += a * (w[L.QMU + e] - w[L.LAM + e]);
#pragma unroll 1
        for (int k = lane; k < N; k += W) {
            w[L.PL + k] += a * (w[L.QNL + k] - w[L.PL + k]);
            w[L.PU + k] += a * (w[L.QNU + k] - w[L.PU + k]);
        }
        // BFGS on the Lagrangian gradients with the new multipliers (sqp.cpp:366-396)
        for (int e = lane; e < L.L; e += W) {
            w[L.HO + e] = w[L.GF[s] + e];
            w[L.HN + e] = w[L.GF[t] + e];
        }
        Lanes<W>::sync();
        add_jt<NX, W>(o, s, L.LAM, L.HO);
        add_jt<NX, W>(o, t, L.LAM, L.HN);
        // blocks are independent; a lost block resets all of them below, so
        // updating the others in parallel changes nothing (sqp.cpp:377-396)
        bool lost = false;
#pragma unroll 1
        for (int blk = lane; blk <= N && !lost; blk += W) {
            const int off = blk == 0 ? 0 : (blk < N ? L.xo(blk) : L.xo(N));
            const int len = blk == 0 ? 1 : (blk < N ? NX + 1 : NX);
            double sv[NX + 1], yv[NX + 1];
            for (int i = 0; i < len; ++i) {
                sv[i] = a * w[L.QDXI + off + i];
                yv[i] = w[L.HN + off + i] - w[L.HO + off + i];
            }
            lost = bfgs_block<NX, W>(o, blk, len, sv, yv);
        }
        lost = Lanes<W>::any(lost);
        Lanes<W>::sync();
        if (lost) {
            identity_blocks<NX, W>(o);
            lg.bfgs_reset = 1;
        }
        f = ft;
        s = t;
        *cur = s;
        o.cnt->sqp += 1;  // completed SQP steps, as K3 counts them
        push_log();
    }
    finish_log();
    return SqpOut{false, G_OK};
}

// ------------------------------------------------------------------- EKF
/// predict (ekf.cpp:26-57): np RK4 steps on (x, P), P symmetrised per step.
template <int NX>
__device__ __noinline__ int ekf_predict(const Model<NX>& m, double* x, double* P, double u, double t, double tn,
                                        int np) {
    const double h = (tn - t) / np;
    const double f = u * kMlMinToLs;
    double sd[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) sd[i] = f * m.sb[i];
#pragma unroll 1
    for (int step = 0; step < np; ++step) {
        double ax[NX], aP[NX * NX], pk[NX], pP[NX * NX];
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
            double xs[NX], Ps[NX * NX];
            const double c = (j == 3) ? 1.0 : 0.5;
#pragma unroll
            for (int i = 0; i < NX; ++i) xs[i] = j == 0 ? x[i] : (j == 3 ? x[i] + h * pk[i] : x[i] + c * h * pk[i]);
#pragma unroll
            for (int e = 0; e < NX * NX; ++e)
                Ps[e] = j == 0 ? P[e] : (j == 3 ? P[e] + h * pP[e] : P[e] + c * h * pP[e]);
            double dx[NX], A[NX * NX], dP[NX * NX];
            const int st = drift_jac<NX>(m, xs, u, dx, A);
            if (st) return st;
#pragma unroll
            for (int jj = 0; jj < NX; ++jj)  // dP = A P
#pragma unroll
                for (int i = 0; i < NX; ++i) {
                    double s = 0.0;
#pragma unroll
                    for (int l = 0; l < NX; ++l) s += A[l * NX + i] * Ps[jj * NX + l];
                    dP[jj * NX + i] = 1.0 * s + 0.0;
                }
#pragma unroll
            for (int jj = 0; jj < NX; ++jj)  // + P A'
#pragma unroll
                for (int i = 0; i < NX; ++i) {
                    double s = 0.0;
#pragma unroll
                    for (int l = 0; l < NX; ++l) s += Ps[l * NX + i] * A[l * NX + jj];
                    dP[jj * NX + i] = 1.0 * s + 1.0 * dP[jj * NX + i];
                }
#pragma unroll
            for (int jj = 0; jj < NX; ++jj)  // + s s' (diagonal s, all terms)
#pragma unroll
                for (int i = 0; i < NX; ++i) {
                    double s = 0.0;
#pragma unroll
                    for (int l = 0; l < NX; ++l) s += (i == l ? sd[i] : 0.0) * (jj == l ? sd[jj] : 0.0);
                    dP[jj * NX + i] = 1.0 * s + 1.0 * dP[jj * NX + i];
                }
            const double wgt = (j == 1 || j == 2) ? 2.0 : 1.0;
#pragma unroll
            for (int i = 0; i < NX; ++i) {
                ax[i] = j == 0 ? dx[i] : ax[i] + wgt * dx[i];
                pk[i] = dx[i];
            }
#pragma unroll
            for (int e = 0; e < NX * NX; ++e) {
                aP[e] = j == 0 ? dP[e] : aP[e] + wgt * dP[e];
                pP[e] = dP[e];
            }
        }
        const double h6 = h / 6.0;
#pragma unroll
        for (int i = 0; i < NX; ++i) x[i] += h6 * ax[i];
#pragma unroll
        for (int e = 0; e < NX * NX; ++e) P[e] += h6 * aP[e];
#pragma unroll
        for (int jj = 0; jj < NX; ++jj)
#pragma unroll
            for (int i = jj + 1; i < NX; ++i) {
                const double mm = 0.5 * (P[jj * NX + i] + P[i * NX + jj]);
                P[jj * NX + i] = mm;
                P[i * NX + jj] = mm;
            }
        bool fin = true;
#pragma unroll
        for (int i = 0; i < NX; ++i) fin = fin && dfinite(x[i]);
#pragma unroll
        for (int e = 0; e < NX * NX; ++e) fin = fin && dfinite(P[e]);
        if (!fin) return G_NONFINITE;
    }
    return G_OK;
}

/// filter_update (ekf.cpp:59-96), Joseph form, n_y = 1. Returns true on
/// NotPositiveDefinite of R_e.
template <int NX>
__device__ __noinline__ bool ekf_update(const Model<NX>& m, double* x, double* P, double y, double R) {
    const double cv = meas_jac_T<NX>(m, x[NX - 1]);
    double C[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) C[i] = (i == NX - 1) ? cv : 0.0;
    const double e = y - x[NX - 1] / m.p.V;
    double PC[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < NX; ++k) s += P[k * NX + i] * C[k];
        PC[i] = 1.0 * s + 0.0;
    }
    double Re;
    {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < NX; ++k) s += C[k] * PC[k];
        Re = 1.0 * s + 1.0 * R;
    }
    if (Re <= 0.0 || !dfinite(Re)) return true;
    const double l = sqrt(Re);
    double K[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) {
        double t = PC[i] / l;
        K[i] = t / l;
    }
#pragma unroll
    for (int i = 0; i < NX; ++i) x[i] = 1.0 * (0.0 + K[i] * e) + 1.0 * x[i];
    double IKC[NX * NX];
#pragma unroll
    for (int j = 0; j < NX; ++j)
#pragma unroll
        for (int i = 0; i < NX; ++i) IKC[j * NX + i] = -1.0 * (0.0 + K[i] * C[j]) + 1.0 * ((i == j) ? 1.0 : 0.0);
    double T[NX * NX], Pn[NX * NX];
#pragma unroll
    for (int j = 0; j < NX; ++j)
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < NX; ++k) s += IKC[k * NX + i] * P[j * NX + k];
            T[j * NX + i] = 1.0 * s + 0.0;
        }
#pragma unroll
    for (int j = 0; j < NX; ++j)
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < NX; ++k) s += T[k * NX + i] * IKC[k * NX + j];
            Pn[j * NX + i] = 1.0 * s + 0.0;
        }
    double KR[NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) KR[i] = 1.0 * (0.0 + K[i] * R) + 0.0;
#pragma unroll
    for (int j = 0; j < NX; ++j)
#pragma unroll
        for (int i = 0; i < NX; ++i) Pn[j * NX + i] = 1.0 * (0.0 + KR[i] * K[j]) + 1.0 * Pn[j * NX + i];
#pragma unroll
    for (int j = 0; j < NX; ++j)
#pragma unroll
        for (int i = j + 1; i < NX; ++i) {
            const double mm = 0.5 * (Pn[j * NX + i] + Pn[i * NX + j]);
            Pn[j * NX + i] = mm;
            Pn[i * NX + j] = mm;
        }
#pragma unroll
    for (int e2 = 0; e2 < NX * NX; ++e2) P[e2] = Pn[e2];
    return false;
}

/// Result of one nmpc_step (nmpc_step_ws).
struct StepRes {
    int status;       // G_OK or the status of the exception that escaped
    bool filter_npd;  // NotPositiveDefinite from filter_update after the jitter retry
    bool converged;
    bool adopted;     // last_xi / last_duals replaced by this step's solution
    double u;
};

/// nmpc_step (controllers.cpp:114-212) on the carried NmpcState: the filter
/// prediction (xhat, Pf), the previous solution in LXI / LLAM / LPL / LPU when
/// have_last, the stage setpoints already in SP. Returns the clamped first
/// input; xf / Pn receive the posterior (NmpcDiagnostics::filtered). State
/// transitions follow the reference under exceptions: a throw before
/// sqp_solve returns leaves the state untouched; once it has returned,
/// last_xi / last_duals are adopted, and a throw from predict leaves only the
/// filter at its old value.
template <int NX, int W>
__device__ __forceinline__ StepRes nmpc_step_ws(Ocp<NX, W>& o, const nmpcmc_scenario& sc, double t, double y,
                                                double* xhat, double* Pf, bool& have_last, double* xf, double* Pn) {
    StepRes r{G_OK, false, false, false, 0.0};
    const WsT<W> ws = o.ws;
    const Layout<NX> L = o.lay;
    const int N = o.N;
    const int lane = Lanes<W>::lane();
    const bool fl = dfinite(o.umin), fh = dfinite(o.umax);
    auto clampu = [&](double u) { return smax(o.umin, smin(o.umax, u)); };
#pragma unroll
    for (int e = 0; e < NX; ++e) xf[e] = xhat[e];
#pragma unroll
    for (int e = 0; e < NX * NX; ++e) Pn[e] = Pf[e];
    if (ekf_update<NX>(o.m, xf, Pn, y, sc.R_filter)) {  // jitter retry (controllers.cpp:123-132)
#pragma unroll
        for (int e = 0; e < NX; ++e) xf[e] = xhat[e];
#pragma unroll
        for (int e = 0; e < NX * NX; ++e) Pn[e] = Pf[e];
        if (ekf_update<NX>(o.m, xf, Pn, y, sc.R_filter + 1e-10)) {
            r.status = G_NPD;
            r.filter_npd = true;
            return r;
        }
    }
#pragma unroll
    for (int e = 0; e < NX; ++e) o.x0[e] = xf[e];
    // warm / cold start (controllers.cpp:147-186)
    if (have_last) {
#pragma unroll 1
        for (int k = lane; k < N; k += W) ws[L.US + k] = clampu(ws[L.LXI + L.uo(k + 1 < N ? k + 1 : N - 1)]);
        Lanes<W>::sync();
        const int st = xi_from_u<NX, W>(o, 0);
        if (st == G_DOMAIN) {
            r.status = G_DOMAIN;
            return r;
        }
        if (st != G_OK) {  // shifted_warm_start (controllers.cpp:97-110), clamped inputs
            const int w = Layout<NX>::W;
            for (int e = lane; e < L.L; e += W) {
                double x = e < L.L - w ? ws[L.LXI + e + w] : ws[L.LXI + e];
                if (e % w == 0) x = clampu(x);
                ws[L.XI[0] + e] = x;
            }
        }
        // shifted_multipliers (controllers.cpp:87-93), projected (sqp.cpp:219-222)
        for (int e = lane; e < L.NN; e += W)
            ws[L.LAM + e] = (L.NN >= 2 * NX && e < L.NN - NX) ? ws[L.LLAM + e + NX] : ws[L.LLAM + e];
#pragma unroll 1
        for (int k = lane; k < N; k += W) {
            const int src = k < N - 1 ? k + 1 : k;
            ws[L.PL + k] = smax(0.0, ws[L.LPL + src]);
            ws[L.PU + k] = smax(0.0, ws[L.LPU + src]);
        }
    } else {
        const double un = fl && fh ? 0.5 * (o.umin + o.umax) : clampu(0.0);
#pragma unroll 1
        for (int k = lane; k < N; k += W) ws[L.US + k] = un;
        Lanes<W>::sync();
        const int st = xi_from_u<NX, W>(o, 0);
        if (st == G_DOMAIN) {
            r.status = G_DOMAIN;
            return r;
        }
        if (st != G_OK) {
#pragma unroll 1
            for (int k = lane; k < N; k += W) {
                ws[L.XI[0] + L.uo(k)] = un;
#pragma unroll
                for (int e = 0; e < NX; ++e) ws[L.XI[0] + L.xo(k + 1) + e] = xf[e];
            }
        }
        for (int e = lane; e < L.NN; e += W) ws[L.LAM + e] = 0.0;
#pragma unroll 1
        for (int k = lane; k < N; k += W) ws[L.PL + k] = 0.0, ws[L.PU + k] = 0.0;
    }
    Lanes<W>::sync();
    int cur = 0;
    const SqpOut so = sqp_solve<NX, W>(o, sc.sqp, &cur);
    if (so.status != G_OK) {
        r.status = so.status;
        return r;
    }
    const double u = clampu(ws[L.XI[cur] + L.uo(0)]);
    for (int e = lane; e < L.L; e += W) ws[L.LXI + e] = ws[L.XI[cur] + e];
    for (int e = lane; e < L.NN; e += W) ws[L.LLAM + e] = ws[L.LAM + e];
#pragma unroll 1
    for (int k = lane; k < N; k += W) ws[L.LPL + k] = ws[L.PL + k], ws[L.LPU + k] = ws[L.PU + k];
    Lanes<W>::sync();
    have_last = true;
    r.adopted = true;
    r.converged = so.converged;
    double xp[NX], Pp[NX * NX];
#pragma unroll
    for (int e = 0; e < NX; ++e) xp[e] = xf[e];
#pragma unroll
    for (int e = 0; e < NX * NX; ++e) Pp[e] = Pn[e];
    {
        const int st = ekf_predict<NX>(o.m, xp, Pp, u, t, t + sc.horizon_Ts, sc.np);
        if (st != G_OK) {
            r.status = st;
            return r;
        }
    }
#pragma unroll
    for (int e = 0; e < NX; ++e) xhat[e] = xp[e];
#pragma unroll
    for (int e = 0; e < NX * NX; ++e) Pf[e] = Pp[e];
    r.u = u;
    r.converged = so.converged;
    return r;
}

// ------------------------------------------------------------ closed loop
/// The NMPC branch of run_closed_loop (montecarlo.cpp:80-157) for one sample
/// with a controller model of NX states and a truth plant of TX states.
template <int TX, int NX, int W>
__device__ __noinline__ void closed_loop(const nmpcmc_scenario& sc, uint64_t sim_index, int nbar, const WsT<W>& ws,
                                         nmpcmc_sim_record* rec, nmpcmc_work_counters* cntp, double* traj,
                                         int fd = 0) {
    const Cstr p = sample_truth(sc, sim_index);
    NormalStream rng;
    rng.init(sc.base_seed, sim_index);
    Plant<TX> pl;
#pragma unroll
    for (int i = 0; i < TX; ++i) pl.x[i] = sc.x0[i];
    const bool has_R = sc.has_noise_R != 0;
    const double lR = has_R ? chol_semidef_1x1(sc.noise_R) : 0.0;
    const int stride = sc.record_stride < 1 ? 1 : sc.record_stride;
    Cnt cnt = {};
    const int lane = Lanes<W>::lane();
    Ocp<NX, W> o{make_model<NX>(sc.ctrl), Layout<NX>(sc.N), ws, sc.N, sc.Nc, sc.horizon_Ts, sc.horizon_Ts / sc.Nc,
              sc.u_min, sc.u_max, sc.Qz, 0.0, {}, &cnt};
    o.invV = 1.0 / o.m.p.V;
    o.m.fd = fd;
    const Layout<NX> L = o.lay;
    const int N = o.N;
    // make_nmpc_state (controllers.cpp:25-48)
    double xhat[NX], Pf[NX * NX];
#pragma unroll
    for (int i = 0; i < NX; ++i) xhat[i] = sc.x0_hat[i];
#pragma unroll
    for (int e = 0; e < NX * NX; ++e) Pf[e] = sc.P0[e];
    bool have_last = false;
    double t = sc.t0;
    double z = pl.x[TX - 1] / p.V, zbar = setpoint_at(sc, t);
    double acc = 0.0;
    {
        const double r = z - zbar;
        acc += r * r;
    }
    int status = G_OK, solves = 0, fails = 0, row = 0;
    bool counts_lost = false;
#pragma unroll 1
    for (int i = 0; i < nbar; ++i) {
        const double y = measure<TX>(p, pl, has_R, lR, rng);
        // ---- nmpc_step (controllers.cpp:114-212)
        if (!dfinite(y)) {
            status = G_NONFINITE;
            break;
        }
#pragma unroll 1
        for (int k = lane; k < N; k += W) ws[L.SP + k] = setpoint_at(sc, t + (k + 1) * sc.Ts);
        Lanes<W>::sync();
        double xf[NX], Pn[NX * NX];
        const StepRes sr = nmpc_step_ws<NX, W>(o, sc, t, y, xhat, Pf, have_last, xf, Pn);
        if (sr.status != G_OK) {
            status = sr.status;
            counts_lost = sr.filter_npd;
            break;
        }
        const double u = sr.u;
        ++solves;
        if (!sr.converged) ++fails;
        cnt.steps += 1;
        if (traj != nullptr && i % stride == 0) {
            if (lane == 0) {
                double* rw = traj + (size_t)row * 5;
                rw[0] = t, rw[1] = z, rw[2] = zbar, rw[3] = u, rw[4] = y;
            }
            ++row;
        }
        status = simulate_interval<TX>(p, pl, t, t + sc.Ts, u, sc.Ns, rng);
        if (status != G_OK) break;
        t = sc.t0 + (i + 1) * sc.Ts;
        z = pl.x[TX - 1] / p.V;
        zbar = setpoint_at(sc, t);
        const double r = z - zbar;
        acc += r * r;
    }
    if (lane != 0) return;
    if (status == G_OK) {
        rec->phi = acc / (double)(nbar + 1);
        rec->failed = 0;
        if (traj != nullptr) {
            double* rw = traj + (size_t)row * 5;
            rw[0] = t, rw[1] = z, rw[2] = zbar;
        }
    } else {
        rec->phi = kNaN;
        rec->failed = 1;
    }
    rec->ocp_solves = counts_lost ? 0 : solves;
    rec->ocp_failures = counts_lost ? 0 : fails;
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

constexpr int kGenBlock = 64;

/// One thread per sample; threads pull sample indices from an atomic counter
/// (run_monte_carlo's worker pool, montecarlo.cpp:218-238). Slot t of the
/// workspace belongs to global thread t.
template <int TX, int NX>
__global__ void __launch_bounds__(kGenBlock) nmpc_gen_kernel(const __grid_constant__ nmpcmc_scenario sc,
                                                             uint64_t first_sim, int64_t n_sims, int nbar,
                                                             nmpcmc_sim_record* records,
                                                             nmpcmc_work_counters* counters, double* traj,
                                                             int traj_rows, double* ws_all, int64_t slots,
                                                             unsigned long long* next) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= slots) return;
    const Ws ws{ws_all + tid, slots};
#pragma unroll 1
    for (;;) {
        const unsigned long long i = atomicAdd(next, 1ULL);
        if (i >= (unsigned long long)n_sims) break;
        closed_loop<TX, NX, 1>(sc, first_sim + i, nbar, ws, records + i, counters ? counters + i : nullptr,
                               traj ? traj + (size_t)i * traj_rows * 5 : nullptr);
    }
}

/// K3w: one warp per sample, persistent one-warp blocks pulling samples from
/// an atomic counter; workspace = one contiguous slab per block.
template <int TX, int NX>
#ifdef NMPCMC_K3W_MAXNREG
__global__ void __maxnreg__(NMPCMC_K3W_MAXNREG) nmpc_genw_kernel(
#else
__global__ void __launch_bounds__(32, NMPCMC_K3W_MIN_BLOCKS) nmpc_genw_kernel(
#endif
const __grid_constant__ nmpcmc_scenario sc, uint64_t first_sim,
                                                       int64_t n_sims, int nbar, nmpcmc_sim_record* records,
                                                       nmpcmc_work_counters* counters, double* traj, int traj_rows,
                                                       double* ws_all, int64_t slab, unsigned long long* next,
                                                       int fd) {
    const WsT<32> ws{ws_all + (int64_t)blockIdx.x * slab, 1};
#pragma unroll 1
    for (;;) {
        unsigned long long i = 0;
        if ((threadIdx.x & 31) == 0) i = atomicAdd(next, 1ULL);
        i = __shfl_sync(kMask, i, 0);
        if (i >= (unsigned long long)n_sims) break;
        closed_loop<TX, NX, 32>(sc, first_sim + i, nbar, ws, records + i, counters ? counters + i : nullptr,
                                traj ? traj + (size_t)i * traj_rows * 5 : nullptr, fd);
    }
}

/// Batched OCP service (nmpcmc_gpu_solve_ocp_batch): sqp_solve on the
/// regulator OcpProblem of the controller model for each (x0[b], t0[b]), cold
/// start as nmpc_step (controllers.cpp:166-185) or the given xi0 with zero
/// duals. One warp per instance (K3w's code path).
template <int NX>
__global__ void __launch_bounds__(32) ocp_batch_kernel(const __grid_constant__ nmpcmc_scenario sc, int64_t batch,
                                                       const double* x0, const double* t0, const double* xi0,
                                                       double* xi_out, double* lam_out, double* pil_out,
                                                       double* piu_out, int32_t* converged, int32_t* status,
                                                       double* ws_all, int64_t slab, unsigned long long* next,
                                                       int32_t* iters_out, int max_trace,
                                                       nmpcmc_sqp_iter_log* trace, int32_t* trace_len) {
    const WsT<32> ws{ws_all + (int64_t)blockIdx.x * slab, 1};
    const int lane = Lanes<32>::lane();
#pragma unroll 1
    for (;;) {
        unsigned long long bi = 0;
        if (lane == 0) bi = atomicAdd(next, 1ULL);
        bi = __shfl_sync(kMask, bi, 0);
        if (bi >= (unsigned long long)batch) break;
        const int64_t b = (int64_t)bi;
        Cnt cnt = {};
        Ocp<NX, 32> o{make_model<NX>(sc.ctrl), Layout<NX>(sc.N), ws, sc.N, sc.Nc, sc.horizon_Ts,
                      sc.horizon_Ts / sc.Nc, sc.u_min, sc.u_max, sc.Qz, 0.0, {}, &cnt};
        o.invV = 1.0 / o.m.p.V;
        const Layout<NX> L = o.lay;
        const int N = o.N;
#pragma unroll
        for (int i = 0; i < NX; ++i) o.x0[i] = x0[b * NX + i];
        if (trace != nullptr) {
            o.trace = trace + b * max_trace;
            o.trace_cap = max_trace;
            o.trace_len = trace_len + b;
            if (lane == 0) trace_len[b] = 0;
        }
        for (int k = lane; k < N; k += 32) ws[L.SP + k] = setpoint_at(sc, t0[b] + (k + 1) * sc.Ts);
        int st = G_OK;
        if (xi0 != nullptr) {
            for (int e = lane; e < L.L; e += 32) ws[L.XI[0] + e] = xi0[b * L.L + e];
        } else {
            const bool fl = dfinite(o.umin), fh = dfinite(o.umax);
            const double un = fl && fh ? 0.5 * (o.umin + o.umax) : smax(o.umin, smin(o.umax, 0.0));
            for (int k = lane; k < N; k += 32) ws[L.US + k] = un;
            Lanes<32>::sync();
            st = xi_from_u<NX, 32>(o, 0);
            if (st != G_OK && st != G_DOMAIN) {  // NonFiniteState: flat guess
                for (int k = lane; k < N; k += 32) {
                    ws[L.XI[0] + L.uo(k)] = un;
#pragma unroll
                    for (int e = 0; e < NX; ++e) ws[L.XI[0] + L.xo(k + 1) + e] = o.x0[e];
                }
                st = G_OK;
            }
        }
        for (int e = lane; e < L.NN; e += 32) ws[L.LAM + e] = 0.0;
        for (int k = lane; k < N; k += 32) ws[L.PL + k] = 0.0, ws[L.PU + k] = 0.0;
        Lanes<32>::sync();
        int cur = 0;
        SqpOut so{false, st};
        if (st == G_OK) so = sqp_solve<NX, 32>(o, sc.sqp, &cur);
        const bool ok = so.status == G_OK;
        for (int e = lane; e < L.L; e += 32) xi_out[b * L.L + e] = ok ? (double)ws[L.XI[cur] + e] : 0.0;
        for (int e = lane; e < L.NN; e += 32) lam_out[b * L.NN + e] = ok ? (double)ws[L.LAM + e] : 0.0;
        for (int k = lane; k < N; k += 32) {
            pil_out[b * N + k] = ok ? (double)ws[L.PL + k] : 0.0;
            piu_out[b * N + k] = ok ? (double)ws[L.PU + k] : 0.0;
        }
        if (lane == 0) {
            converged[b] = ok && so.converged ? 1 : 0;
            status[b] = ok ? 0 : so.status;
            if (iters_out != nullptr) iters_out[b] = (int32_t)cnt.sqp;
        }
        Lanes<32>::sync();
    }
}

inline int launch_ocp_batch(const nmpcmc_scenario& sc, int64_t batch, const double* x0, const double* t0,
                            const double* xi0, double* xi, double* lam, double* pil, double* piu, int32_t* conv,
                            int32_t* status, double* ws, int64_t blocks, unsigned long long* counter,
                            cudaStream_t stream, int32_t* iters = nullptr, int max_trace = 0,
                            nmpcmc_sqp_iter_log* trace = nullptr, int32_t* trace_len = nullptr) {
    const bool c3 = sc.ctrl_variant == NMPCMC_THREE_STATE;
    const int64_t slab = c3 ? Layout<3>(sc.N).total : Layout<1>(sc.N).total;
    const size_t smem = c3 ? sweep_smem_bytes<3>(sc.N) : sweep_smem_bytes<1>(sc.N);
    if (smem > kSweepSmemMax) return NMPCMC_UNSUPPORTED;
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
    if (c3)
        ocp_batch_kernel<3><<<(unsigned)blocks, 32, smem, stream>>>(sc, batch, x0, t0, xi0, xi, lam, pil, piu, conv,
                                                                    status, ws, slab, counter, iters, max_trace,
                                                                    trace, trace_len);
    else
        ocp_batch_kernel<1><<<(unsigned)blocks, 32, smem, stream>>>(sc, batch, x0, t0, xi0, xi, lam, pil, piu, conv,
                                                                    status, ws, slab, counter, iters, max_trace,
                                                                    trace, trace_len);
    return NMPCMC_OK;
}


/// Batched sqp_solve (sqp.cpp:182-411) on stagewise quadratic NLPs (Qnlp):
/// instance b's data at prob + b * stride = x0[NX] u_min u_max, then N
/// stages of Qnlp<NX>::kStage doubles; start xi0[b*L ..] (null: zeros) with
/// zero duals and identity Hessian blocks, as sqp_solve without a warm start.
/// One warp per instance (K3w's code path; only objective() / constraints()
/// differ from the regulator OCP).
template <int NX>
__global__ void __launch_bounds__(32) qnlp_batch_kernel(int N, nmpcmc_sqp_options opt, int64_t batch,
                                                        const double* prob, int64_t stride, const double* xi0,
                                                        double* xi_out, double* lam_out, double* pil_out,
                                                        double* piu_out, int32_t* converged, int32_t* iters,
                                                        int32_t* status, double* ws_all, int64_t slab,
                                                        unsigned long long* next) {
    const WsT<32> ws{ws_all + (int64_t)blockIdx.x * slab, 1};
    const int lane = Lanes<32>::lane();
#pragma unroll 1
    for (;;) {
        unsigned long long bi = 0;
        if (lane == 0) bi = atomicAdd(next, 1ULL);
        bi = __shfl_sync(kMask, bi, 0);
        if (bi >= (unsigned long long)batch) break;
        const int64_t b = (int64_t)bi;
        const double* P = prob + b * stride;
        Cnt cnt = {};
        Ocp<NX, 32> o{Model<NX>{}, Layout<NX>(N), ws, N, 1, 0.0, 0.0, __ldg(P + NX), __ldg(P + NX + 1), 0.0, 0.0,
                      {}, &cnt, P + NX + 2};
#pragma unroll
        for (int i = 0; i < NX; ++i) o.x0[i] = __ldg(P + i);
        const Layout<NX> L = o.lay;
        for (int e = lane; e < L.L; e += 32) ws[L.XI[0] + e] = xi0 != nullptr ? xi0[b * L.L + e] : 0.0;
        for (int e = lane; e < L.NN; e += 32) ws[L.LAM + e] = 0.0;
        for (int k = lane; k < N; k += 32) ws[L.PL + k] = 0.0, ws[L.PU + k] = 0.0;
        Lanes<32>::sync();
        int cur = 0;
        const SqpOut so = sqp_solve<NX, 32>(o, opt, &cur);
        const bool ok = so.status == G_OK;
        for (int e = lane; e < L.L; e += 32) xi_out[b * L.L + e] = ok ? (double)ws[L.XI[cur] + e] : 0.0;
        for (int e = lane; e < L.NN; e += 32) lam_out[b * L.NN + e] = ok ? (double)ws[L.LAM + e] : 0.0;
        for (int k = lane; k < N; k += 32) {
            pil_out[b * N + k] = ok ? (double)ws[L.PL + k] : 0.0;
            piu_out[b * N + k] = ok ? (double)ws[L.PU + k] : 0.0;
        }
        if (lane == 0) {
            converged[b] = ok && so.converged ? 1 : 0;
            iters[b] = (int32_t)cnt.sqp;
            status[b] = ok ? 0 : so.status;
        }
        Lanes<32>::sync();
    }
}

inline int64_t qnlp_stride(int N, int nx) {
    return nx == 3 ? 3 + 2 + (int64_t)N * Qnlp<3>::kStage : 1 + 2 + (int64_t)N * Qnlp<1>::kStage;
}

inline int64_t qnlp_ws_doubles(int N, int nx) { return nx == 3 ? Layout<3>(N).total : Layout<1>(N).total; }

inline int launch_qnlp_batch(int N, int nx, const nmpcmc_sqp_options& opt, int64_t batch, const double* prob,
                             const double* xi0, double* xi, double* lam, double* pil, double* piu, int32_t* conv,
                             int32_t* iters, int32_t* status, double* ws, int64_t blocks, unsigned long long* counter,
                             cudaStream_t stream) {
    const size_t smem = nx == 3 ? sweep_smem_bytes<3>(N) : sweep_smem_bytes<1>(N);
    if (smem > kSweepSmemMax || blocks < 1) return NMPCMC_UNSUPPORTED;
    const int64_t slab = qnlp_ws_doubles(N, nx), stride = qnlp_stride(N, nx);
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
    if (nx == 3) {
        cudaFuncSetAttribute(qnlp_batch_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        qnlp_batch_kernel<3><<<(unsigned)blocks, 32, smem, stream>>>(N, opt, batch, prob, stride, xi0, xi, lam, pil,
                                                                     piu, conv, iters, status, ws, slab, counter);
    } else {
        cudaFuncSetAttribute(qnlp_batch_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        qnlp_batch_kernel<1><<<(unsigned)blocks, 32, smem, stream>>>(N, opt, batch, prob, stride, xi0, xi, lam, pil,
                                                                     piu, conv, iters, status, ws, slab, counter);
    }
    return NMPCMC_OK;
}

/// Layout of one device-resident NmpcState (controllers.hpp:54-65) of the
/// batched controller API (nmpcmc_gpu_nmpc_step_batch): the filter
/// prediction (x_hat, P), the warm flag (last_xi non-empty) and the previous
/// solution in the reference's orders: xi = (u_0, x_1, ..., u_{N-1}, x_N),
/// lambda stage-ordered, pi_l, pi_u.
template <int NX>
struct StateLay {
    int XH, P, WARM, XI, LAM, PL, PU, total;
    __host__ __device__ explicit StateLay(int N)
        : XH(0), P(NX), WARM(NX + NX * NX), XI(WARM + 1), LAM(XI + N * (1 + NX)), PL(LAM + N * NX), PU(PL + N),
          total(PU + N) {}
};

/// Batched nmpc_step (controllers.cpp:114-212): one warp per controller
/// instance b, on K3w's code path. The instance's NmpcState lives in
/// states[b * stride ..] (StateLay) and is updated in place with the
/// reference's transitions under exceptions (nmpc_step_ws). setpoints:
/// sp[b * N + k] for stage k+1, or the scenario's profile at t + (k+1) Ts
/// when sp is null (as run_closed_loop passes them).
template <int NX>
__global__ void __launch_bounds__(32) nmpc_step_kernel(const __grid_constant__ nmpcmc_scenario sc, int64_t batch,
                                                       double* states, const double* t, const double* y,
                                                       const double* sp, double* u_out, nmpcmc_nmpc_diag* diag,
                                                       double* ws_all, int64_t slab, unsigned long long* next) {
    const WsT<32> ws{ws_all + (int64_t)blockIdx.x * slab, 1};
    const int lane = Lanes<32>::lane();
    const StateLay<NX> SL(sc.N);
#pragma unroll 1
    for (;;) {
        unsigned long long bi = 0;
        if (lane == 0) bi = atomicAdd(next, 1ULL);
        bi = __shfl_sync(kMask, bi, 0);
        if (bi >= (unsigned long long)batch) break;
        const int64_t b = (int64_t)bi;
        Cnt cnt = {};
        Ocp<NX, 32> o{make_model<NX>(sc.ctrl), Layout<NX>(sc.N), ws, sc.N, sc.Nc, sc.horizon_Ts,
                      sc.horizon_Ts / sc.Nc, sc.u_min, sc.u_max, sc.Qz, 0.0, {}, &cnt};
        o.invV = 1.0 / o.m.p.V;
        const Layout<NX> L = o.lay;
        const int N = o.N;
        double* S = states + b * SL.total;
        double xhat[NX], Pf[NX * NX], xf[NX], Pn[NX * NX];
#pragma unroll
        for (int i = 0; i < NX; ++i) xhat[i] = S[SL.XH + i], xf[i] = kNaN;
#pragma unroll
        for (int e = 0; e < NX * NX; ++e) Pf[e] = S[SL.P + e], Pn[e] = kNaN;
        const bool warm = S[SL.WARM] != 0.0;
        bool have_last = warm;
        const double tb = t[b], yb = y[b];
        const double innov = yb - xhat[NX - 1] / o.m.p.V;  // filter_update's e (ekf.cpp:66)
        StepRes sr{G_OK, false, false, false, kNaN};
        if (!dfinite(yb)) {
            sr.status = G_NONFINITE;  // nmpc_step: measurement is not finite
        } else {
            if (warm) {
                for (int e = lane; e < L.L; e += 32) ws[L.LXI + e] = S[SL.XI + e];
                for (int e = lane; e < L.NN; e += 32) ws[L.LLAM + e] = S[SL.LAM + e];
                for (int k = lane; k < N; k += 32) ws[L.LPL + k] = S[SL.PL + k], ws[L.LPU + k] = S[SL.PU + k];
            }
            for (int k = lane; k < N; k += 32)
                ws[L.SP + k] = sp != nullptr ? sp[b * N + k] : setpoint_at(sc, tb + (k + 1) * sc.Ts);
            Lanes<32>::sync();
            sr = nmpc_step_ws<NX, 32>(o, sc, tb, yb, xhat, Pf, have_last, xf, Pn);
        }
        if (sr.adopted) {
            for (int e = lane; e < L.L; e += 32) S[SL.XI + e] = ws[L.LXI + e];
            for (int e = lane; e < L.NN; e += 32) S[SL.LAM + e] = ws[L.LLAM + e];
            for (int k = lane; k < N; k += 32) S[SL.PL + k] = ws[L.LPL + k], S[SL.PU + k] = ws[L.LPU + k];
        }
        if (lane == 0) {
            if (sr.adopted) S[SL.WARM] = 1.0;
            if (sr.status == G_OK) {
#pragma unroll
                for (int i = 0; i < NX; ++i) S[SL.XH + i] = xhat[i];
#pragma unroll
                for (int e = 0; e < NX * NX; ++e) S[SL.P + e] = Pf[e];
            }
            u_out[b] = sr.status == G_OK ? sr.u : kNaN;
            if (diag != nullptr) {
                nmpcmc_nmpc_diag d;
                for (int i = 0; i < 3; ++i) d.x_filtered[i] = i < NX ? xf[i] : 0.0;
                for (int e = 0; e < 9; ++e) d.P_filtered[e] = e < NX * NX ? Pn[e] : 0.0;
                d.innovation = dfinite(yb) ? innov : kNaN;
                d.converged = sr.converged ? 1 : 0;
                d.sqp_iterations = (int32_t)cnt.sqp;
                d.warm_started = warm ? 1 : 0;
                d.status = sr.status;
                diag[b] = d;
            }
        }
        Lanes<32>::sync();
    }
}

/// Doubles of one device-resident NmpcState (StateLay) for this scenario.
inline int64_t nmpc_state_doubles(const nmpcmc_scenario& sc) {
    return sc.ctrl_variant == NMPCMC_THREE_STATE ? StateLay<3>(sc.N).total : StateLay<1>(sc.N).total;
}

inline int launch_nmpc_step(const nmpcmc_scenario& sc, int64_t batch, double* states, const double* t,
                            const double* y, const double* sp, double* u, nmpcmc_nmpc_diag* diag, double* ws,
                            int64_t blocks, unsigned long long* counter, cudaStream_t stream) {
    const bool c3 = sc.ctrl_variant == NMPCMC_THREE_STATE;
    const int64_t slab = c3 ? Layout<3>(sc.N).total : Layout<1>(sc.N).total;
    const size_t smem = c3 ? sweep_smem_bytes<3>(sc.N) : sweep_smem_bytes<1>(sc.N);
    if (smem > kSweepSmemMax || blocks < 1) return NMPCMC_UNSUPPORTED;
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
    if (c3) {
        cudaFuncSetAttribute(nmpc_step_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        nmpc_step_kernel<3><<<(unsigned)blocks, 32, smem, stream>>>(sc, batch, states, t, y, sp, u, diag, ws, slab,
                                                                    counter);
    } else {
        cudaFuncSetAttribute(nmpc_step_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        nmpc_step_kernel<1><<<(unsigned)blocks, 32, smem, stream>>>(sc, batch, states, t, y, sp, u, diag, ws, slab,
                                                                    counter);
    }
    return NMPCMC_OK;
}

/// Doubles of workspace per slot.
inline int64_t gen_ws_doubles(const nmpcmc_scenario& sc) {
    return sc.ctrl_variant == NMPCMC_THREE_STATE ? Layout<3>(sc.N).total : Layout<1>(sc.N).total;
}

/// Resident slots: SMs x resident 64-thread blocks, at most n.
template <int TX, int NX>
inline int64_t gen_slots_t(int sm_count, int64_t n) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, nmpc_gen_kernel<TX, NX>, kGenBlock, 0);
    if (b < 1) b = 1;
    int64_t slots = (int64_t)sm_count * b * kGenBlock;
    return slots < n ? slots : n;
}
inline int64_t gen_slots(const nmpcmc_scenario& sc, int sm_count, int64_t n) {
    const bool t3 = sc.truth_variant == NMPCMC_THREE_STATE, c3 = sc.ctrl_variant == NMPCMC_THREE_STATE;
    if (t3) return c3 ? gen_slots_t<3, 3>(sm_count, n) : gen_slots_t<3, 1>(sm_count, n);
    return c3 ? gen_slots_t<1, 3>(sm_count, n) : gen_slots_t<1, 1>(sm_count, n);
}

/// K3w resident blocks (one warp each): occupancy, capped so the per-warp
/// slabs stay L2-resident (~72 KB each at N = 60, NX = 3).
template <int TX, int NX>
inline int64_t genw_blocks_t(int sm_count, int64_t n, int64_t slab_doubles, int N) {
    const size_t smem = sweep_smem_bytes<NX>(N);
    cudaFuncSetAttribute(nmpc_genw_kernel<TX, NX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(ocp_batch_kernel<NX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, nmpc_genw_kernel<TX, NX>, 32, smem);
    if (b < 1) b = 1;
    int64_t blocks = (int64_t)sm_count * b;
#ifndef NMPCMC_K3W_L2_CAP_MB
#define NMPCMC_K3W_L2_CAP_MB 96
#endif
    const int64_t l2_cap = (int64_t)((unsigned long long)NMPCMC_K3W_L2_CAP_MB << 20) / (slab_doubles * 8);
    if (blocks > l2_cap) blocks = l2_cap < sm_count ? sm_count : l2_cap;
    return blocks < n ? blocks : n;
}
inline int64_t genw_blocks(const nmpcmc_scenario& sc, int sm_count, int64_t n) {
    const bool t3 = sc.truth_variant == NMPCMC_THREE_STATE, c3 = sc.ctrl_variant == NMPCMC_THREE_STATE;
    const int64_t slab = gen_ws_doubles(sc);
    if (t3) return c3 ? genw_blocks_t<3, 3>(sm_count, n, slab, sc.N) : genw_blocks_t<3, 1>(sm_count, n, slab, sc.N);
    return c3 ? genw_blocks_t<1, 3>(sm_count, n, slab, sc.N) : genw_blocks_t<1, 1>(sm_count, n, slab, sc.N);
}
/// K3w needs its sweep arrays in shared memory (N up to ~1,000 stages at NX = 3).
inline size_t genw_smem(const nmpcmc_scenario& sc) {
    return sc.ctrl_variant == NMPCMC_THREE_STATE ? sweep_smem_bytes<3>(sc.N) : sweep_smem_bytes<1>(sc.N);
}
inline bool genw_fits(const nmpcmc_scenario& sc) { return genw_smem(sc) <= kSweepSmemMax; }
inline int launch_genw(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
                       nmpcmc_work_counters* d_cnt, double* d_traj, int rows, double* ws, int64_t blocks,
                       unsigned long long* counter, cudaStream_t stream, int fd = 0) {
    if (blocks < 1 || !genw_fits(sc)) return NMPCMC_INVALID_ARGUMENT;
    const int64_t slab = gen_ws_doubles(sc);
    const size_t smem = genw_smem(sc);
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
    const bool t3 = sc.truth_variant == NMPCMC_THREE_STATE, c3 = sc.ctrl_variant == NMPCMC_THREE_STATE;
#define NMPCMC_GENW_LAUNCH(T, C)                                                                              \
    nmpc_genw_kernel<T, C><<<(unsigned)blocks, 32, smem, stream>>>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, ws, \
                                                                slab, counter, fd)
    if (t3 && c3) NMPCMC_GENW_LAUNCH(3, 3);
    else if (t3) NMPCMC_GENW_LAUNCH(3, 1);
    else if (c3) NMPCMC_GENW_LAUNCH(1, 3);
    else NMPCMC_GENW_LAUNCH(1, 1);
#undef NMPCMC_GENW_LAUNCH
    return NMPCMC_OK;
}

inline int launch_gen(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
                      nmpcmc_work_counters* d_cnt, double* d_traj, int rows, double* ws, int64_t slots,
                      unsigned long long* counter, cudaStream_t stream) {
    if (slots < 1) return NMPCMC_INVALID_ARGUMENT;
    const unsigned grid = (unsigned)((slots + kGenBlock - 1) / kGenBlock);
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), stream);
    const bool t3 = sc.truth_variant == NMPCMC_THREE_STATE, c3 = sc.ctrl_variant == NMPCMC_THREE_STATE;
#define NMPCMC_GEN_LAUNCH(T, C) \
    nmpc_gen_kernel<T, C><<<grid, kGenBlock, 0, stream>>>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, ws, slots, counter)
    if (t3 && c3) NMPCMC_GEN_LAUNCH(3, 3);
    else if (t3) NMPCMC_GEN_LAUNCH(3, 1);
    else if (c3) NMPCMC_GEN_LAUNCH(1, 3);
    else NMPCMC_GEN_LAUNCH(1, 1);
#undef NMPCMC_GEN_LAUNCH
    return NMPCMC_OK;
}

}  // namespace gen
}  // namespace nmpcmc_dev
