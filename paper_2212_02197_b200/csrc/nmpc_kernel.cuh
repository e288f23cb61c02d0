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
// Execution model:
//  * one warp = one sample; the whole per-sample workspace (~51 arrays of
//    N+1 doubles: the iterate, multipliers, defect jacobians, BFGS blocks and
//    the Riccati IPM state) lives in shared memory, so the inner loops never
//    touch HBM;
//  * stage-parallel work (the N independent shooting intervals, residuals,
//    expand / step-length / update loops, BFGS blocks) is spread over the 32
//    lanes, k = lane, lane+32, ...;
//  * the inherently serial recursions (Riccati sweeps, ordered reductions,
//    xi_from_inputs, EKF, plant) are executed redundantly by all 32 lanes in
//    lockstep -- SIMT issues them once, no divergence, no broadcasts;
//  * exceptions become per-sample status codes with the reference's catch
//    scopes.
#pragma once

#include "device_common.cuh"

namespace nmpcmc_dev {

constexpr unsigned FULLMASK = 0xffffffffu;
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
__device__ __forceinline__ int warp_min_int(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(FULLMASK, v, o));
    return v;
}
__device__ __forceinline__ bool warp_any(bool p) { return __any_sync(FULLMASK, p); }

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
    for (int step = 0; step < nc; ++step) {
        Stage1 s1, s2, s3, s4;
        int st = eval1(p, F, u, s1, WITH_SENS);
        if (st) return st;
        double kx1 = 0, ku1 = 0, kx2 = 0, ku2 = 0, kx3 = 0, ku3 = 0, kx4 = 0, ku4 = 0;
        if (WITH_SENS) {
            kx1 = epi0(dot1(s1.a, Sx));
            ku1 = epi1(dot1(s1.a, Su), s1.b);
        }
        st = eval1(p, F + h2 * s1.k, u, s2, WITH_SENS);
        if (st) return st;
        if (WITH_SENS) {
            kx2 = epi0(dot1(s2.a, Sx + h2 * kx1));
            ku2 = epi1(dot1(s2.a, Su + h2 * ku1), s2.b);
        }
        st = eval1(p, F + h2 * s2.k, u, s3, WITH_SENS);
        if (st) return st;
        if (WITH_SENS) {
            kx3 = epi0(dot1(s3.a, Sx + h2 * kx2));
            ku3 = epi1(dot1(s3.a, Su + h2 * ku2), s3.b);
        }
        st = eval1(p, F + 1.0 * h * s3.k, u, s4, WITH_SENS);
        if (st) return st;
        if (WITH_SENS) {
            kx4 = epi0(dot1(s4.a, Sx + 1.0 * h * kx3));
            ku4 = epi1(dot1(s4.a, Su + 1.0 * h * ku3), s4.b);
        }
        F += h6 * (s1.k + 2.0 * s2.k + 2.0 * s3.k + s4.k);
        if (WITH_SENS) {
            Sx += h6 * (kx1 + 2.0 * kx2 + 2.0 * kx3 + kx4);
            Su += h6 * (ku1 + 2.0 * ku2 + 2.0 * ku3 + ku4);
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
/// Per-sample shared-memory workspace: kWsArrays arrays of `s` doubles at
/// smem_nmpc + id * s (one warp = one block = one sample). Stage arrays are
/// indexed by k; for the interleaved decision vector
/// xi = (u_0, x_1, ..., u_{N-1}, x_N) (ocp.hpp:37-43) U[k] = u_k and X[k] = x_{k+1}.
/// Index-based access keeps every address in the shared window (LDS/STS).
extern __shared__ __align__(16) double smem_nmpc[];
constexpr int kWsArrays = 51;

struct Ws {
    int s;
    __device__ __forceinline__ double* U(int b) const { return smem_nmpc + (2 * b) * s; }
    __device__ __forceinline__ double* X(int b) const { return smem_nmpc + (2 * b + 1) * s; }
    __device__ __forceinline__ double* lam() const { return smem_nmpc + 4 * s; }
    __device__ __forceinline__ double* pil() const { return smem_nmpc + 5 * s; }
    __device__ __forceinline__ double* piu() const { return smem_nmpc + 6 * s; }
    __device__ __forceinline__ double* gX() const { return smem_nmpc + 7 * s; }
    __device__ __forceinline__ double* g() const { return smem_nmpc + 8 * s; }
    __device__ __forceinline__ double* Jx() const { return smem_nmpc + 9 * s; }
    __device__ __forceinline__ double* Ju() const { return smem_nmpc + 10 * s; }
    __device__ __forceinline__ double* tgX() const { return smem_nmpc + 11 * s; }
    __device__ __forceinline__ double* tg() const { return smem_nmpc + 12 * s; }
    __device__ __forceinline__ double* tJx() const { return smem_nmpc + 13 * s; }
    __device__ __forceinline__ double* tJu() const { return smem_nmpc + 14 * s; }
    __device__ __forceinline__ double* Wq() const { return smem_nmpc + 15 * s; }
    __device__ __forceinline__ double* Wm() const { return smem_nmpc + 16 * s; }
    __device__ __forceinline__ double* Wr() const { return smem_nmpc + 17 * s; }
    __device__ __forceinline__ double* sig() const { return smem_nmpc + 18 * s; }
    __device__ __forceinline__ double* sp() const { return smem_nmpc + 19 * s; }
    __device__ __forceinline__ double* dU() const { return smem_nmpc + 20 * s; }
    __device__ __forceinline__ double* dX() const { return smem_nmpc + 21 * s; }
    __device__ __forceinline__ double* mu() const { return smem_nmpc + 22 * s; }
    __device__ __forceinline__ double* nl() const { return smem_nmpc + 23 * s; }
    __device__ __forceinline__ double* nu() const { return smem_nmpc + 24 * s; }
    __device__ __forceinline__ double* sl() const { return smem_nmpc + 25 * s; }
    __device__ __forceinline__ double* su() const { return smem_nmpc + 26 * s; }
    __device__ __forceinline__ double* rsu() const { return smem_nmpc + 27 * s; }
    __device__ __forceinline__ double* rsx() const { return smem_nmpc + 28 * s; }
    __device__ __forceinline__ double* rdyn() const { return smem_nmpc + 29 * s; }
    __device__ __forceinline__ double* rl() const { return smem_nmpc + 30 * s; }
    __device__ __forceinline__ double* ru() const { return smem_nmpc + 31 * s; }
    __device__ __forceinline__ double* rcl() const { return smem_nmpc + 32 * s; }
    __device__ __forceinline__ double* rcu() const { return smem_nmpc + 33 * s; }
    __device__ __forceinline__ double* dsl() const { return smem_nmpc + 34 * s; }
    __device__ __forceinline__ double* dsu() const { return smem_nmpc + 35 * s; }
    __device__ __forceinline__ double* dnl() const { return smem_nmpc + 36 * s; }
    __device__ __forceinline__ double* dnu() const { return smem_nmpc + 37 * s; }
    __device__ __forceinline__ double* ddU() const { return smem_nmpc + 38 * s; }
    __device__ __forceinline__ double* ddX() const { return smem_nmpc + 39 * s; }
    __device__ __forceinline__ double* ddmu() const { return smem_nmpc + 40 * s; }
    __device__ __forceinline__ double* cholh() const { return smem_nmpc + 41 * s; }
    __device__ __forceinline__ double* gain() const { return smem_nmpc + 42 * s; }
    __device__ __forceinline__ double* gmat() const { return smem_nmpc + 43 * s; }
    __device__ __forceinline__ double* val() const { return smem_nmpc + 44 * s; }
    __device__ __forceinline__ double* pvec() const { return smem_nmpc + 45 * s; }
    __device__ __forceinline__ double* dff() const { return smem_nmpc + 46 * s; }
    __device__ __forceinline__ double* rhat() const { return smem_nmpc + 47 * s; }
    __device__ __forceinline__ double* bar() const { return smem_nmpc + 48 * s; }
    __device__ __forceinline__ double* tmp() const { return smem_nmpc + 49 * s; }
};

__host__ __device__ inline int ws_stride(int N) { return ((N + 1) + 3) & ~3; }
__host__ __device__ inline size_t ws_bytes(int N) { return (size_t)kWsArrays * ws_stride(N) * sizeof(double); }

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
};

/// Work counters accumulated per sample (lane-uniform).
struct Cnt {
    long long steps, shoot_full, shoot_fonly, ipm_stage, sqp_stage, qp, sqp, ls;
};

// ------------------------------------------------------------ OCP evals
/// eval_objective (ocp.cpp:76-99): phi in k order; gradient only on x slots.
/// X holds x_{k+1} at index k; writes gX[k] = d phi / d x_{k+1}.
__device__ __forceinline__ double eval_objective(const Ocp& o, const Ws& w, const double* X, double* gX, int lane) {
    const double ts = o.Ts;
    for (int k = lane; k < o.N; k += 32) {
        const double res = X[k] / o.p.V - w.sp()[k];  // output(x) - zbar
        const double qres = epi0(dot1(o.Qz, res));
        w.tmp()[k] = ts * dot1(res, qres);
        const double gx = epi0(dot1(o.inv_V, qres));
        gX[k] = 0.0 + 2.0 * ts * gx;
    }
    __syncwarp();
    double phi = 0.0;
    for (int k = 0; k < o.N; ++k) phi += w.tmp()[k];
    __syncwarp();
    return phi;
}

/// eval_constraints (ocp.cpp:101-135) + status of the first failing stage in
/// k order (the reference throws at the first failing shoot). Writes
/// g[k] = x_{k+1} - F_k, Jx[k], Ju[k]. Returns 0 or ST_*.
__device__ __forceinline__ int eval_constraints(const Ocp& o, const double* U, const double* X, double* g, double* Jx,
                                double* Ju, int lane, Cnt& cnt) {
    int first_bad = 0x7fffffff;
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
    cnt.shoot_full += o.N;
    first_bad = warp_min_int(first_bad);
    __syncwarp();
    return first_bad == 0x7fffffff ? ST_OK : (first_bad & 15);
}

/// xi_from_inputs (ocp.cpp:137-154): forward shooting from x0 with the
/// inputs already in U; serial in k, executed by all lanes.
__device__ __forceinline__ int xi_from_inputs(const Ocp& o, const double* U, double* X, Cnt& cnt) {
    double xk = o.x0;
    for (int k = 0; k < o.N; ++k) {
        double F, Sx, Su;
        const int st = shoot1<false>(o.p, xk, U[k], o.h, o.Nc, F, Sx, Su);
        cnt.shoot_fonly += 1;
        if (st) {
            __syncwarp();
            return st;
        }
        X[k] = F;
        xk = F;
    }
    __syncwarp();
    return ST_OK;
}

// ------------------------------------------------------------------- QP
/// b_k = F_k - x_{k+1} recovered from g_k = x_{k+1} - F_k: IEEE subtraction is
/// antisymmetric, and an exact-zero defect is +0 either way.
__device__ __forceinline__ double bneg(double g) { return g == 0.0 ? 0.0 : -g; }

/// solve_qp (qp.cpp:173-423) for the stagewise box QP built by
/// build_stages (sqp.cpp:130-171) from W, grad f and the defect blocks:
///   stage k: R = Wr[k], Q = Wq[k], M = Wm[k] (k >= 1), q = gX[k-1], r = 0,
///            Jx = Jx[k], Ju = Ju[k], b = F_k - x_{k+1} = -g[k],
///            lb = umin - u_k, ub = umax - u_k;  terminal Q = Wq[N], q = gX[N-1].
/// Result in dU/dX (step), mu, nl/nu (bound multipliers). Returns the QP
/// status (0 Optimal, 1 MaxIter, 2 Failed) or ST_DOMAIN as -1 (lb > ub).
enum { QP_OPTIMAL = 0, QP_MAXITER = 1, QP_FAILED = 2, QP_DOMAIN = -1 };

__device__ __forceinline__ int solve_qp(const Ocp& o, const Ws& w, const double* U, const double* cgX,
                                        const double* cg, const double* cJx, const double* cJu, double tol,
                                        int max_iter, int lane, Cnt& cnt, int* iters_out) {
    const int N = o.N;
    const double tau = 0.995;
    // data_scale / bounds / init (qp.cpp:183-226)
    double ds = 1.0;
    int nfin = 0;
    bool bad = false;
    for (int k = lane; k < N; k += 32) {
        const double lb = o.umin - U[k];
        const double ub = o.umax - U[k];
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
        ds = smax(ds, fold_absmax(0.0, 0.0));        // inf_norm(r_k), r = 0
        ds = smax(ds, fold_absmax(0.0, bneg(cg[k])));  // inf_norm(b_k)
        ds = smax(ds, fold_absmax(0.0, cgX[k]));     // inf_norm(q_{k+1})
        w.dU()[k] = 0.0;
        w.dX()[k] = 0.0;
        w.mu()[k] = 0.0;
        w.sl()[k] = fl ? smax(1.0, fabs(lb)) : 0.0;
        w.nl()[k] = fl ? 1.0 : 0.0;
        w.su()[k] = fu ? smax(1.0, fabs(ub)) : 0.0;
        w.nu()[k] = fu ? 1.0 : 0.0;
        w.rcl()[k] = 0.0;
        w.rcu()[k] = 0.0;
    }
    if (warp_any(bad)) return QP_DOMAIN;
    ds = warp_max(ds);
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) nfin += __shfl_xor_sync(FULLMASK, nfin, o2);
    const int m = nfin;
    const double eps = tol * ds;
    __syncwarp();

    int status = QP_MAXITER;
    int iter = 0;
    for (;; ++iter) {
        // residuals() (qp.cpp:237-284)
        double ninf = 0.0, dinf = 0.0, linf = 0.0, uinf = 0.0;
        for (int k = lane; k < N; k += 32) {
            const double R = w.Wr()[k], Ju = cJu[k];
            const double vk = w.dU()[k], muk = w.mu()[k];
            double r = epi1(dot1(R, vk), 0.0);
            if (k >= 1) r = epi1(dot1(w.Wm()[k], w.dX()[k - 1]), r);
            r = epim1(dot1(Ju, muk), r);
            r += w.nu()[k] - w.nl()[k];
            w.rsu()[k] = r;
            double rd = w.dX()[k] + -1.0 * bneg(cg[k]);
            if (k >= 1) rd = epim1(dot1(cJx[k], w.dX()[k - 1]), rd);
            rd = epim1(dot1(Ju, vk), rd);
            w.rdyn()[k] = rd;
            // x row of stage k+1 (k+1 = 1..N)
            const int kk = k + 1;
            double rx = epi1(dot1(w.Wq()[kk], w.dX()[k]), cgX[k]);
            if (kk < N) {
                rx = epi1(dot1(w.Wm()[kk], w.dU()[kk]), rx);
                rx = epim1(dot1(cJx[kk], w.mu()[kk]), rx);
            }
            rx += w.mu()[k];
            w.rsx()[k] = rx;
            const double lb = o.umin - U[k], ub = o.umax - U[k];
            const double rlk = dfinite(lb) ? vk - w.sl()[k] - lb : 0.0;
            const double ruk = dfinite(ub) ? ub - vk - w.su()[k] : 0.0;
            w.rl()[k] = rlk;
            w.ru()[k] = ruk;
            ninf = fold_absmax(fold_absmax(ninf, r), rx);
            dinf = fold_absmax(dinf, rd);
            linf = fold_absmax(linf, rlk);
            uinf = fold_absmax(uinf, ruk);
        }
        ninf = warp_max(ninf);
        dinf = warp_max(dinf);
        linf = warp_max(linf);
        uinf = warp_max(uinf);
        __syncwarp();
        // gap = (dot(sl, nl) + dot(su, nu)) / m: two serial chains, lanes 0 and 1
        double gap = 0.0;
        {
            const double* a = (lane & 1) ? w.su() : w.sl();
            const double* b = (lane & 1) ? w.nu() : w.nl();
            double s = 0.0;
            for (int k = 0; k < N; ++k) s += a[k] * b[k];
            const double dl = __shfl_sync(FULLMASK, s, 0);
            const double du = __shfl_sync(FULLMASK, s, 1);
            gap = m > 0 ? (dl + du) / m : 0.0;
        }
        if (ninf <= eps && dinf <= eps && linf <= eps && uinf <= eps && gap <= eps) {
            status = QP_OPTIMAL;
            break;
        }
        if (iter >= max_iter) {
            status = QP_MAXITER;
            break;
        }
        // barrier diagonal + affine rc (qp.cpp:353-372)
        for (int k = lane; k < N; k += 32) {
            const double lb = o.umin - U[k], ub = o.umax - U[k];
            const bool fl = dfinite(lb), fu = dfinite(ub);
            double bk = 0.0;
            if (fl) bk += w.nl()[k] / w.sl()[k];
            if (fu) bk += w.nu()[k] / w.su()[k];
            w.bar()[k] = bk;
            const double rcl = fl ? -w.sl()[k] * w.nl()[k] : 0.0;
            const double rcu = fu ? -w.su()[k] * w.nu()[k] : 0.0;
            w.rcl()[k] = rcl;
            w.rcu()[k] = rcu;
            double v = w.rsu()[k];
            if (fl) v -= (rcl - w.nl()[k] * w.rl()[k]) / w.sl()[k];
            if (fu) v += (rcu - w.nu()[k] * w.ru()[k]) / w.su()[k];
            w.rhat()[k] = v;
        }
        __syncwarp();
        // riccati_factor (qp.cpp:73-110) fused with the affine backward
        // vector sweep (qp.cpp:122-141); serial in k, all lanes.
        bool npd = false;
        {
            double P = w.Wq()[N];
            double pv = w.rsx()[N - 1];  // pvec[N] = qhat[N]
            w.val()[N] = P;
            w.pvec()[N] = pv;
            for (int k = N - 1; k >= 0; --k) {
                const double Ju = cJu[k];
                const double pju = epi0(dot1(P, Ju));
                double hh = epi0(dot1(Ju, pju));
                hh = hh + w.Wr()[k];
                hh = hh + w.bar()[k];
                if (hh <= 0.0 || !dfinite(hh)) {
                    npd = true;
                    break;
                }
                const double l = sqrt(hh);
                w.cholh()[k] = l;
                // vector part at stage k
                const double tmpv = epi1(dot1(P, -w.rdyn()[k]), pv);
                double hv = epi1(dot1(Ju, tmpv), w.rhat()[k]);
                hv = hv / l;
                hv = hv / l;
                hv = -hv;
                w.dff()[k] = hv;
                if (k >= 1) {
                    const double Jx = cJx[k];
                    const double pjx = epi0(dot1(P, Jx));
                    double gg = epi0(dot1(Ju, pjx));
                    gg = gg + w.Wm()[k];
                    double gn = gg / l;
                    gn = gn / l;
                    const double gain = -gn;
                    double pn = epi0(dot1(Jx, pjx));
                    pn = pn + w.Wq()[k];
                    pn = epi1(dot1(gg, gain), pn);
                    w.val()[k] = pn;
                    w.gain()[k] = gain;
                    w.gmat()[k] = gg;
                    double pvn = epi1(dot1(Jx, tmpv), w.rsx()[k - 1]);
                    pvn = epi1(dot1(gg, hv), pvn);
                    w.pvec()[k] = pvn;
                    P = pn;
                    pv = pvn;
                }
            }
        }
        if (npd) {
            status = QP_FAILED;
            break;
        }
        // forward rollout (qp.cpp:142-155) + expand (qp.cpp:308-317)
        auto rollout = [&]() {
            double dx = 0.0;
            for (int k = 0; k < N; ++k) {
                double du = w.dff()[k];
                if (k >= 1) du = epi1(dot1(w.gain()[k], dx), du);
                w.ddU()[k] = du;
                double dxn = -w.rdyn()[k];
                if (k >= 1) dxn = epi1(dot1(cJx[k], dx), dxn);
                dxn = epi1(dot1(cJu[k], du), dxn);
                dx = dxn;
                w.ddX()[k] = dx;
                const double mm = epi1(dot1(w.val()[k + 1], dx), w.pvec()[k + 1]);
                w.ddmu()[k] = -mm;
            }
        };
        auto expand_and_step = [&](double frac) {
            double alpha = 1.0;
            for (int k = lane; k < N; k += 32) {
                const double lb = o.umin - U[k], ub = o.umax - U[k];
                const bool fl = dfinite(lb), fu = dfinite(ub);
                const double dv = w.ddU()[k];
                const double dsl = fl ? dv + w.rl()[k] : 0.0;
                const double dsu = fu ? w.ru()[k] - dv : 0.0;
                const double dnl = fl ? (w.rcl()[k] - w.nl()[k] * dsl) / w.sl()[k] : 0.0;
                const double dnu = fu ? (w.rcu()[k] - w.nu()[k] * dsu) / w.su()[k] : 0.0;
                w.dsl()[k] = dsl;
                w.dsu()[k] = dsu;
                w.dnl()[k] = dnl;
                w.dnu()[k] = dnu;
                if (fl) {
                    if (dsl < 0.0) alpha = smin(alpha, -frac * w.sl()[k] / dsl);
                    if (dnl < 0.0) alpha = smin(alpha, -frac * w.nl()[k] / dnl);
                }
                if (fu) {
                    if (dsu < 0.0) alpha = smin(alpha, -frac * w.su()[k] / dsu);
                    if (dnu < 0.0) alpha = smin(alpha, -frac * w.nu()[k] / dnu);
                }
            }
            return warp_min(alpha);
        };
        rollout();
        __syncwarp();
        double sigma = 0.0;
        {
            const double alpha_aff = expand_and_step(1.0);
            if (m > 0 && gap > 0.0) {
                for (int k = lane; k < N; k += 32) {
                    const double lb = o.umin - U[k], ub = o.umax - U[k];
                    w.tmp()[2 * k] = dfinite(lb) ? (w.sl()[k] + alpha_aff * w.dsl()[k]) * (w.nl()[k] + alpha_aff * w.dnl()[k]) : 0.0;
                    w.tmp()[2 * k + 1] = dfinite(ub) ? (w.su()[k] + alpha_aff * w.dsu()[k]) * (w.nu()[k] + alpha_aff * w.dnu()[k]) : 0.0;
                }
                __syncwarp();
                double gap_aff = 0.0;
                for (int k = 0; k < N; ++k) {
                    const double lb = o.umin - U[k], ub = o.umax - U[k];
                    if (dfinite(lb)) gap_aff += w.tmp()[2 * k];
                    if (dfinite(ub)) gap_aff += w.tmp()[2 * k + 1];
                }
                gap_aff /= m;
                const double ratio = smax(0.0, gap_aff / gap);
                sigma = smin(1.0, ratio * ratio * ratio);
            }
        }
        __syncwarp();
        // corrector rc + condensed rhs (qp.cpp:390-395, :288-305)
        for (int k = lane; k < N; k += 32) {
            const double lb = o.umin - U[k], ub = o.umax - U[k];
            const bool fl = dfinite(lb), fu = dfinite(ub);
            if (fl) w.rcl()[k] = sigma * gap - w.sl()[k] * w.nl()[k] - w.dsl()[k] * w.dnl()[k];
            if (fu) w.rcu()[k] = sigma * gap - w.su()[k] * w.nu()[k] - w.dsu()[k] * w.dnu()[k];
            double v = w.rsu()[k];
            if (fl) v -= (w.rcl()[k] - w.nl()[k] * w.rl()[k]) / w.sl()[k];
            if (fu) v += (w.rcu()[k] - w.nu()[k] * w.ru()[k]) / w.su()[k];
            w.rhat()[k] = v;
        }
        __syncwarp();
        // corrector backward vector sweep with the cached factor (qp.cpp:122-141)
        {
            double pv = w.rsx()[N - 1];
            w.pvec()[N] = pv;
            for (int k = N - 1; k >= 0; --k) {
                const double Ju = cJu[k];
                const double l = w.cholh()[k];
                const double tmpv = epi1(dot1(w.val()[k + 1], -w.rdyn()[k]), pv);
                double hv = epi1(dot1(Ju, tmpv), w.rhat()[k]);
                hv = hv / l;
                hv = hv / l;
                hv = -hv;
                w.dff()[k] = hv;
                if (k >= 1) {
                    double pvn = epi1(dot1(cJx[k], tmpv), w.rsx()[k - 1]);
                    pvn = epi1(dot1(w.gmat()[k], hv), pvn);
                    w.pvec()[k] = pvn;
                    pv = pvn;
                }
            }
        }
        rollout();
        __syncwarp();
        const double alpha = expand_and_step(tau);
        // update (qp.cpp:397-410)
        for (int k = lane; k < N; k += 32) {
            const double lb = o.umin - U[k], ub = o.umax - U[k];
            w.dU()[k] = w.dU()[k] + alpha * w.ddU()[k];
            w.dX()[k] = w.dX()[k] + alpha * w.ddX()[k];
            w.mu()[k] = w.mu()[k] + alpha * w.ddmu()[k];
            if (dfinite(lb)) {
                w.sl()[k] += alpha * w.dsl()[k];
                w.nl()[k] += alpha * w.dnl()[k];
            }
            if (dfinite(ub)) {
                w.su()[k] += alpha * w.dsu()[k];
                w.nu()[k] += alpha * w.dnu()[k];
            }
        }
        cnt.ipm_stage += N;
        __syncwarp();
    }
    // final clamp (qp.cpp:414-419)
    for (int k = lane; k < N; k += 32) {
        const double lb = o.umin - U[k], ub = o.umax - U[k];
        w.dU()[k] = smin(smax(w.dU()[k], lb), ub);
    }
    __syncwarp();
    *iters_out = iter;
    return status;
}

// ------------------------------------------------------------------ SQP
struct SqpOut {
    bool converged;
    int status;  // ST_OK or ST_DOMAIN (propagating)
};

/// Lagrangian gradient pieces (sqp.cpp:102-128) at stage k.
/// hu = (0 - Ju_k lam_k) [+ (pi_u - pi_l)],  hx_k (slot x_{k+1}) = (gX_k + lam_k) - Jx_{k+1} lam_{k+1}.
__device__ __forceinline__ double lag_u(const double* Ju, const double* lam, int k) {
    return 0.0 - Ju[k] * lam[k];
}
__device__ __forceinline__ double lag_x(const double* gX, const double* Jx, const double* lam, int k, int N) {
    double h = gX[k] + lam[k];
    if (k + 1 < N) h -= Jx[k + 1] * lam[k + 1];
    return h;
}

/// check_convergence (sqp.cpp:86-96) with grad_l = lagrangian_gradient(gX, J, lam, pl, pu).
__device__ __forceinline__ bool kkt_check(const Ocp& o, const Ws& w, const double* gX, const double* g, const double* Jx,
                          const double* Ju, const double* lam, const double* pl, const double* pu, int m,
                          double eps, int lane) {
    const int N = o.N;
    double gl = 0.0, gi = 0.0;
    for (int k = lane; k < N; k += 32) {
        const double hu = lag_u(Ju, lam, k) + (pu[k] - pl[k]);
        const double hx = lag_x(gX, Jx, lam, k, N);
        gl = fold_absmax(fold_absmax(gl, hu), hx);
        gi = fold_absmax(gi, g[k]);
    }
    gl = warp_max(gl);
    gi = warp_max(gi);
    // mults = one_norm(lam) + one_norm(pi_l) + one_norm(pi_u): three serial
    // chains in one instruction stream (lanes 0, 1, 2)
    const double* a = (lane % 3 == 0) ? lam : (lane % 3 == 1) ? pl : pu;
    double s = 0.0;
    for (int k = 0; k < N; ++k) s += fabs(a[k]);
    const double n1 = __shfl_sync(FULLMASK, s, 0);
    const double n2 = __shfl_sync(FULLMASK, s, 1);
    const double n3 = __shfl_sync(FULLMASK, s, 2);
    double s_d = 1.0;
    if (m > 0) {
        const double mults = n1 + n2 + n3;
        s_d = smax(100.0, mults / m) / 100.0;
    }
    return gl / s_d <= eps && gi <= eps;
}

__device__ __forceinline__ void reset_blocks(const Ws& w, int N, int lane) {
    for (int k = lane; k <= N; k += 32) {
        w.Wq()[k] = 1.0;
        w.Wm()[k] = 0.0;
        w.Wr()[k] = 1.0;
    }
    __syncwarp();
}

/// bfgs_block_update (sqp.cpp:61-84) for a block of size n (1 or 2) stored as
/// (q, m, r) = (w00, w01 = w10, w11). Returns -1 on NotPositiveDefinite.
__device__ __forceinline__ int bfgs_block(double& q, double& mm, double& r, int n, const double* s,
                                          const double* y, bool uslot_only) {
    // For n == 1 the block is either a pure u slot (stored in r) or a pure x
    // slot (stored in q).
    if (n == 1) {
        double& wv = uslot_only ? r : q;
        const double ws = epi0(dot1(wv, s[0]));
        const double sws = dot1(s[0], ws);
        if (!(sws > kEpsMach)) return 0;
        const double sy = dot1(s[0], y[0]);
        const double theta = sy >= 0.2 * sws ? 1.0 : 0.8 * sws / (sws - sy);
        const double rr = theta * y[0] + (1.0 - theta) * ws;
        const double sr = dot1(s[0], rr);
        if (!(smin(sws, sr) > kEpsMach)) return 0;
        wv += rr * rr / sr - ws * ws / sws;
        if (wv <= 0.0 || !dfinite(wv)) return -1;
        return 1;
    }
    const double ws0 = epi0(0.0 + q * s[0] + mm * s[1]);
    const double ws1 = epi0(0.0 + mm * s[0] + r * s[1]);
    const double sws = 0.0 + s[0] * ws0 + s[1] * ws1;
    if (!(sws > kEpsMach)) return 0;
    const double sy = 0.0 + s[0] * y[0] + s[1] * y[1];
    const double theta = sy >= 0.2 * sws ? 1.0 : 0.8 * sws / (sws - sy);
    const double r0 = theta * y[0] + (1.0 - theta) * ws0;
    const double r1 = theta * y[1] + (1.0 - theta) * ws1;
    const double sr = 0.0 + s[0] * r0 + s[1] * r1;
    if (!(smin(sws, sr) > kEpsMach)) return 0;
    q += r0 * r0 / sr - ws0 * ws0 / sws;
    mm += r1 * r0 / sr - ws1 * ws0 / sws;  // w(1,0) == w(0,1): same products, commuted
    r += r1 * r1 / sr - ws1 * ws1 / sws;
    mm = 0.5 * (mm + mm);                  // symmetrize
    // cholesky_factor audit (linalg.cpp:69-103)
    if (q <= 0.0 || !dfinite(q)) return -1;
    const double l00 = sqrt(q);
    const double l10 = mm / l00;
    const double d = r - l10 * l10;
    if (d <= 0.0 || !dfinite(d)) return -1;
    return 1;
}

/// sqp_solve (sqp.cpp:182-411) on the iterate in (U, X) with duals in
/// lam/pil/piu (already warm-started). Returns status ST_DOMAIN if a
/// DomainError escapes (sim failure), otherwise ST_OK and converged flag.
__device__ __forceinline__ SqpOut sqp_solve(const Ocp& o, const Ws& w, double* U, double* X, const nmpcmc_sqp_options& opt,
                            int lane, Cnt& cnt) {
    const int N = o.N;
    SqpOut out{false, ST_OK};
    const int m_e = N;
    const int m_l = dfinite(o.umin) ? N : 0;
    const int m_u = dfinite(o.umax) ? N : 0;
    const int m = m_e + m_l + m_u;
    reset_blocks(w, N, lane);
    bool first_merit = true;

    // initial evaluation: NonFiniteState -> unconverged return (sqp.cpp:238-246)
    double f = eval_objective(o, w, X, w.gX(), lane);
    int st = eval_constraints(o, U, X, w.g(), w.Jx(), w.Ju(), lane, cnt);
    if (st == ST_DOMAIN) return SqpOut{false, ST_DOMAIN};
    if (st == ST_NONFINITE) return out;

    double* gX = w.gX();
    double* g = w.g();
    double* Jx = w.Jx();
    double* Ju = w.Ju();
    double* tgX = w.tgX();
    double* tg = w.tg();
    double* tJx = w.tJx();
    double* tJu = w.tJu();
    for (int iter = 0;; ++iter) {
        if (kkt_check(o, w, gX, g, Jx, Ju, w.lam(), w.pil(), w.piu(), m, opt.eps, lane)) {
            out.converged = true;
            break;
        }
        if (iter >= opt.max_iter) break;
        cnt.sqp_stage += N;

        int qp_iters = 0;
        int qs = solve_qp(o, w, U, gX, g, Jx, Ju, opt.qp_tol, opt.qp_max_iter, lane, cnt, &qp_iters);
        cnt.qp += 1;
        if (qs == QP_DOMAIN) return SqpOut{false, ST_DOMAIN};
        if (qs == QP_FAILED) {
            reset_blocks(w, N, lane);
            qs = solve_qp(o, w, U, gX, g, Jx, Ju, opt.qp_tol, opt.qp_max_iter, lane, cnt, &qp_iters);
            cnt.qp += 1;
            if (qs == QP_DOMAIN) return SqpOut{false, ST_DOMAIN};
            if (qs == QP_FAILED) break;  // rep.qp_failed
        }
        // KKT certificate with the fresh QP multipliers (sqp.cpp:285-310)
        if (kkt_check(o, w, gX, g, Jx, Ju, w.mu(), w.nl(), w.nu(), m, opt.eps, lane)) {
            for (int k = lane; k < N; k += 32) {
                w.lam()[k] = w.mu()[k];
                w.pil()[k] = w.nl()[k];
                w.piu()[k] = w.nu()[k];
            }
            __syncwarp();
            out.converged = true;
            break;
        }
        // merit_weights_update (sqp.cpp:12-20)
        for (int k = lane; k < N; k += 32) {
            const double am = fabs(w.mu()[k]);
            w.sig()[k] = first_merit ? am : smax(am, 0.5 * (w.sig()[k] + am));
        }
        first_merit = false;
        __syncwarp();

        // line_search (sqp.cpp:22-59)
        double penalty0 = 0.0, dd = 0.0;
        {
            for (int k = lane; k < N; k += 32) {
                w.tmp()[k] = w.sig()[k] * fabs(g[k]);
                w.tmp()[N + k] = gX[k] * w.dX()[k];
            }
            bool du_bad = false;
            for (int k = lane; k < N; k += 32) du_bad |= !dfinite(w.dU()[k]);
            du_bad = warp_any(du_bad);
            __syncwarp();
            // two serial chains (lanes even/odd): penalty0 and dot(grad f, dxi)
            const double* a = (lane & 1) ? w.tmp() + N : w.tmp();
            double s = 0.0;
            for (int k = 0; k < N; ++k) s += a[k];
            penalty0 = __shfl_sync(FULLMASK, s, 0);
            const double dot_gd = du_bad ? kNaN : __shfl_sync(FULLMASK, s, 1);
            dd = dot_gd - penalty0;
            __syncwarp();
        }
        const double merit_before = f + penalty0;
        double alpha = 1.0, merit = 0.0, f_trial = 0.0;
        bool ok = false;
        int trial_status = ST_OK;
        for (int bt = 0;; ++bt) {
            for (int k = lane; k < N; k += 32) {
                w.ddU()[k] = U[k] + alpha * w.dU()[k];  // trial iterate
                w.ddX()[k] = X[k] + alpha * w.dX()[k];
            }
            __syncwarp();
            f_trial = eval_objective(o, w, w.ddX(), tgX, lane);
            trial_status = eval_constraints(o, w.ddU(), w.ddX(), tg, tJx, tJu, lane, cnt);
            if (trial_status == ST_DOMAIN) return SqpOut{false, ST_DOMAIN};
            merit = HUGE_VAL;
            if (trial_status == ST_OK) {
                for (int k = lane; k < N; k += 32) w.tmp()[k] = w.sig()[k] * fabs(tg[k]);
                __syncwarp();
                merit = f_trial;
                for (int k = 0; k < N; ++k) merit += w.tmp()[k];
                __syncwarp();
            }
            cnt.ls += 1;
            ok = dfinite(merit) && merit <= merit_before + opt.c1 * alpha * dd;
            if (ok || bt >= opt.max_backtracks) break;
            alpha *= opt.backtrack_factor;
        }
        if (!ok && !dfinite(merit)) break;  // exhausted with no finite trial

        // accept: xi_new = xi + a * dxi equals the last trial bitwise, and so
        // do f, grad f and the constraint blocks (sqp.cpp:331-352)
        const double a = alpha;
        for (int k = lane; k < N; k += 32) {
            U[k] = w.ddU()[k];
            X[k] = w.ddX()[k];
        }
        for (int k = lane; k < N; k += 32) {
            w.lam()[k] += a * (w.mu()[k] - w.lam()[k]);
            w.pil()[k] += a * (w.nl()[k] - w.pil()[k]);
            w.piu()[k] += a * (w.nu()[k] - w.piu()[k]);
        }
        __syncwarp();
        // damped block BFGS on (s, y) with y = h_new - h_old (sqp.cpp:362-400)
        bool lost = false;
        for (int blk = lane; blk <= N; blk += 32) {
            double s[2], y[2];
            int n;
            bool uonly = false;
            if (blk == 0) {
                n = 1;
                uonly = true;
                s[0] = a * w.dU()[0];
                y[0] = lag_u(tJu, w.lam(), 0) - lag_u(Ju, w.lam(), 0);
            } else if (blk < N) {
                n = 2;
                s[0] = a * w.dX()[blk - 1];
                s[1] = a * w.dU()[blk];
                y[0] = lag_x(tgX, tJx, w.lam(), blk - 1, N) - lag_x(gX, Jx, w.lam(), blk - 1, N);
                y[1] = lag_u(tJu, w.lam(), blk) - lag_u(Ju, w.lam(), blk);
            } else {
                n = 1;
                s[0] = a * w.dX()[N - 1];
                y[0] = lag_x(tgX, tJx, w.lam(), N - 1, N) - lag_x(gX, Jx, w.lam(), N - 1, N);
            }
            double q = w.Wq()[blk], mm = w.Wm()[blk], r = w.Wr()[blk];
            const int res = bfgs_block(q, mm, r, n, s, y, uonly);
            if (res < 0) lost = true;
            if (res > 0) {
                w.Wq()[blk] = q;
                w.Wm()[blk] = mm;
                w.Wr()[blk] = r;
            }
        }
        lost = warp_any(lost);
        __syncwarp();
        if (lost) reset_blocks(w, N, lane);

        f = f_trial;
        double* t;
        t = gX; gX = tgX; tgX = t;
        t = g; g = tg; tg = t;
        t = Jx; Jx = tJx; tJx = t;
        t = Ju; Ju = tJu; tJu = t;
        cnt.sqp += 1;
    }
    return out;
}

// ------------------------------------------------------------ closed loop
/// The NMPC branch of run_closed_loop (montecarlo.cpp:80-157) for one sample.
template <int NX>
__device__ __forceinline__ void nmpc_closed_loop(const nmpcmc_scenario& sc, uint64_t sim_index, int nbar,
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
    const int N = o.N;
    Ws w{ws_stride(N)};
    Cnt cnt = {};

    // NmpcState (make_nmpc_state, controllers.cpp:25-48)
    double xhat = sc.x0_hat[0], Pf = sc.P0[0];
    bool have_last = false;  // last_xi empty -> cold start
    bool have_duals = false;
    int cur = 0;             // buffer holding last_xi

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

    for (int i = 0; i < nbar; ++i) {
        const double y = measure<NX>(p, pl, has_R, lR, rng);
        // ---- nmpc_step (controllers.cpp:114-212)
        if (!dfinite(y)) {
            status = ST_NONFINITE;
            break;
        }
        for (int k = lane; k < N; k += 32) w.sp()[k] = setpoint_at(sc, t + (k + 1) * sc.Ts);
        // filter_update (ekf.cpp:59-96) with the jitter retry (controllers.cpp:123-132)
        double xf, Pn;
        {
            const double c = o.inv_V;
            const double e = y - xhat / o.p.V;
            const double pc = epi0(dot1(Pf, c));
            double Rr = sc.R_filter;
            double Re = epi1(dot1(c, pc), Rr);
            if (Re <= 0.0 || !dfinite(Re)) {
                Rr = Rr + 1e-10;
                Re = epi1(dot1(c, pc), Rr);
                if (Re <= 0.0 || !dfinite(Re)) {
                    status = ST_NPD;
                    counts_lost = true;
                    break;
                }
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
        }
        o.x0 = xf;
        const int nb = cur ^ 1;  // buffer for this step's iterate
        double* U = w.U(nb);
        double* X = w.X(nb);
        const double* LU = w.U(cur);
        const double* LX = w.X(cur);
        if (have_last) {
            // shifted_inputs (controllers.cpp:70-83) + xi_from_inputs, fallback
            // shifted_warm_start (controllers.cpp:97-110)
            for (int k = lane; k < N; k += 32) {
                const int src = min(k + 1, N - 1);
                U[k] = smax(o.umin, smin(o.umax, LU[src]));
            }
            __syncwarp();
            const int st = xi_from_inputs(o, U, X, cnt);
            if (st == ST_DOMAIN) {
                status = ST_DOMAIN;
                break;
            }
            if (st == ST_NONFINITE) {
                for (int k = lane; k < N; k += 32) {
                    const int src = min(k + 1, N - 1);
                    U[k] = smax(o.umin, smin(o.umax, LU[src]));
                    X[k] = LX[src];
                }
                __syncwarp();
            }
            // shifted_multipliers (controllers.cpp:87-93), in place; sqp_solve
            // then projects the warm bound multipliers onto >= 0 (sqp.cpp:219-222)
            if (have_duals) {
                double l1 = 0, l2 = 0, l3 = 0;
                for (int k = lane; k < N; k += 32) {
                    const int src = N >= 2 ? min(k + 1, N - 1) : k;
                    l1 = w.lam()[src];
                    l2 = w.pil()[src];
                    l3 = w.piu()[src];
                    w.tmp()[k] = l1;
                    w.tmp()[N + k] = l2;
                    w.ddmu()[k] = l3;
                }
                __syncwarp();
                for (int k = lane; k < N; k += 32) {
                    w.lam()[k] = w.tmp()[k];
                    w.pil()[k] = smax(0.0, w.tmp()[N + k]);  // sqp.cpp:219-222
                    w.piu()[k] = smax(0.0, w.ddmu()[k]);
                }
                __syncwarp();
            }
        } else {
            // nominal_input (controllers.cpp:58-66) + cold xi_from_inputs
            const bool fl = dfinite(o.umin), fh = dfinite(o.umax);
            const double u_nom = fl && fh ? 0.5 * (o.umin + o.umax) : smax(o.umin, smin(o.umax, 0.0));
            for (int k = lane; k < N; k += 32) U[k] = u_nom;
            __syncwarp();
            const int st = xi_from_inputs(o, U, X, cnt);
            if (st == ST_DOMAIN) {
                status = ST_DOMAIN;
                break;
            }
            if (st == ST_NONFINITE) {
                for (int k = lane; k < N; k += 32) {
                    U[k] = u_nom;
                    X[k] = o.x0;
                }
                __syncwarp();
            }
            for (int k = lane; k < N; k += 32) {
                w.lam()[k] = 0.0;
                w.pil()[k] = 0.0;
                w.piu()[k] = 0.0;
            }
            __syncwarp();
        }
        const SqpOut so = sqp_solve(o, w, U, X, sc.sqp, lane, cnt);
        if (so.status != ST_OK) {
            status = so.status;
            break;
        }
        const double u = smax(o.umin, smin(o.umax, U[0]));
        cur = nb;
        have_last = true;
        have_duals = true;
        // predict (ekf.cpp:26-57), np RK4 steps on (x, P)
        {
            const double t_next = t + o.Ts;
            const double h = (t_next - t) / sc.np;
            double x = xf, P = Pn;
            int st = ST_OK;
            for (int s = 0; s < sc.np && st == ST_OK; ++s) {
                double k1x, k1p, k2x, k2p, k3x, k3p, k4x, k4p;
                if ((st = joint_rhs1(o.p, x, P, u, k1x, k1p))) break;
                if ((st = joint_rhs1(o.p, x + 0.5 * h * k1x, P + 0.5 * h * k1p, u, k2x, k2p))) break;
                if ((st = joint_rhs1(o.p, x + 0.5 * h * k2x, P + 0.5 * h * k2p, u, k3x, k3p))) break;
                if ((st = joint_rhs1(o.p, x + h * k3x, P + h * k3p, u, k4x, k4p))) break;
                x += (h / 6.0) * (k1x + 2.0 * k2x + 2.0 * k3x + k4x);
                P += (h / 6.0) * (k1p + 2.0 * k2p + 2.0 * k3p + k4p);
                if (!dfinite(x) || !dfinite(P)) st = ST_NONFINITE;
            }
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
        if (record && i % stride == 0 && lane == 0) {
            double* rw = traj + (size_t)row * 5;
            rw[0] = t;
            rw[1] = z;
            rw[2] = zbar;
            rw[3] = u;
            rw[4] = y;
        }
        if (record && i % stride == 0) ++row;
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
}

template <int NX>
__global__ void __launch_bounds__(32) nmpc_kernel(const __grid_constant__ nmpcmc_scenario sc, uint64_t first_sim,
                                                  int64_t n_sims, int nbar, nmpcmc_sim_record* records,
                                                  nmpcmc_work_counters* counters, double* traj, int traj_rows) {
    const int64_t i = blockIdx.x;
    if (i >= n_sims) return;
    nmpc_closed_loop<NX>(sc, first_sim + (uint64_t)i, nbar, records + i,
                         counters ? counters + i : nullptr,
                         traj ? traj + (size_t)i * traj_rows * 5 : nullptr);
}

inline int launch_nmpc(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
                       nmpcmc_work_counters* d_cnt, double* d_traj, int rows, int sm_count,
                       cudaStream_t stream) {
    (void)sm_count;
    if (sc.ctrl_variant != NMPCMC_ONE_STATE) return NMPCMC_UNSUPPORTED;
    const size_t smem = ws_bytes(sc.N);
    if (smem > 227 * 1024) return NMPCMC_UNSUPPORTED;
    if (sc.truth_variant == NMPCMC_THREE_STATE) {
        cudaFuncSetAttribute(nmpc_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        nmpc_kernel<3><<<(unsigned)n, 32, smem, stream>>>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows);
    } else {
        cudaFuncSetAttribute(nmpc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        nmpc_kernel<1><<<(unsigned)n, 32, smem, stream>>>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows);
    }
    return NMPCMC_OK;
}

}  // namespace nmpcmc_dev
