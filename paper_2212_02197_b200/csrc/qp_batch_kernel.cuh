// qp_batch_kernel.cuh -- K5: batched standalone stagewise QP solver (SURVEY.md
// §8(f) row 4). One thread per QP; every QP of a batch has the same (N, n_x,
// n_u), runtime dimensions up to n_x <= 8, n_u <= 4.
//
// Restates, with the reference's floating-point operation order (bitwise vs
// the compiled reference, tests/test_gpu_qp.py):
//   solve_qp               qp.cpp:173-423 (Mehrotra predictor-corrector IPM)
//   riccati_factor_solve   qp.cpp:157-171
//   riccati_factor         qp.cpp:73-110     riccati_solve_vectors  qp.cpp:116-155
//   gemm/gemv/cholesky/symmetrize/axpy   linalg.cpp:69-235
// DomainError (lb > ub) and NotPositiveDefinite (riccati_factor_solve) become
// per-QP status codes.
//
// Input (packed, read-only): for each QP, N+1 stage blocks of QPB_STAGE
// doubles: Q[nx*nx] M[nx*nu] R[nu*nu] q[nx] r[nu] Jx[nx*nx] Ju[nx*nu] b[nx]
// lb[nu] ub[nu], matrices column-major; members a stage does not use are
// ignored (stage 0: Q M q Jx; stage N: all but Q q).
// Output per QP: delta_xi[N(nu+nx)] mu[N nx] nu_l[N nu] nu_u[N nu].
#pragma once

#include <stdint.h>

#include "device_common.cuh"

namespace nmpcmc_dev {
namespace qpb {

constexpr int QX = 8, QU = 4;
constexpr int kBlock = 64;

struct Dims {
    int N, nx, nu, max_iter, mode;
    double tol;
};

/// Packed-input view of one QP.
struct In {
    const double* p;
    int nx, nu;
    int oM, oR, oq, or_, oJx, oJu, ob, olb, oub, SB;
    __device__ In(const double* base, int nx_, int nu_) : p(base), nx(nx_), nu(nu_) {
        oM = nx * nx;
        oR = oM + nx * nu;
        oq = oR + nu * nu;
        or_ = oq + nx;
        oJx = or_ + nu;
        oJu = oJx + nx * nx;
        ob = oJu + nx * nu;
        olb = ob + nx;
        oub = olb + nu;
        SB = oub + nu;
    }
    __device__ double at(int k, int off) const { return __ldg(p + (int64_t)k * SB + off); }
    __device__ double Q(int k, int i, int j) const { return at(k, j * nx + i); }
    __device__ double M(int k, int i, int j) const { return at(k, oM + j * nx + i); }  // nx x nu
    __device__ double R(int k, int i, int j) const { return at(k, oR + j * nu + i); }
    __device__ double q(int k, int i) const { return at(k, oq + i); }
    __device__ double r(int k, int i) const { return at(k, or_ + i); }
    __device__ double Jx(int k, int i, int j) const { return at(k, oJx + j * nx + i); }
    __device__ double Ju(int k, int i, int j) const { return at(k, oJu + j * nx + i); }  // nx x nu
    __device__ double b(int k, int i) const { return at(k, ob + i); }
    __device__ double lb(int k, int i) const { return at(k, olb + i); }
    __device__ double ub(int k, int i) const { return at(k, oub + i); }
};

__host__ __device__ inline int stage_doubles(int nx, int nu) {
    return 2 * nx * nx + 2 * nx * nu + nu * nu + 2 * nx + 3 * nu;
}
__host__ __device__ inline int64_t solution_doubles(int N, int nx, int nu) {
    return (int64_t)N * (nu + nx) + (int64_t)N * nx + 2 * (int64_t)N * nu;
}

/// SoA workspace view: element e of slot t at ws[e * T + t].
struct Ws {
    double* p;
    int64_t T;
    __device__ __forceinline__ double& operator[](int64_t e) const { return p[e * T]; }
};

/// Workspace offsets for one QP.
struct Lay {
    int64_t DXI, MU, SL, SU, NL, NU, RS, RD, RL, RU, CL, CU, DSL, DSU, DNL, DNU, BAR, SDX, SDM, CH, GN, GM, VAL,
        PV, DFF, RH, total;
    __host__ __device__ Lay(int N, int nx, int nu) {
        const int64_t L = (int64_t)N * (nu + nx), NX = (int64_t)N * nx, NV = (int64_t)N * nu;
        int64_t o = 0;
        auto take = [&](int64_t n) {
            const int64_t a = o;
            o += n;
            return a;
        };
        DXI = take(L), MU = take(NX), SL = take(NV), SU = take(NV), NL = take(NV), NU = take(NV);
        RS = take(L), RD = take(NX), RL = take(NV), RU = take(NV), CL = take(NV), CU = take(NV);
        DSL = take(NV), DSU = take(NV), DNL = take(NV), DNU = take(NV), BAR = take(NV);
        SDX = take(L), SDM = take(NX);
        CH = take((int64_t)N * nu * nu), GN = take((int64_t)N * nu * nx), GM = take((int64_t)N * nu * nx);
        VAL = take((int64_t)(N + 1) * nx * nx), PV = take((int64_t)(N + 1) * nx), DFF = take(NV), RH = take(NV);
        total = o;
    }
};

struct Ctx {
    In in;
    Ws w;
    Lay L;
    int N, nx, nu;
    __device__ int uo(int k) const { return k * (nu + nx); }
    __device__ int xo(int k) const { return (k - 1) * (nu + nx) + nu; }
    __device__ double& val(int k, int i, int j) const { return w[L.VAL + ((int64_t)k * nx + j) * nx + i]; }
    __device__ double& chol(int k, int i, int j) const { return w[L.CH + ((int64_t)k * nu + j) * nu + i]; }
    __device__ double& gain(int k, int i, int j) const { return w[L.GN + ((int64_t)k * nx + j) * nu + i]; }  // nu x nx
    __device__ double& gmat(int k, int i, int j) const { return w[L.GM + ((int64_t)k * nx + j) * nu + i]; }
};

/// cholesky_factor (linalg.cpp:69-103, non-semidefinite) of the nu x nu
/// h (column-major, local) into stage k's factor. True on NotPositiveDefinite.
__device__ bool chol_factor(const Ctx& c, int k, const double* h) {
    const int n = c.nu;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) c.chol(k, i, j) = 0.0;
    for (int j = 0; j < n; ++j) {
        double d = h[j * n + j];
        for (int q = 0; q < j; ++q) d -= c.chol(k, j, q) * c.chol(k, j, q);
        if (d <= 0.0 || !dfinite(d)) return true;
        const double ljj = sqrt(d);
        c.chol(k, j, j) = ljj;
        for (int i = j + 1; i < n; ++i) {
            double s = h[j * n + i];
            for (int q = 0; q < j; ++q) s -= c.chol(k, i, q) * c.chol(k, j, q);
            c.chol(k, i, j) = s / ljj;
        }
    }
    return false;
}
/// cholesky_solve_in_place (linalg.cpp:111-128) with stage k's factor.
__device__ void chol_solve(const Ctx& c, int k, double* b) {
    const int n = c.nu;
    for (int i = 0; i < n; ++i) {
        double s = b[i];
        for (int q = 0; q < i; ++q) s -= c.chol(k, i, q) * b[q];
        b[i] = s / c.chol(k, i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = b[i];
        for (int q = i + 1; q < n; ++q) s -= c.chol(k, q, i) * b[q];
        b[i] = s / c.chol(k, i, i);
    }
}

/// riccati_factor (qp.cpp:73-110); barrier = nullptr-equivalent when !bar.
__device__ bool rfactor(const Ctx& c, bool bar) {
    const int N = c.N, nx = c.nx, nu = c.nu;
    // P_{k+1} carried from stage to stage (no store-to-load round trip)
    double pn[QX * QX];
    for (int j = 0; j < nx; ++j)
        for (int i = 0; i < nx; ++i) {
            pn[j * nx + i] = c.in.Q(N, i, j);
            c.val(N, i, j) = pn[j * nx + i];
        }
    for (int k = N - 1; k >= 0; --k) {
        double pju[QX * QU], h[QU * QU];
        for (int j = 0; j < nu; ++j)  // pju = P_{k+1} Ju
            for (int i = 0; i < nx; ++i) {
                double s = 0.0;
                for (int l = 0; l < nx; ++l) s += pn[l * nx + i] * c.in.Ju(k, l, j);
                pju[j * nx + i] = 1.0 * s + 0.0;
            }
        for (int j = 0; j < nu; ++j)  // h = Ju' pju
            for (int i = 0; i < nu; ++i) {
                double s = 0.0;
                for (int l = 0; l < nx; ++l) s += c.in.Ju(k, l, i) * pju[j * nx + l];
                h[j * nu + i] = 1.0 * s + 0.0;
            }
        for (int j = 0; j < nu; ++j)
            for (int i = 0; i < nu; ++i) h[j * nu + i] += c.in.R(k, i, j);
        if (bar)
            for (int i = 0; i < nu; ++i) h[i * nu + i] += c.w[c.L.BAR + k * nu + i];
        for (int cc = 0; cc < nu; ++cc)  // symmetrize
            for (int r = cc + 1; r < nu; ++r) {
                const double v = 0.5 * (h[cc * nu + r] + h[r * nu + cc]);
                h[cc * nu + r] = v;
                h[r * nu + cc] = v;
            }
        if (chol_factor(c, k, h)) return true;
        if (k >= 1) {
            double pjx[QX * QX], g[QU * QX], p[QX * QX];
            for (int j = 0; j < nx; ++j)  // pjx = P_{k+1} Jx
                for (int i = 0; i < nx; ++i) {
                    double s = 0.0;
                    for (int l = 0; l < nx; ++l) s += pn[l * nx + i] * c.in.Jx(k, l, j);
                    pjx[j * nx + i] = 1.0 * s + 0.0;
                }
            for (int j = 0; j < nx; ++j)  // g = Ju' pjx + M'
                for (int i = 0; i < nu; ++i) {
                    double s = 0.0;
                    for (int l = 0; l < nx; ++l) s += c.in.Ju(k, l, i) * pjx[j * nx + l];
                    g[j * nu + i] = 1.0 * s + 0.0;
                }
            for (int j = 0; j < nx; ++j)
                for (int i = 0; i < nu; ++i) g[j * nu + i] += c.in.M(k, j, i);
            for (int j = 0; j < nx; ++j) {  // gain = -cholesky_solve(chol_h, g)
                double col[QU];
                for (int i = 0; i < nu; ++i) col[i] = g[j * nu + i];
                chol_solve(c, k, col);
                for (int i = 0; i < nu; ++i) c.gain(k, i, j) = -col[i];
            }
            for (int j = 0; j < nx; ++j)  // p = Jx' pjx + Q
                for (int i = 0; i < nx; ++i) {
                    double s = 0.0;
                    for (int l = 0; l < nx; ++l) s += c.in.Jx(k, l, i) * pjx[j * nx + l];
                    p[j * nx + i] = 1.0 * s + 0.0;
                }
            for (int j = 0; j < nx; ++j)
                for (int i = 0; i < nx; ++i) p[j * nx + i] += c.in.Q(k, i, j);
            for (int j = 0; j < nx; ++j)  // p = 1.0 g' gain + 1.0 p
                for (int i = 0; i < nx; ++i) {
                    double s = 0.0;
                    for (int l = 0; l < nu; ++l) s += g[i * nu + l] * c.gain(k, l, j);
                    p[j * nx + i] = 1.0 * s + 1.0 * p[j * nx + i];
                }
            for (int cc = 0; cc < nx; ++cc)
                for (int r = cc + 1; r < nx; ++r) {
                    const double v = 0.5 * (p[cc * nx + r] + p[r * nx + cc]);
                    p[cc * nx + r] = v;
                    p[r * nx + cc] = v;
                }
            for (int j = 0; j < nx; ++j) {
                for (int i = 0; i < nx; ++i) {
                    c.val(k, i, j) = p[j * nx + i];
                    pn[j * nx + i] = p[j * nx + i];
                }
                for (int i = 0; i < nu; ++i) c.gmat(k, i, j) = g[j * nu + i];
            }
        }
    }
    return false;
}

/// Right-hand sides of riccati_solve_vectors: rhat_k = rh(k), qhat_k,
/// bhat_k. RHS_QP: the solve_qp condensed system (RH, RS x-rows, -RD);
/// otherwise the QP data (r, q, b) for riccati_factor_solve.
template <bool RHS_QP>
__device__ void rsolve(const Ctx& c, int64_t DX, int64_t DM) {
    const int N = c.N, nx = c.nx, nu = c.nu;
    const Ws& w = c.w;
    auto qh = [&](int k, int i) -> double { return RHS_QP ? w[c.L.RS + c.xo(k) + i] : c.in.q(k, i); };
    auto bh = [&](int k, int i) -> double { return RHS_QP ? -w[c.L.RD + k * nx + i] : c.in.b(k, i); };
    auto rh = [&](int k, int i) -> double { return RHS_QP ? w[c.L.RH + k * nu + i] : c.in.r(k, i); };
    double pvn[QX];  // p_{k+1} carried from stage to stage
    for (int i = 0; i < nx; ++i) {
        pvn[i] = qh(N, i);
        w[c.L.PV + N * nx + i] = pvn[i];
    }
    for (int k = N - 1; k >= 0; --k) {
        double tmp[QX], h[QU];
        for (int i = 0; i < nx; ++i) {
            double s = 0.0;
            for (int j = 0; j < nx; ++j) s += c.val(k + 1, i, j) * bh(k, j);
            tmp[i] = 1.0 * s + 1.0 * pvn[i];
        }
        for (int i = 0; i < nu; ++i) {
            double s = 0.0;
            for (int j = 0; j < nx; ++j) s += c.in.Ju(k, j, i) * tmp[j];
            h[i] = 1.0 * s + 1.0 * rh(k, i);
        }
        chol_solve(c, k, h);
        for (int i = 0; i < nu; ++i) w[c.L.DFF + k * nu + i] = -h[i];
        if (k >= 1) {
            for (int i = 0; i < nx; ++i) {
                double s = 0.0;
                for (int j = 0; j < nx; ++j) s += c.in.Jx(k, j, i) * tmp[j];
                double p = 1.0 * s + 1.0 * qh(k, i);
                double s2 = 0.0;
                for (int j = 0; j < nu; ++j) s2 += c.gmat(k, j, i) * w[c.L.DFF + k * nu + j];
                p = 1.0 * s2 + 1.0 * p;
                w[c.L.PV + k * nx + i] = p;
                pvn[i] = p;
            }
        }
    }
    double dx[QX];
    for (int i = 0; i < nx; ++i) dx[i] = 0.0;
    for (int k = 0; k < N; ++k) {
        double du[QU], dn[QX];
        for (int i = 0; i < nu; ++i) {
            double v = w[c.L.DFF + k * nu + i];
            if (k >= 1) {
                double s = 0.0;
                for (int j = 0; j < nx; ++j) s += c.gain(k, i, j) * dx[j];
                v = 1.0 * s + 1.0 * v;
            }
            du[i] = v;
            w[DX + c.uo(k) + i] = v;
        }
        for (int i = 0; i < nx; ++i) dn[i] = bh(k, i);
        if (k >= 1)
            for (int i = 0; i < nx; ++i) {
                double s = 0.0;
                for (int j = 0; j < nx; ++j) s += c.in.Jx(k, i, j) * dx[j];
                dn[i] = 1.0 * s + 1.0 * dn[i];
            }
        for (int i = 0; i < nx; ++i) {
            double s = 0.0;
            for (int j = 0; j < nu; ++j) s += c.in.Ju(k, i, j) * du[j];
            dn[i] = 1.0 * s + 1.0 * dn[i];
        }
        for (int i = 0; i < nx; ++i) {
            dx[i] = dn[i];
            w[DX + c.xo(k + 1) + i] = dx[i];
        }
        for (int i = 0; i < nx; ++i) {
            double s = 0.0;
            for (int j = 0; j < nx; ++j) s += c.val(k + 1, i, j) * dx[j];
            w[DM + k * nx + i] = -(1.0 * s + 1.0 * w[c.L.PV + (k + 1) * nx + i]);
        }
    }
}

enum : int { QPB_OPTIMAL = 0, QPB_MAXITER = 1, QPB_FAILED = 2, QPB_DOMAIN = 3, QPB_NOT_PD = 4 };

__device__ __forceinline__ double inf_fold(double m, double x) { return smax(m, fabs(x)); }

/// solve_qp (qp.cpp:173-423). Returns the status; iterations in *iters.
__device__ int solve_qp(const Ctx& c, double tol, int max_iter, int* iters) {
    const int N = c.N, nx = c.nx, nu = c.nu, nv = N * nu;
    const int64_t Lx = (int64_t)N * (nu + nx), NX = (int64_t)N * nx;
    const Ws& w = c.w;
    const Lay& L = c.L;
    auto lbv = [&](int idx) { return c.in.lb(idx / nu, idx % nu); };
    auto ubv = [&](int idx) { return c.in.ub(idx / nu, idx % nu); };
    *iters = 0;
    int m = 0;
    double scale = 1.0;
    for (int k = 0; k < N; ++k) {
        for (int i = 0; i < nu; ++i) {
            const double lb = c.in.lb(k, i), ub = c.in.ub(k, i);
            if (lb > ub) return QPB_DOMAIN;
            if (dfinite(lb)) ++m, scale = smax(scale, fabs(lb));
            if (dfinite(ub)) ++m, scale = smax(scale, fabs(ub));
        }
        double nr = 0.0, nb = 0.0;
        for (int i = 0; i < nu; ++i) nr = inf_fold(nr, c.in.r(k, i));
        scale = smax(scale, nr);
        for (int i = 0; i < nx; ++i) nb = inf_fold(nb, c.in.b(k, i));
        scale = smax(scale, nb);
    }
    for (int k = 1; k <= N; ++k) {
        double nq = 0.0;
        for (int i = 0; i < nx; ++i) nq = inf_fold(nq, c.in.q(k, i));
        scale = smax(scale, nq);
    }
    const double eps = tol * scale;
    for (int64_t e = 0; e < Lx; ++e) w[L.DXI + e] = 0.0;
    for (int64_t e = 0; e < NX; ++e) w[L.MU + e] = 0.0;
    for (int idx = 0; idx < nv; ++idx) {
        const bool fl = dfinite(lbv(idx)), fu = dfinite(ubv(idx));
        w[L.SL + idx] = fl ? smax(1.0, fabs(lbv(idx))) : 0.0;
        w[L.NL + idx] = fl ? 1.0 : 0.0;
        w[L.SU + idx] = fu ? smax(1.0, fabs(ubv(idx))) : 0.0;
        w[L.NU + idx] = fu ? 1.0 : 0.0;
        w[L.RL + idx] = 0.0, w[L.RU + idx] = 0.0, w[L.CL + idx] = 0.0, w[L.CU + idx] = 0.0;
        w[L.DSL + idx] = 0.0, w[L.DSU + idx] = 0.0, w[L.DNL + idx] = 0.0, w[L.DNU + idx] = 0.0;
    }
    auto residuals = [&]() {
        for (int k = 0; k < N; ++k) {
            for (int i = 0; i < nu; ++i) {
                double s = 0.0;
                for (int j = 0; j < nu; ++j) s += c.in.R(k, i, j) * w[L.DXI + c.uo(k) + j];
                double ru = 1.0 * s + 1.0 * c.in.r(k, i);
                if (k >= 1) {
                    double s2 = 0.0;
                    for (int j = 0; j < nx; ++j) s2 += c.in.M(k, j, i) * w[L.DXI + c.xo(k) + j];
                    ru = 1.0 * s2 + 1.0 * ru;
                }
                double s3 = 0.0;
                for (int j = 0; j < nx; ++j) s3 += c.in.Ju(k, j, i) * w[L.MU + k * nx + j];
                ru = -1.0 * s3 + 1.0 * ru;
                const int idx = k * nu + i;
                ru += w[L.NU + idx] - w[L.NL + idx];
                w[L.RS + c.uo(k) + i] = ru;
            }
            double rd[QX];
            for (int i = 0; i < nx; ++i) rd[i] = w[L.DXI + c.xo(k + 1) + i] + -1.0 * c.in.b(k, i);
            if (k >= 1)
                for (int i = 0; i < nx; ++i) {
                    double s = 0.0;
                    for (int j = 0; j < nx; ++j) s += c.in.Jx(k, i, j) * w[L.DXI + c.xo(k) + j];
                    rd[i] = -1.0 * s + 1.0 * rd[i];
                }
            for (int i = 0; i < nx; ++i) {
                double s = 0.0;
                for (int j = 0; j < nu; ++j) s += c.in.Ju(k, i, j) * w[L.DXI + c.uo(k) + j];
                w[L.RD + k * nx + i] = -1.0 * s + 1.0 * rd[i];
            }
        }
        for (int k = 1; k <= N; ++k) {
            double rx[QX];
            for (int i = 0; i < nx; ++i) {
                double s = 0.0;
                for (int j = 0; j < nx; ++j) s += c.in.Q(k, i, j) * w[L.DXI + c.xo(k) + j];
                rx[i] = 1.0 * s + 1.0 * c.in.q(k, i);
            }
            if (k < N) {
                for (int i = 0; i < nx; ++i) {
                    double s = 0.0;
                    for (int j = 0; j < nu; ++j) s += c.in.M(k, i, j) * w[L.DXI + c.uo(k) + j];
                    rx[i] = 1.0 * s + 1.0 * rx[i];
                }
                for (int i = 0; i < nx; ++i) {
                    double s = 0.0;
                    for (int j = 0; j < nx; ++j) s += c.in.Jx(k, j, i) * w[L.MU + k * nx + j];
                    rx[i] = -1.0 * s + 1.0 * rx[i];
                }
            }
            for (int i = 0; i < nx; ++i) w[L.RS + c.xo(k) + i] = rx[i] + w[L.MU + (k - 1) * nx + i];
        }
        for (int idx = 0; idx < nv; ++idx) {
            const int k = idx / nu;
            const double v = w[L.DXI + c.uo(k) + idx % nu];
            w[L.RL + idx] = dfinite(lbv(idx)) ? v - w[L.SL + idx] - lbv(idx) : 0.0;
            w[L.RU + idx] = dfinite(ubv(idx)) ? ubv(idx) - v - w[L.SU + idx] : 0.0;
        }
    };
    auto condensed = [&]() {
        for (int k = 0; k < N; ++k)
            for (int i = 0; i < nu; ++i) {
                const int idx = k * nu + i;
                double v = w[L.RS + c.uo(k) + i];
                if (dfinite(lbv(idx))) v -= (w[L.CL + idx] - w[L.NL + idx] * w[L.RL + idx]) / w[L.SL + idx];
                if (dfinite(ubv(idx))) v += (w[L.CU + idx] - w[L.NU + idx] * w[L.RU + idx]) / w[L.SU + idx];
                w[L.RH + idx] = v;
            }
        rsolve<true>(c, L.SDX, L.SDM);
    };
    auto expand = [&]() {
        for (int idx = 0; idx < nv; ++idx) {
            const int k = idx / nu;
            const double dv = w[L.SDX + c.uo(k) + idx % nu];
            const bool fl = dfinite(lbv(idx)), fu = dfinite(ubv(idx));
            const double dsl = fl ? dv + w[L.RL + idx] : 0.0;
            const double dsu = fu ? w[L.RU + idx] - dv : 0.0;
            w[L.DSL + idx] = dsl;
            w[L.DSU + idx] = dsu;
            w[L.DNL + idx] = fl ? (w[L.CL + idx] - w[L.NL + idx] * dsl) / w[L.SL + idx] : 0.0;
            w[L.DNU + idx] = fu ? (w[L.CU + idx] - w[L.NU + idx] * dsu) / w[L.SU + idx] : 0.0;
        }
    };
    auto max_step = [&](double frac) {
        double a = 1.0;
        auto cap = [&](double val, double dir) {
            if (dir < 0.0) a = smin(a, -frac * val / dir);
        };
        for (int idx = 0; idx < nv; ++idx) {
            if (dfinite(lbv(idx))) {
                cap(w[L.SL + idx], w[L.DSL + idx]);
                cap(w[L.NL + idx], w[L.DNL + idx]);
            }
            if (dfinite(ubv(idx))) {
                cap(w[L.SU + idx], w[L.DSU + idx]);
                cap(w[L.NU + idx], w[L.DNU + idx]);
            }
        }
        return a;
    };
    int status = QPB_FAILED;
    for (int iter = 0;; ++iter) {
        residuals();
        double gap = 0.0;
        if (m > 0) {
            double a = 0.0, b = 0.0;
            for (int idx = 0; idx < nv; ++idx) a += w[L.SL + idx] * w[L.NL + idx];
            for (int idx = 0; idx < nv; ++idx) b += w[L.SU + idx] * w[L.NU + idx];
            gap = (a + b) / m;
        }
        double ns = 0.0, nd = 0.0, nl = 0.0, nu_ = 0.0;
        for (int64_t e = 0; e < Lx; ++e) ns = inf_fold(ns, w[L.RS + e]);
        for (int64_t e = 0; e < NX; ++e) nd = inf_fold(nd, w[L.RD + e]);
        for (int idx = 0; idx < nv; ++idx) nl = inf_fold(nl, w[L.RL + idx]);
        for (int idx = 0; idx < nv; ++idx) nu_ = inf_fold(nu_, w[L.RU + idx]);
        if (ns <= eps && nd <= eps && nl <= eps && nu_ <= eps && gap <= eps) {
            status = QPB_OPTIMAL;
            break;
        }
        if (iter >= max_iter) {
            status = QPB_MAXITER;
            break;
        }
        for (int idx = 0; idx < nv; ++idx) {
            double b = 0.0;
            if (dfinite(lbv(idx))) b += w[L.NL + idx] / w[L.SL + idx];
            if (dfinite(ubv(idx))) b += w[L.NU + idx] / w[L.SU + idx];
            w[L.BAR + idx] = b;
        }
        if (rfactor(c, true)) {
            status = QPB_FAILED;
            break;
        }
        for (int idx = 0; idx < nv; ++idx) {
            w[L.CL + idx] = dfinite(lbv(idx)) ? -w[L.SL + idx] * w[L.NL + idx] : 0.0;
            w[L.CU + idx] = dfinite(ubv(idx)) ? -w[L.SU + idx] * w[L.NU + idx] : 0.0;
        }
        condensed();
        expand();
        double sigma = 0.0;
        if (m > 0 && gap > 0.0) {
            const double aa = max_step(1.0);
            double ga = 0.0;
            for (int idx = 0; idx < nv; ++idx) {
                if (dfinite(lbv(idx)))
                    ga += (w[L.SL + idx] + aa * w[L.DSL + idx]) * (w[L.NL + idx] + aa * w[L.DNL + idx]);
                if (dfinite(ubv(idx)))
                    ga += (w[L.SU + idx] + aa * w[L.DSU + idx]) * (w[L.NU + idx] + aa * w[L.DNU + idx]);
            }
            ga /= m;
            const double ratio = smax(0.0, ga / gap);
            sigma = smin(1.0, ratio * ratio * ratio);
        }
        for (int idx = 0; idx < nv; ++idx) {
            if (dfinite(lbv(idx)))
                w[L.CL + idx] = sigma * gap - w[L.SL + idx] * w[L.NL + idx] - w[L.DSL + idx] * w[L.DNL + idx];
            if (dfinite(ubv(idx)))
                w[L.CU + idx] = sigma * gap - w[L.SU + idx] * w[L.NU + idx] - w[L.DSU + idx] * w[L.DNU + idx];
        }
        condensed();
        expand();
        const double alpha = max_step(0.995);
        for (int64_t e = 0; e < Lx; ++e) w[L.DXI + e] += alpha * w[L.SDX + e];
        for (int64_t e = 0; e < NX; ++e) w[L.MU + e] += alpha * w[L.SDM + e];
        for (int idx = 0; idx < nv; ++idx) {
            if (dfinite(lbv(idx))) {
                w[L.SL + idx] += alpha * w[L.DSL + idx];
                w[L.NL + idx] += alpha * w[L.DNL + idx];
            }
            if (dfinite(ubv(idx))) {
                w[L.SU + idx] += alpha * w[L.DSU + idx];
                w[L.NU + idx] += alpha * w[L.DNU + idx];
            }
        }
        *iters = iter + 1;
    }
    for (int k = 0; k < N; ++k)
        for (int i = 0; i < nu; ++i) {
            double& v = w[L.DXI + c.uo(k) + i];
            v = smin(smax(v, c.in.lb(k, i)), c.in.ub(k, i));
        }
    return status;
}

/// One thread per QP (grid-stride). mode 0: solve_qp; 1: riccati_factor_solve.
__global__ void __launch_bounds__(kBlock) qp_batch_kernel(Dims d, int64_t batch, const double* __restrict__ in,
                                                          double* __restrict__ out, int32_t* status,
                                                          int32_t* iterations, double* ws_all, int64_t slots) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= slots) return;
    const int SB = stage_doubles(d.nx, d.nu);
    const int64_t SO = solution_doubles(d.N, d.nx, d.nu);
    const Lay L(d.N, d.nx, d.nu);
    for (int64_t b = tid; b < batch; b += slots) {
        const Ctx c{In(in + b * (int64_t)(d.N + 1) * SB, d.nx, d.nu), Ws{ws_all + tid, slots}, L, d.N, d.nx, d.nu};
        const int64_t Lx = (int64_t)d.N * (d.nu + d.nx), NX = (int64_t)d.N * d.nx, NV = (int64_t)d.N * d.nu;
        double* o = out + b * SO;
        int st, it = 0;
        if (d.mode == 1) {
            st = rfactor(c, false) ? QPB_NOT_PD : QPB_OPTIMAL;
            if (st == QPB_OPTIMAL) rsolve<false>(c, L.DXI, L.MU);
            for (int64_t e = 0; e < Lx; ++e) o[e] = st == QPB_OPTIMAL ? c.w[L.DXI + e] : 0.0;
            for (int64_t e = 0; e < NX; ++e) o[Lx + e] = st == QPB_OPTIMAL ? c.w[L.MU + e] : 0.0;
            for (int64_t e = 0; e < 2 * NV; ++e) o[Lx + NX + e] = 0.0;
        } else {
            st = solve_qp(c, d.tol, d.max_iter, &it);
            const bool ok = st != QPB_DOMAIN;
            for (int64_t e = 0; e < Lx; ++e) o[e] = ok ? c.w[L.DXI + e] : 0.0;
            for (int64_t e = 0; e < NX; ++e) o[Lx + e] = ok ? c.w[L.MU + e] : 0.0;
            for (int64_t e = 0; e < NV; ++e) o[Lx + NX + e] = ok ? c.w[L.NL + e] : 0.0;
            for (int64_t e = 0; e < NV; ++e) o[Lx + NX + NV + e] = ok ? c.w[L.NU + e] : 0.0;
        }
        status[b] = st;
        iterations[b] = it;
    }
}

inline int64_t qp_slots(int sm_count, int64_t batch) {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, qp_batch_kernel, kBlock, 0);
    if (blocks < 1) blocks = 1;
    const int64_t s = (int64_t)sm_count * blocks * kBlock;
    return s < batch ? s : batch;
}

}  // namespace qpb
}  // namespace nmpcmc_dev
