// nmpcmc_port.cpp -- CPU restatement of the reference's closed-loop Monte
// Carlo path. TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke()
// and bench.py's CPU arm as the checker, never by the product.
//
// This is an independent restatement (own data structures, own code) of the
// algorithm in /root/reference/proj/core/src, written for generic state
// dimension (the three-state controller model included) and keeping the
// reference's floating-point operation order exactly, so it agrees bitwise
// with the compiled reference (oracle/_ref) in both libm modes
// (tests/test_oracle_port.py). Each function cites the reference it follows.
//
// Build: oracle/Makefile (twice: -DPORT_XLIBM for the exact-libm variant).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <limits>
#include <thread>
#include <vector>

#include "nmpcmc_gpu.h"

// Op-counting build (oracle/port/flopcount.cpp) supplies its own libm and
// phase/unit markers; they are empty here.
#ifndef PORT_PHASE
#define PORT_PHASE(ph)
#define PORT_UNIT(u, n)
#define PORT_TO_DOUBLE(x) (x)
#define PORT_REAL double
#endif

#if defined(PORT_CUSTOM_LIBM)
#define PFX(name) nmpcmc_portc_##name
#elif defined(PORT_XLIBM)
extern "C" {
double nmx_exp(double);
double nmx_log(double);
void nmx_sincos(double, double*, double*);
}
static inline double P_EXP(double x) { return nmx_exp(x); }
static inline double P_LOG(double x) { return nmx_log(x); }
static inline void P_SINCOS(double x, double* s, double* c) { nmx_sincos(x, s, c); }
#define PFX(name) nmpcmc_portx_##name
#else
static inline double P_EXP(double x) { return std::exp(x); }
static inline double P_LOG(double x) { return std::log(x); }
static inline void P_SINCOS(double x, double* s, double* c) {
    *s = std::sin(x);
    *c = std::cos(x);
}
#define PFX(name) nmpcmc_port_##name
#endif

namespace port {

using Vec = std::vector<double>;

// Failure taxonomy (errors.hpp:9-32) -- only what the path can raise.
struct NotPD {};
struct NonFinite {};
struct Domain {};

// ------------------------------------------------------------ dense algebra
/// Column-major dense matrix (linalg.hpp:20-56).
struct Mat {
    int r = 0, c = 0;
    Vec v;
    Mat() = default;
    Mat(int rows, int cols) : r(rows), c(cols), v(static_cast<size_t>(rows) * cols, 0.0) {}
    double& at(int i, int j) { return v[static_cast<size_t>(j) * r + i]; }
    double at(int i, int j) const { return v[static_cast<size_t>(j) * r + i]; }
    static Mat eye(int n) {
        Mat m(n, n);
        for (int i = 0; i < n; ++i) m.at(i, i) = 1.0;
        return m;
    }
};

/// C := alpha op(A) op(B) + (beta == 0 ? 0 : beta C) with k-ascending sums
/// and the (j, i, k) loop order of gemm_into (linalg.cpp:144-164).
static void mm(double alpha, const Mat& A, bool ta, const Mat& B, bool tb, double beta, Mat& C) {
    const int rows = ta ? A.c : A.r, inner = ta ? A.r : A.c, cols = tb ? B.r : B.c;
    if (beta == 0.0) C = Mat(rows, cols);
    for (int j = 0; j < cols; ++j)
        for (int i = 0; i < rows; ++i) {
            double s = 0.0;
            for (int k = 0; k < inner; ++k) s += (ta ? A.at(k, i) : A.at(i, k)) * (tb ? B.at(j, k) : B.at(k, j));
            C.at(i, j) = alpha * s + (beta == 0.0 ? 0.0 : beta * C.at(i, j));
        }
}
static Mat mul(const Mat& A, bool ta, const Mat& B, bool tb) {
    Mat C;
    mm(1.0, A, ta, B, tb, 0.0, C);
    return C;
}

/// y := alpha op(A) x + (beta == 0 ? 0 : beta y) (gemv_into, linalg.cpp:179-189).
static void mv(double alpha, const Mat& A, bool ta, const Vec& x, double beta, Vec& y) {
    const int rows = ta ? A.c : A.r, inner = ta ? A.r : A.c;
    if (beta == 0.0) y.assign(rows, 0.0);
    for (int i = 0; i < rows; ++i) {
        double s = 0.0;
        for (int j = 0; j < inner; ++j) s += (ta ? A.at(j, i) : A.at(i, j)) * x[j];
        y[i] = alpha * s + (beta == 0.0 ? 0.0 : beta * y[i]);
    }
}

static double dotv(const Vec& a, const Vec& b) {  // linalg.cpp:197-202
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}
static double ninf(const Vec& a) {  // inf_norm, linalg.cpp:204-208
    double m = 0.0;
    for (double x : a) m = std::max(m, std::abs(x));
    return m;
}
static double n1(const Vec& a) {  // one_norm, linalg.cpp:210-214
    double s = 0.0;
    for (double x : a) s += std::abs(x);
    return s;
}
static bool finite(const Vec& a) {
    for (double x : a)
        if (!std::isfinite(x)) return false;
    return true;
}
static void sym(Mat& A) {  // symmetrize, linalg.cpp:227-235
    for (int j = 0; j < A.c; ++j)
        for (int i = j + 1; i < A.r; ++i) {
            const double m = 0.5 * (A.at(i, j) + A.at(j, i));
            A.at(i, j) = m;
            A.at(j, i) = m;
        }
}

/// Lower Cholesky factor; semidefinite variant zeroes columns with a pivot
/// within 1e-13 max(max|a_ii|, 1) (cholesky_impl, linalg.cpp:69-103).
static Mat chol(const Mat& A, bool semi) {
    const int n = A.r;
    double big = 0.0;
    if (semi)
        for (int i = 0; i < n; ++i) big = std::max(big, std::abs(A.at(i, i)));
    const double tol = semi ? 1e-13 * std::max(big, 1.0) : 0.0;
    Mat L(n, n);
    for (int j = 0; j < n; ++j) {
        double d = A.at(j, j);
        for (int k = 0; k < j; ++k) d -= L.at(j, k) * L.at(j, k);
        if (semi && std::abs(d) <= tol) continue;
        if (d <= 0.0 || !std::isfinite(d)) throw NotPD{};
        const double p = std::sqrt(d);
        L.at(j, j) = p;
        for (int i = j + 1; i < n; ++i) {
            double s = A.at(i, j);
            for (int k = 0; k < j; ++k) s -= L.at(i, k) * L.at(j, k);
            L.at(i, j) = s / p;
        }
    }
    return L;
}

/// Solve L L' x = b in place (cholesky_solve_in_place, linalg.cpp:111-128).
static void chol_solve(const Mat& L, Vec& b) {
    const int n = L.r;
    for (int i = 0; i < n; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= L.at(i, k) * b[k];
        b[i] = s / L.at(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = b[i];
        for (int k = i + 1; k < n; ++k) s -= L.at(k, i) * b[k];
        b[i] = s / L.at(i, i);
    }
}
static Mat chol_solve_mat(const Mat& L, const Mat& B) {  // cholesky_solve, linalg.cpp:130-142
    Mat X = B;
    Vec col(B.r);
    for (int j = 0; j < B.c; ++j) {
        for (int i = 0; i < B.r; ++i) col[i] = X.at(i, j);
        chol_solve(L, col);
        for (int i = 0; i < B.r; ++i) X.at(i, j) = col[i];
    }
    return X;
}

// --------------------------------------------------------------------- RNG
/// Philox4x32-10 counter stream with Box-Muller normals (rng.cpp:10-91).
struct Rng {
    uint64_t seed, stream, blk = 0;
    uint32_t w[4] = {0, 0, 0, 0};
    int used = 4;
    bool spare_ok = false;
    double spare = 0.0;
    Rng(uint64_t s, uint64_t st) : seed(s), stream(st) {}
    static void block(const uint32_t in[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
        uint32_t x0 = in[0], x1 = in[1], x2 = in[2], x3 = in[3];
        for (int round = 0; round < 10; ++round) {
            if (round) {
                k0 += 0x9E3779B9u;
                k1 += 0xBB67AE85u;
            }
            const uint64_t p0 = uint64_t(0xD2511F53u) * x0, p1 = uint64_t(0xCD9E8D57u) * x2;
            const uint32_t y0 = uint32_t(p1 >> 32) ^ x1 ^ k0, y1 = uint32_t(p1);
            const uint32_t y2 = uint32_t(p0 >> 32) ^ x3 ^ k1, y3 = uint32_t(p0);
            x0 = y0, x1 = y1, x2 = y2, x3 = y3;
        }
        out[0] = x0, out[1] = x1, out[2] = x2, out[3] = x3;
    }
    uint32_t u32() {
        if (used == 4) {
            const uint32_t ctr[4] = {uint32_t(blk), uint32_t(blk >> 32), uint32_t(stream), uint32_t(stream >> 32)};
            block(ctr, uint32_t(seed), uint32_t(seed >> 32), w);
            ++blk;
            used = 0;
        }
        return w[used++];
    }
    double uni() {
        const uint64_t hi = u32();
        const uint64_t lo = u32();
        return static_cast<double>(((hi << 32) | lo) >> 11) * 0x1.0p-53;
    }
    double normal() {
        if (spare_ok) {
            spare_ok = false;
            return spare;
        }
        const double a = 1.0 - uni();
        const double b = uni();
        const double rad = std::sqrt(-2.0 * P_LOG(a));
        double s, c;
        P_SINCOS(0x1.921fb54442d18p+2 * b, &s, &c);  // 2*pi folded, as GCC does
        spare = rad * s;
        spare_ok = true;
        return rad * c;
    }
};

// ------------------------------------------------------------------- CSTR
constexpr double kFlow = 1e-3 / 60.0;  // cstr.hpp:46

/// One CSTR variant (cstr.cpp:21-34 stoichiometry + cstr.hpp:21-34 params).
struct Cstr {
    nmpcmc_cstr_params p;
    int nx;  // 3 truth-like, 1 reduced
    double S[3], Cin[3], sb[3];
    Cstr(const nmpcmc_cstr_params& q, int variant) : p(q) {
        nx = variant == NMPCMC_ONE_STATE ? 1 : 3;
        if (nx == 3) {
            S[0] = -1.0, S[1] = -2.0, S[2] = p.beta;
            Cin[0] = p.cA_in, Cin[1] = p.cB_in, Cin[2] = p.cT_in;
            sb[0] = p.sigmaA, sb[1] = p.sigmaB, sb[2] = p.sigmaT;
        } else {
            S[0] = p.beta;
            Cin[0] = p.cT_in;
            sb[0] = p.sigmaT;
        }
    }
    /// concentrations + DomainError (cstr.cpp:13-17, :36-40)
    void conc(const Vec& c, double& cA, double& cB, double& cT) const {
        if (nx == 3) {
            cA = c[0], cB = c[1], cT = c[2];
        } else {
            cT = c[0];
            cA = p.cA_in - (cT - p.cT_in) / p.beta;
            cB = p.cB_in - 2.0 * (cT - p.cT_in) / p.beta;
        }
        if (cT <= 0.0) throw Domain{};
    }
    Vec drift(const Vec& n, double u) const {  // cstr.cpp:42-53
        const double f = u * kFlow;
        Vec c(nx);
        for (int i = 0; i < nx; ++i) c[i] = n[i] / p.V;
        double cA, cB, cT;
        conc(c, cA, cB, cT);
        const double r = p.k0 * P_EXP(-p.EaR / cT) * cA * cB;
        Vec d(nx);
        for (int i = 0; i < nx; ++i) d[i] = Cin[i] * f - c[i] * f + S[i] * r * p.V;
        return d;
    }
    Mat diffusion(double u) const {  // cstr.cpp:55-65
        const double f = u * kFlow;
        Mat s(nx, nx);
        for (int i = 0; i < nx; ++i) s.at(i, i) = f * sb[i];
        return s;
    }
    Mat jac_x(const Vec& x, double u) const {  // cstr.cpp:99-119
        const double f = u * kFlow;
        Vec c(nx);
        for (int i = 0; i < nx; ++i) c[i] = x[i] / p.V;
        double cA, cB, cT;
        conc(c, cA, cB, cT);
        const double k = p.k0 * P_EXP(-p.EaR / cT);
        Mat J(nx, nx);
        if (nx == 3) {
            const double g[3] = {k * cB, k * cA, k * (p.EaR / (cT * cT)) * cA * cB};
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) J.at(i, j) = (i == j ? -f / p.V : 0.0) + S[i] * g[j];
        } else {
            const double g = k * (p.EaR / (cT * cT)) * cA * cB + k * (-cB / p.beta - 2.0 * cA / p.beta);
            J.at(0, 0) = -f / p.V + p.beta * g;
        }
        return J;
    }
    Mat jac_u(const Vec& x) const {  // cstr.cpp:120-127
        Mat J(nx, 1);
        for (int i = 0; i < nx; ++i) J.at(i, 0) = (Cin[i] - x[i] / p.V) * kFlow;
        return J;
    }
    double out(const Vec& x) const { return x[nx - 1] / p.V; }  // cstr.cpp:86-89
};

// ------------------------------------------------------------------ plant
/// simulate_interval + euler_maruyama_step (model.cpp:13-37).
static Vec simulate(const Cstr& m, double t0, double t1, Vec x, double u, int ns, Rng& rng) {
    PORT_PHASE(PLANT);
    const double dt = (t1 - t0) / ns;
    const double sdt = std::sqrt(dt);
    Vec dw(m.nx);
    for (int k = 0; k < ns; ++k) {
        for (int j = 0; j < m.nx; ++j) dw[j] = sdt * rng.normal();
        Vec nx = x;
        const Vec f = m.drift(x, u);
        for (int i = 0; i < m.nx; ++i) nx[i] += dt * f[i];
        mv(1.0, m.diffusion(u), false, dw, 1.0, nx);
        if (!finite(nx)) throw NonFinite{};
        x = nx;
    }
    return x;
}

/// measure (model.cpp:39-48), n_y = 1.
static double measure(const Cstr& m, bool hasR, double R, const Vec& x, Rng& rng) {
    PORT_PHASE(PLANT);
    Vec y{m.out(x)};
    if (hasR) {
        Mat Rm(1, 1);
        Rm.at(0, 0) = R;
        const Mat L = chol(Rm, true);
        const Vec z{rng.normal()};
        mv(1.0, L, false, z, 1.0, y);
    }
    return y[0];
}

// -------------------------------------------------------------------- EKF
/// predict (ekf.cpp:12-57): RK4 on (x, P), symmetrised each step.
static void ekf_predict(const Cstr& m, Vec& x, Mat& P, double u, double t, double tn, int np) {
    PORT_PHASE(EKF);
    const double h = (tn - t) / np;
    auto rhs = [&](const Vec& xs, const Mat& Ps, Vec& dx, Mat& dP) {
        dx = m.drift(xs, u);
        const Mat A = m.jac_x(xs, u);
        mm(1.0, A, false, Ps, false, 0.0, dP);
        mm(1.0, Ps, false, A, true, 1.0, dP);
        const Mat s = m.diffusion(u);
        mm(1.0, s, false, s, true, 1.0, dP);
    };
    const size_t nP = P.v.size();
    for (int step = 0; step < np; ++step) {
        Vec d1, d2, d3, d4, xs(x.size());
        Mat D1, D2, D3, D4, Ps = P;
        rhs(x, P, d1, D1);
        for (size_t i = 0; i < x.size(); ++i) xs[i] = x[i] + 0.5 * h * d1[i];
        for (size_t i = 0; i < nP; ++i) Ps.v[i] = P.v[i] + 0.5 * h * D1.v[i];
        rhs(xs, Ps, d2, D2);
        for (size_t i = 0; i < x.size(); ++i) xs[i] = x[i] + 0.5 * h * d2[i];
        for (size_t i = 0; i < nP; ++i) Ps.v[i] = P.v[i] + 0.5 * h * D2.v[i];
        rhs(xs, Ps, d3, D3);
        for (size_t i = 0; i < x.size(); ++i) xs[i] = x[i] + h * d3[i];
        for (size_t i = 0; i < nP; ++i) Ps.v[i] = P.v[i] + h * D3.v[i];
        rhs(xs, Ps, d4, D4);
        for (size_t i = 0; i < x.size(); ++i) x[i] += (h / 6.0) * (d1[i] + 2.0 * d2[i] + 2.0 * d3[i] + d4[i]);
        for (size_t i = 0; i < nP; ++i) P.v[i] += (h / 6.0) * (D1.v[i] + 2.0 * D2.v[i] + 2.0 * D3.v[i] + D4.v[i]);
        sym(P);
        if (!finite(x) || !finite(P.v)) throw NonFinite{};
    }
}

/// filter_update (ekf.cpp:59-96), Joseph form, n_y = 1.
static void ekf_update(const Cstr& m, Vec& x, Mat& P, double y, double R) {
    PORT_PHASE(EKF);
    const int n = m.nx;
    Mat C(1, n);
    C.at(0, n - 1) = 1.0 / m.p.V;
    const double e = y - m.out(x);
    const Mat PC = mul(P, false, C, true);
    Mat Re(1, 1);
    Re.at(0, 0) = R;
    mm(1.0, C, false, PC, false, 1.0, Re);
    sym(Re);
    const Mat L = chol(Re, false);
    Mat PCt(1, n);
    for (int i = 0; i < n; ++i) PCt.at(0, i) = PC.at(i, 0);
    const Mat Kt = chol_solve_mat(L, PCt);
    Mat K(n, 1);
    for (int i = 0; i < n; ++i) K.at(i, 0) = Kt.at(0, i);
    mv(1.0, K, false, Vec{e}, 1.0, x);
    Mat IKC = Mat::eye(n);
    mm(-1.0, K, false, C, false, 1.0, IKC);
    const Mat T = mul(IKC, false, P, false);
    Mat Pn = mul(T, false, IKC, true);
    Mat Rm(1, 1);
    Rm.at(0, 0) = R;
    const Mat KR = mul(K, false, Rm, false);
    mm(1.0, KR, false, K, true, 1.0, Pn);
    sym(Pn);
    P = Pn;
}

// -------------------------------------------------------------------- OCP
/// The regulator NLP (ocp.hpp:18-34) with the interleaved xi layout
/// (ocp.hpp:37-43): u slot of stage k at k*(nu+nx), x_k at (k-1)*(nu+nx)+nu.
struct Nlp {
    const Cstr* m;
    int N, Nc, nx;
    double Ts, t0, umin, umax, Qz;
    Vec x0;
    Vec sp;  // zbar_1..N
    int stride() const { return 1 + nx; }
    int uo(int k) const { return k * stride(); }
    int xo(int k) const { return (k - 1) * stride() + 1; }
    int size() const { return N * stride(); }
};

struct Shot {
    Vec F;
    Mat Fx, Fu;
};

/// shoot (ocp.cpp:9-74): Nc RK4 steps with forward sensitivities.
static Shot shoot(const Nlp& q, const Vec& x, double u) {
    PORT_PHASE(SHOOT);
    PORT_UNIT(SHOOT, 1);
    const Cstr& m = *q.m;
    const double h = q.Ts / q.Nc;
    Shot s{x, Mat::eye(q.nx), Mat(q.nx, 1)};
    struct St {
        Vec k;
        Mat kx, ku;
    };
    auto stage = [&](const Vec& xs, const Mat& sx, const Mat& su) {
        St r;
        r.k = m.drift(xs, u);
        const Mat A = m.jac_x(xs, u);
        const Mat B = m.jac_u(xs);
        r.kx = mul(A, false, sx, false);
        r.ku = B;
        mm(1.0, A, false, su, false, 1.0, r.ku);
        return r;
    };
    auto fwd = [&](const Vec& a, const Vec& d, double c) {
        Vec o = a;
        for (size_t i = 0; i < o.size(); ++i) o[i] += c * h * d[i];
        return o;
    };
    auto fwdm = [&](const Mat& a, const Mat& d, double c) {
        Mat o = a;
        for (size_t i = 0; i < o.v.size(); ++i) o.v[i] += c * h * d.v[i];
        return o;
    };
    for (int st = 0; st < q.Nc; ++st) {
        const St a = stage(s.F, s.Fx, s.Fu);
        const St b = stage(fwd(s.F, a.k, 0.5), fwdm(s.Fx, a.kx, 0.5), fwdm(s.Fu, a.ku, 0.5));
        const St c = stage(fwd(s.F, b.k, 0.5), fwdm(s.Fx, b.kx, 0.5), fwdm(s.Fu, b.ku, 0.5));
        const St d = stage(fwd(s.F, c.k, 1.0), fwdm(s.Fx, c.kx, 1.0), fwdm(s.Fu, c.ku, 1.0));
        for (int i = 0; i < q.nx; ++i) s.F[i] += (h / 6.0) * (a.k[i] + 2.0 * b.k[i] + 2.0 * c.k[i] + d.k[i]);
        for (size_t i = 0; i < s.Fx.v.size(); ++i)
            s.Fx.v[i] += (h / 6.0) * (a.kx.v[i] + 2.0 * b.kx.v[i] + 2.0 * c.kx.v[i] + d.kx.v[i]);
        for (size_t i = 0; i < s.Fu.v.size(); ++i)
            s.Fu.v[i] += (h / 6.0) * (a.ku.v[i] + 2.0 * b.ku.v[i] + 2.0 * c.ku.v[i] + d.ku.v[i]);
    }
    if (!finite(s.F)) throw NonFinite{};
    return s;
}

/// eval_objective (ocp.cpp:76-99).
static double objective(const Nlp& q, const Vec& xi, Vec* grad) {
    double phi = 0.0;
    if (grad) grad->assign(q.size(), 0.0);
    Mat Q(1, 1), H(1, q.nx);
    Q.at(0, 0) = q.Qz;
    H.at(0, q.nx - 1) = 1.0 / q.m->p.V;
    for (int k = 1; k <= q.N; ++k) {
        Vec xk(xi.begin() + q.xo(k), xi.begin() + q.xo(k) + q.nx);
        Vec res{q.m->out(xk) - q.sp[k - 1]};
        Vec qres;
        mv(1.0, Q, false, res, 0.0, qres);
        phi += q.Ts * dotv(res, qres);
        Vec g;
        mv(1.0, H, true, qres, 0.0, g);
        if (grad)
            for (int i = 0; i < q.nx; ++i) (*grad)[q.xo(k) + i] += 2.0 * q.Ts * g[i];
    }
    return phi;
}

struct Blocks {
    Vec g;
    std::vector<Mat> Fx, Fu;
    std::vector<Vec> b;
};

/// eval_constraints (ocp.cpp:101-135).
static Blocks constraints(const Nlp& q, const Vec& xi) {
    Blocks o;
    o.g.assign(static_cast<size_t>(q.N) * q.nx, 0.0);
    Vec xk = q.x0;
    for (int k = 0; k < q.N; ++k) {
        const Shot s = shoot(q, xk, xi[q.uo(k)]);
        Vec bk(q.nx);
        for (int i = 0; i < q.nx; ++i) {
            const double nx = xi[q.xo(k + 1) + i];
            bk[i] = s.F[i] - nx;
            o.g[k * q.nx + i] = nx - s.F[i];
        }
        o.Fx.push_back(s.Fx);
        o.Fu.push_back(s.Fu);
        o.b.push_back(bk);
        xk.assign(xi.begin() + q.xo(k + 1), xi.begin() + q.xo(k + 1) + q.nx);
    }
    return o;
}

/// xi_from_inputs (ocp.cpp:137-154).
static Vec xi_from_u(const Nlp& q, const Vec& us) {
    PORT_PHASE(XI);
    Vec xi(q.size());
    Vec xk = q.x0;
    for (int k = 0; k < q.N; ++k) {
        xi[q.uo(k)] = us[k];
        const Shot s = shoot(q, xk, us[k]);
        for (int i = 0; i < q.nx; ++i) xi[q.xo(k + 1) + i] = s.F[i];
        xk = s.F;
    }
    return xi;
}

// --------------------------------------------------------------------- QP
/// Stage data (qp.hpp:24-30) with n_u = 1.
struct Stage {
    Mat Q, M, R, Jx, Ju;
    Vec q, r, b;
    double lb = 0, ub = 0;
};
struct QpOut {
    Vec dxi, mu, nl, nu;
    int status = 2;  // 0 Optimal, 1 MaxIter, 2 Failed
};

struct Factor {
    std::vector<Mat> L, K, G, P;
};

/// riccati_factor (qp.cpp:73-110).
static Factor rfactor(const std::vector<Stage>& st, int N, int nx, const Vec& bar) {
    Factor f;
    f.L.resize(N);
    f.K.resize(N);
    f.G.resize(N);
    f.P.resize(N + 1);
    f.P[N] = st[N].Q;
    for (int k = N - 1; k >= 0; --k) {
        const Stage& s = st[k];
        const Mat& Pn = f.P[k + 1];
        const Mat PJu = mul(Pn, false, s.Ju, false);
        Mat H = mul(s.Ju, true, PJu, false);
        H.at(0, 0) += s.R.at(0, 0);
        H.at(0, 0) += bar[k];
        sym(H);
        f.L[k] = chol(H, false);
        if (k >= 1) {
            const Mat PJx = mul(Pn, false, s.Jx, false);
            Mat G = mul(s.Ju, true, PJx, false);
            for (int j = 0; j < nx; ++j) G.at(0, j) += s.M.at(j, 0);
            Mat K = chol_solve_mat(f.L[k], G);
            for (double& v : K.v) v = -v;
            Mat P = mul(s.Jx, true, PJx, false);
            for (int j = 0; j < nx; ++j)
                for (int i = 0; i < nx; ++i) P.at(i, j) += s.Q.at(i, j);
            mm(1.0, G, true, K, false, 1.0, P);
            sym(P);
            f.P[k] = P;
            f.K[k] = K;
            f.G[k] = G;
        }
    }
    return f;
}

/// riccati_solve_vectors (qp.cpp:116-155).
static void rsolve(const std::vector<Stage>& st, int N, int nx, const Factor& f, const Vec& rh,
                   const std::vector<Vec>& qh, const std::vector<Vec>& bh, Vec& dxi, Vec& dmu) {
    std::vector<Vec> pv(N + 1);
    Vec dff(N);
    pv[N] = qh[N];
    for (int k = N - 1; k >= 0; --k) {
        const Stage& s = st[k];
        Vec t = pv[k + 1];
        mv(1.0, f.P[k + 1], false, bh[k], 1.0, t);
        Vec h{rh[k]};
        mv(1.0, s.Ju, true, t, 1.0, h);
        chol_solve(f.L[k], h);
        dff[k] = -h[0];
        if (k >= 1) {
            Vec p = qh[k];
            mv(1.0, s.Jx, true, t, 1.0, p);
            mv(1.0, f.G[k], true, Vec{dff[k]}, 1.0, p);
            pv[k] = p;
        }
    }
    const int w = 1 + nx;
    dxi.assign(static_cast<size_t>(N) * w, 0.0);
    dmu.assign(static_cast<size_t>(N) * nx, 0.0);
    Vec dx(nx, 0.0);
    for (int k = 0; k < N; ++k) {
        Vec du{dff[k]};
        if (k >= 1) mv(1.0, f.K[k], false, dx, 1.0, du);
        dxi[k * w] = du[0];
        Vec dn = bh[k];
        if (k >= 1) mv(1.0, st[k].Jx, false, dx, 1.0, dn);
        mv(1.0, st[k].Ju, false, du, 1.0, dn);
        dx = dn;
        for (int i = 0; i < nx; ++i) dxi[k * w + 1 + i] = dx[i];
        Vec mvec = pv[k + 1];
        mv(1.0, f.P[k + 1], false, dx, 1.0, mvec);
        for (int i = 0; i < nx; ++i) dmu[k * nx + i] = -mvec[i];
    }
}

/// solve_qp (qp.cpp:173-423): Mehrotra predictor-corrector interior point.
static QpOut solve_qp(const std::vector<Stage>& st, int N, int nx, double tol, int max_iter) {
    PORT_PHASE(QP);
    const int w = 1 + nx;
    auto uo = [&](int k) { return k * w; };
    auto xo = [&](int k) { return (k - 1) * w + 1; };
    std::vector<char> fl(N), fu(N);
    int m = 0;
    double scale = 1.0;
    for (int k = 0; k < N; ++k) {
        if (st[k].lb > st[k].ub) throw Domain{};
        fl[k] = std::isfinite(st[k].lb);
        fu[k] = std::isfinite(st[k].ub);
        if (fl[k]) ++m, scale = std::max(scale, std::fabs(st[k].lb));
        if (fu[k]) ++m, scale = std::max(scale, std::fabs(st[k].ub));
        scale = std::max(scale, ninf(st[k].r));
        scale = std::max(scale, ninf(st[k].b));
    }
    for (int k = 1; k <= N; ++k) scale = std::max(scale, ninf(st[k].q));
    const double eps = tol * scale;
    QpOut o;
    o.dxi.assign(static_cast<size_t>(N) * w, 0.0);
    o.mu.assign(static_cast<size_t>(N) * nx, 0.0);
    Vec sl(N, 0.0), su(N, 0.0), nl(N, 0.0), nu(N, 0.0);
    for (int k = 0; k < N; ++k) {
        if (fl[k]) sl[k] = std::max(1.0, std::fabs(st[k].lb)), nl[k] = 1.0;
        if (fu[k]) su[k] = std::max(1.0, std::fabs(st[k].ub)), nu[k] = 1.0;
    }
    Vec rs(o.dxi.size()), rd(o.mu.size()), rl(N), ru(N), cl(N, 0.0), cu(N, 0.0);
    Vec dsl(N), dsu(N), dnl(N), dnu(N);
    auto resid = [&]() {  // qp.cpp:237-284
        for (int k = 0; k < N; ++k) {
            const Stage& s = st[k];
            const Vec v{o.dxi[uo(k)]};
            const Vec mk(o.mu.begin() + k * nx, o.mu.begin() + (k + 1) * nx);
            Vec r = s.r;
            mv(1.0, s.R, false, v, 1.0, r);
            if (k >= 1) mv(1.0, s.M, true, Vec(o.dxi.begin() + xo(k), o.dxi.begin() + xo(k) + nx), 1.0, r);
            mv(-1.0, s.Ju, true, mk, 1.0, r);
            r[0] += nu[k] - nl[k];
            rs[uo(k)] = r[0];
            Vec d(o.dxi.begin() + xo(k + 1), o.dxi.begin() + xo(k + 1) + nx);
            for (int i = 0; i < nx; ++i) d[i] += -1.0 * s.b[i];
            if (k >= 1) mv(-1.0, s.Jx, false, Vec(o.dxi.begin() + xo(k), o.dxi.begin() + xo(k) + nx), 1.0, d);
            mv(-1.0, s.Ju, false, v, 1.0, d);
            for (int i = 0; i < nx; ++i) rd[k * nx + i] = d[i];
        }
        for (int k = 1; k <= N; ++k) {
            const Stage& s = st[k];
            Vec x = s.q;
            mv(1.0, s.Q, false, Vec(o.dxi.begin() + xo(k), o.dxi.begin() + xo(k) + nx), 1.0, x);
            if (k < N) {
                mv(1.0, s.M, false, Vec{o.dxi[uo(k)]}, 1.0, x);
                mv(-1.0, s.Jx, true, Vec(o.mu.begin() + k * nx, o.mu.begin() + (k + 1) * nx), 1.0, x);
            }
            for (int i = 0; i < nx; ++i) x[i] += o.mu[(k - 1) * nx + i];
            for (int i = 0; i < nx; ++i) rs[xo(k) + i] = x[i];
        }
        for (int k = 0; k < N; ++k) {
            const double v = o.dxi[uo(k)];
            rl[k] = fl[k] ? v - sl[k] - st[k].lb : 0.0;
            ru[k] = fu[k] ? st[k].ub - v - su[k] : 0.0;
        }
    };
    auto csolve = [&](const Factor& f, Vec& dxi, Vec& dmu) {  // qp.cpp:288-305
        Vec rh(N);
        std::vector<Vec> qh(N + 1), bh(N);
        for (int k = 0; k < N; ++k) {
            double v = rs[uo(k)];
            if (fl[k]) v -= (cl[k] - nl[k] * rl[k]) / sl[k];
            if (fu[k]) v += (cu[k] - nu[k] * ru[k]) / su[k];
            rh[k] = v;
            bh[k].assign(rd.begin() + k * nx, rd.begin() + (k + 1) * nx);
            for (double& x : bh[k]) x = -x;
        }
        for (int k = 1; k <= N; ++k) qh[k].assign(rs.begin() + xo(k), rs.begin() + xo(k) + nx);
        rsolve(st, N, nx, f, rh, qh, bh, dxi, dmu);
    };
    auto expand = [&](const Vec& dxi) {  // qp.cpp:308-317
        for (int k = 0; k < N; ++k) {
            const double dv = dxi[uo(k)];
            dsl[k] = fl[k] ? dv + rl[k] : 0.0;
            dsu[k] = fu[k] ? ru[k] - dv : 0.0;
            dnl[k] = fl[k] ? (cl[k] - nl[k] * dsl[k]) / sl[k] : 0.0;
            dnu[k] = fu[k] ? (cu[k] - nu[k] * dsu[k]) / su[k] : 0.0;
        }
    };
    auto step = [&](double frac) {  // qp.cpp:321-337
        double a = 1.0;
        auto cap = [&](double val, double dir) {
            if (dir < 0.0) a = std::min(a, -frac * val / dir);
        };
        for (int k = 0; k < N; ++k) {
            if (fl[k]) cap(sl[k], dsl[k]), cap(nl[k], dnl[k]);
            if (fu[k]) cap(su[k], dsu[k]), cap(nu[k], dnu[k]);
        }
        return a;
    };
    Vec dxi, dmu;
    for (int it = 0;; ++it) {
        resid();
        const double gap = m > 0 ? (dotv(sl, nl) + dotv(su, nu)) / m : 0.0;
        if (ninf(rs) <= eps && ninf(rd) <= eps && ninf(rl) <= eps && ninf(ru) <= eps && gap <= eps) {
            o.status = 0;
            break;
        }
        if (it >= max_iter) {
            o.status = 1;
            break;
        }
        Vec bar(N, 0.0);
        for (int k = 0; k < N; ++k) {
            if (fl[k]) bar[k] += nl[k] / sl[k];
            if (fu[k]) bar[k] += nu[k] / su[k];
        }
        Factor f;
        try {
            f = rfactor(st, N, nx, bar);
        } catch (const NotPD&) {
            o.status = 2;
            break;
        }
        for (int k = 0; k < N; ++k) {
            cl[k] = fl[k] ? -sl[k] * nl[k] : 0.0;
            cu[k] = fu[k] ? -su[k] * nu[k] : 0.0;
        }
        csolve(f, dxi, dmu);
        expand(dxi);
        double sig = 0.0;
        if (m > 0 && gap > 0.0) {
            const double aa = step(1.0);
            double ga = 0.0;
            for (int k = 0; k < N; ++k) {
                if (fl[k]) ga += (sl[k] + aa * dsl[k]) * (nl[k] + aa * dnl[k]);
                if (fu[k]) ga += (su[k] + aa * dsu[k]) * (nu[k] + aa * dnu[k]);
            }
            ga /= m;
            const double ratio = std::max(0.0, ga / gap);
            sig = std::min(1.0, ratio * ratio * ratio);
        }
        for (int k = 0; k < N; ++k) {
            if (fl[k]) cl[k] = sig * gap - sl[k] * nl[k] - dsl[k] * dnl[k];
            if (fu[k]) cu[k] = sig * gap - su[k] * nu[k] - dsu[k] * dnu[k];
        }
        csolve(f, dxi, dmu);
        expand(dxi);
        const double a = step(0.995);
        for (size_t i = 0; i < dxi.size(); ++i) o.dxi[i] += a * dxi[i];
        for (size_t i = 0; i < dmu.size(); ++i) o.mu[i] += a * dmu[i];
        for (int k = 0; k < N; ++k) {
            if (fl[k]) sl[k] += a * dsl[k], nl[k] += a * dnl[k];
            if (fu[k]) su[k] += a * dsu[k], nu[k] += a * dnu[k];
        }
        PORT_UNIT(IPM, N);
    }
    for (int k = 0; k < N; ++k) {
        double& v = o.dxi[uo(k)];
        v = std::min(std::max(v, st[k].lb), st[k].ub);
    }
    o.nl = nl;
    o.nu = nu;
    return o;
}

// -------------------------------------------------------------------- SQP
struct Duals {
    Vec lam, pl, pu;
};

/// h += J_g' lam (add_constraint_term, sqp.cpp:102-116).
static void add_jt(const Nlp& q, const Blocks& cb, const Vec& lam, Vec& h) {
    for (int k = 0; k < q.N; ++k) {
        const double* l = lam.data() + k * q.nx;
        for (int i = 0; i < q.nx; ++i) h[q.xo(k + 1) + i] += l[i];
        for (int j = 0; j < q.nx; ++j) h[q.uo(k)] -= cb.Fu[k].at(j, 0) * l[j];
        if (k >= 1)
            for (int i = 0; i < q.nx; ++i)
                for (int j = 0; j < q.nx; ++j) h[q.xo(k) + i] -= cb.Fx[k].at(j, i) * l[j];
    }
}
static Vec lag_grad(const Nlp& q, const Vec& gf, const Blocks& cb, const Duals& d) {  // sqp.cpp:118-128
    Vec h = gf;
    add_jt(q, cb, d.lam, h);
    for (int k = 0; k < q.N; ++k) h[q.uo(k)] += d.pu[k] - d.pl[k];
    return h;
}
static bool kkt_ok(const Vec& gl, const Vec& g, const Duals& d, int m, double eps) {  // sqp.cpp:86-96
    double sd = 1.0;
    if (m > 0) sd = std::max(100.0, (n1(d.lam) + n1(d.pl) + n1(d.pu)) / m) / 100.0;
    return ninf(gl) / sd <= eps && ninf(g) <= eps;
}

/// Damped BFGS on one block (bfgs_block_update, sqp.cpp:61-84). NotPD on
/// loss of definiteness.
static void bfgs(Mat& W, const Vec& s, const Vec& y) {
    const double tiny = std::numeric_limits<double>::epsilon();
    Vec Ws;
    mv(1.0, W, false, s, 0.0, Ws);
    const double sWs = dotv(s, Ws);
    if (!(sWs > tiny)) return;
    const double sy = dotv(s, y);
    const double th = sy >= 0.2 * sWs ? 1.0 : 0.8 * sWs / (sWs - sy);
    Vec r(s.size());
    for (size_t i = 0; i < s.size(); ++i) r[i] = th * y[i] + (1.0 - th) * Ws[i];
    const double sr = dotv(s, r);
    if (!(std::min(sWs, sr) > tiny)) return;
    for (int j = 0; j < W.c; ++j)
        for (int i = 0; i < W.r; ++i) W.at(i, j) += r[i] * r[j] / sr - Ws[i] * Ws[j] / sWs;
    sym(W);
    chol(W, false);
}

static void identity_blocks(std::vector<Mat>& W, int N, int nx) {  // reset_blocks, sqp.cpp:173-178
    W.assign(N + 1, Mat());
    W[0] = Mat::eye(1);
    for (int k = 1; k < N; ++k) W[k] = Mat::eye(nx + 1);
    W[N] = Mat::eye(nx);
}

/// build_stages (sqp.cpp:130-171).
static std::vector<Stage> stages(const Nlp& q, const std::vector<Mat>& W, const Vec& gf, const Blocks& cb,
                                 const Vec& xi) {
    const int nx = q.nx;
    std::vector<Stage> st(q.N + 1);
    for (int k = 0; k < q.N; ++k) {
        Stage& s = st[k];
        if (k == 0) {
            s.R = W[0];
        } else {
            s.Q = Mat(nx, nx);
            s.M = Mat(nx, 1);
            s.R = Mat(1, 1);
            for (int j = 0; j < nx; ++j)
                for (int i = 0; i < nx; ++i) s.Q.at(i, j) = W[k].at(i, j);
            for (int i = 0; i < nx; ++i) s.M.at(i, 0) = W[k].at(i, nx);
            s.R.at(0, 0) = W[k].at(nx, nx);
            s.q.assign(gf.begin() + q.xo(k), gf.begin() + q.xo(k) + nx);
        }
        s.r = Vec{gf[q.uo(k)]};
        s.Jx = cb.Fx[k];
        s.Ju = cb.Fu[k];
        s.b = cb.b[k];
        s.lb = q.umin - xi[q.uo(k)];
        s.ub = q.umax - xi[q.uo(k)];
    }
    st[q.N].Q = W[q.N];
    st[q.N].q.assign(gf.begin() + q.xo(q.N), gf.begin() + q.xo(q.N) + nx);
    return st;
}

struct SqpRes {
    Vec xi;
    Duals d;
    bool converged = false;
};

/// sqp_solve (sqp.cpp:182-411); opts per SqpOptions (sqp.hpp:50-58).
static SqpRes sqp(const Nlp& q, Vec xi, Duals d, const nmpcmc_sqp_options& op) {
    PORT_PHASE(SQP);
    const int nx = q.nx, N = q.N;
    const int m = N * nx + (std::isfinite(q.umin) ? N : 0) + (std::isfinite(q.umax) ? N : 0);
    SqpRes out;
    out.xi = xi;
    out.d = d;
    std::vector<Mat> W;
    identity_blocks(W, N, nx);
    Vec gf, sig;
    double f;
    Blocks cb;
    try {
        f = objective(q, out.xi, &gf);
        cb = constraints(q, out.xi);
    } catch (const NonFinite&) {
        return out;
    }
    bool first = true;
    for (int it = 0;; ++it) {
        const Vec gl = lag_grad(q, gf, cb, out.d);
        if (kkt_ok(gl, cb.g, out.d, m, op.eps)) {
            out.converged = true;
            break;
        }
        if (it >= op.max_iter) break;
        PORT_UNIT(SQP, N);
        QpOut qp = solve_qp(stages(q, W, gf, cb, out.xi), N, nx, op.qp_tol, op.qp_max_iter);
        if (qp.status == 2) {
            identity_blocks(W, N, nx);
            qp = solve_qp(stages(q, W, gf, cb, out.xi), N, nx, op.qp_tol, op.qp_max_iter);
            if (qp.status == 2) break;
        }
        const Duals fresh{qp.mu, qp.nl, qp.nu};
        if (kkt_ok(lag_grad(q, gf, cb, fresh), cb.g, fresh, m, op.eps)) {
            out.d = fresh;
            out.converged = true;
            break;
        }
        // merit_weights_update (sqp.cpp:12-20)
        if (first) sig.assign(qp.mu.size(), 0.0);
        for (size_t i = 0; i < qp.mu.size(); ++i) {
            const double am = std::fabs(qp.mu[i]);
            sig[i] = first ? am : std::max(am, 0.5 * (sig[i] + am));
        }
        first = false;
        // line_search (sqp.cpp:22-59)
        double pen = 0.0;
        for (size_t i = 0; i < cb.g.size(); ++i) pen += sig[i] * std::fabs(cb.g[i]);
        const double m0 = f + pen;
        const double dd = dotv(gf, qp.dxi) - pen;
        double a = 1.0, merit = 0.0;
        bool ok = false;
        Vec trial(out.xi.size());
        for (int bt = 0;; ++bt) {
            for (size_t i = 0; i < trial.size(); ++i) trial[i] = out.xi[i] + a * qp.dxi[i];
            merit = std::numeric_limits<double>::infinity();
            try {
                const double ft = objective(q, trial, nullptr);
                const Blocks ct = constraints(q, trial);
                merit = ft;
                for (size_t i = 0; i < ct.g.size(); ++i) merit += sig[i] * std::fabs(ct.g[i]);
            } catch (const NonFinite&) {
            }
            ok = std::isfinite(merit) && merit <= m0 + op.c1 * a * dd;
            if (ok || bt >= op.max_backtracks) break;
            a *= op.backtrack_factor;
        }
        if (!ok && !std::isfinite(merit)) break;
        Vec xn(out.xi.size());
        for (size_t i = 0; i < xn.size(); ++i) xn[i] = out.xi[i] + a * qp.dxi[i];
        Vec gfn;
        double fn;
        Blocks cbn;
        try {
            fn = objective(q, xn, &gfn);
            cbn = constraints(q, xn);
        } catch (const NonFinite&) {
            break;
        }
        out.xi = xn;
        for (size_t i = 0; i < out.d.lam.size(); ++i) out.d.lam[i] += a * (qp.mu[i] - out.d.lam[i]);
        for (size_t i = 0; i < out.d.pl.size(); ++i) {
            out.d.pl[i] += a * (qp.nl[i] - out.d.pl[i]);
            out.d.pu[i] += a * (qp.nu[i] - out.d.pu[i]);
        }
        Vec ho = gf, hn = gfn;
        add_jt(q, cb, out.d.lam, ho);
        add_jt(q, cbn, out.d.lam, hn);
        bool lost = false;
        for (int blk = 0; blk <= N && !lost; ++blk) {
            const int off = blk == 0 ? 0 : (blk < N ? q.xo(blk) : q.xo(N));
            const int len = blk == 0 ? 1 : (blk < N ? nx + 1 : nx);
            Vec s(len), y(len);
            for (int i = 0; i < len; ++i) {
                s[i] = a * qp.dxi[off + i];
                y[i] = hn[off + i] - ho[off + i];
            }
            try {
                bfgs(W[blk], s, y);
            } catch (const NotPD&) {
                lost = true;
            }
        }
        if (lost) identity_blocks(W, N, nx);
        f = fn;
        gf = gfn;
        cb = cbn;
    }
    return out;
}

// -------------------------------------------------------------- controllers
/// NMPC controller state (controllers.hpp:54-65).
struct Nmpc {
    Cstr model;
    Vec xhat;
    Mat P;
    Vec last_xi;
    Duals last;
};

/// nmpc_step (controllers.cpp:114-212). Returns the applied input; sets *conv.
static double nmpc_step(Nmpc& s, const nmpcmc_scenario& sc, double t, double y, const Vec& sp, bool* conv) {
    if (!std::isfinite(y)) throw NonFinite{};
    Vec xf = s.xhat;
    Mat Pf = s.P;
    try {
        ekf_update(s.model, xf, Pf, y, sc.R_filter);
    } catch (const NotPD&) {
        xf = s.xhat;
        Pf = s.P;
        ekf_update(s.model, xf, Pf, y, sc.R_filter + 1e-10);
    }
    Nlp q{&s.model, sc.N, sc.Nc, s.model.nx, sc.horizon_Ts, t, sc.u_min, sc.u_max, sc.Qz, xf, sp};
    const int N = q.N, nx = q.nx;
    Vec xi0;
    Duals d0{Vec(static_cast<size_t>(N) * nx, 0.0), Vec(N, 0.0), Vec(N, 0.0)};
    auto clampu = [&](double u) { return std::max(q.umin, std::min(q.umax, u)); };
    if (static_cast<int>(s.last_xi.size()) == q.size()) {
        Vec us(N);
        for (int k = 0; k < N; ++k) us[k] = clampu(s.last_xi[q.uo(std::min(k + 1, N - 1))]);
        try {
            xi0 = xi_from_u(q, us);
        } catch (const NonFinite&) {
            const int w = q.stride();
            xi0.assign(s.last_xi.size(), 0.0);
            std::copy(s.last_xi.begin() + w, s.last_xi.end(), xi0.begin());
            std::copy(s.last_xi.end() - w, s.last_xi.end(), xi0.end() - w);
            for (int k = 0; k < N; ++k) xi0[q.uo(k)] = clampu(xi0[q.uo(k)]);
        }
        auto shift = [](const Vec& v, int blk) {
            if (v.size() < static_cast<size_t>(2 * blk)) return v;
            Vec o(v.size());
            std::copy(v.begin() + blk, v.end(), o.begin());
            std::copy(v.end() - blk, v.end(), o.end() - blk);
            return o;
        };
        d0.lam = shift(s.last.lam, nx);
        d0.pl = shift(s.last.pl, 1);
        d0.pu = shift(s.last.pu, 1);
        for (int k = 0; k < N; ++k) d0.pl[k] = std::max(0.0, d0.pl[k]), d0.pu[k] = std::max(0.0, d0.pu[k]);
    } else {
        const double un = std::isfinite(q.umin) && std::isfinite(q.umax) ? 0.5 * (q.umin + q.umax) : clampu(0.0);
        try {
            xi0 = xi_from_u(q, Vec(N, un));
        } catch (const NonFinite&) {
            xi0.assign(q.size(), 0.0);
            for (int k = 0; k < N; ++k) {
                xi0[q.uo(k)] = un;
                for (int i = 0; i < nx; ++i) xi0[q.xo(k + 1) + i] = xf[i];
            }
        }
    }
    const SqpRes r = sqp(q, xi0, d0, sc.sqp);
    const double u = clampu(r.xi[q.uo(0)]);
    s.last_xi = r.xi;
    s.last = r.d;
    ekf_predict(s.model, xf, Pf, u, t, t + sc.horizon_Ts, sc.np);
    s.xhat = xf;
    s.P = Pf;
    *conv = r.converged;
    return u;
}

static double sp_at(const nmpcmc_scenario& sc, double t) {  // SetpointProfile::at, montecarlo.cpp:26-32
    const PORT_REAL* e = std::upper_bound(sc.sp_times, sc.sp_times + sc.n_setpoints, t);
    return sc.sp_values[(e - sc.sp_times) - 1];
}

/// run_closed_loop (montecarlo.cpp:80-157) + the catch(...) of the
/// run_monte_carlo worker (montecarlo.cpp:226-236).
static void closed_loop(const nmpcmc_scenario& sc, uint64_t idx, nmpcmc_sim_record* rec, double* traj, int rows) {
    const double nan = std::numeric_limits<double>::quiet_NaN();
    nmpcmc_cstr_params tp = sc.truth;
    if (sc.perturb) {  // include/nmpcmc_gpu.h perturbation rule
        Rng pr(sc.base_seed, idx | 0x8000000000000000ULL);
        const double z0 = pr.normal(), z1 = pr.normal(), z2 = pr.normal();
        tp.cA_in = PORT_TO_DOUBLE(tp.cA_in * (1.0 + sc.perturb_rel_std[0] * z0));
        tp.cB_in = PORT_TO_DOUBLE(tp.cB_in * (1.0 + sc.perturb_rel_std[1] * z1));
        tp.EaR = PORT_TO_DOUBLE(tp.EaR * (1.0 + sc.perturb_rel_std[2] * z2));
    }
    const Cstr truth(tp, sc.truth_variant);
    const int nbar = static_cast<int>(std::llround((sc.tf - sc.t0) / sc.Ts));
    Rng rng(sc.base_seed, idx);
    const bool nm = sc.controller == NMPCMC_CTRL_NMPC;
    Nmpc ctl{Cstr(sc.ctrl, sc.ctrl_variant), {}, {}, {}, {}};
    if (nm) {
        const int n = ctl.model.nx;
        ctl.xhat.assign(sc.x0_hat, sc.x0_hat + n);
        ctl.P = Mat(n, n);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) ctl.P.at(i, j) = sc.P0[j * n + i];
    }
    double Ihat = sc.pi.I_hat;
    const int stride = std::max(1, sc.record_stride);
    if (traj)
        for (int i = 0; i < rows * 5; ++i) traj[i] = nan;
    int row = 0, solves = 0, fails = 0;
    Vec x(sc.x0, sc.x0 + truth.nx);
    double t = sc.t0;
    double z = truth.out(x), zb = sp_at(sc, t);
    double acc = 0.0;
    try {
        {
            const double r = z - zb;
            acc += r * r;
        }
        for (int i = 0; i < nbar; ++i) {
            const double y = measure(truth, sc.has_noise_R != 0, sc.noise_R, x, rng);
            double u;
            if (nm) {
                Vec sp(sc.N);
                for (int k = 1; k <= sc.N; ++k) sp[k - 1] = sp_at(sc, t + k * sc.Ts);
                bool conv = false;
                u = nmpc_step(ctl, sc, t, y, sp, &conv);
                PORT_UNIT(STEP, 1);
                ++solves;
                if (!conv) ++fails;
            } else {  // pi_step (controllers.cpp:12-23)
                const double e = sp_at(sc, t) - y;
                const double P = sc.pi.kP * e;
                const double I = Ihat + sc.Ts * sc.pi.kI * e;
                const double uh = sc.pi.u_bar + P + I;
                u = std::max(sc.u_min, std::min(sc.u_max, uh));
                Ihat = I + sc.Ts * sc.pi.kaw * (uh - u);
            }
            if (traj && i % stride == 0) {
                double* w = traj + row * 5;
                w[0] = t, w[1] = z, w[2] = zb, w[3] = u, w[4] = y;
                ++row;
            }
            x = simulate(truth, t, t + sc.Ts, x, u, sc.Ns, rng);
            t = sc.t0 + (i + 1) * sc.Ts;
            z = truth.out(x);
            zb = sp_at(sc, t);
            const double r = z - zb;
            acc += r * r;
        }
        rec->phi = PORT_TO_DOUBLE(acc / static_cast<double>(nbar + 1));
        rec->failed = 0;
        if (traj) {
            double* w = traj + row * 5;
            w[0] = t, w[1] = z, w[2] = zb;
        }
        rec->ocp_solves = solves;
        rec->ocp_failures = fails;
        rec->status = 0;
    } catch (const NonFinite&) {
        *rec = {PORT_TO_DOUBLE(nan), 1, solves, fails, NMPCMC_NON_FINITE_STATE};
    } catch (const Domain&) {
        *rec = {PORT_TO_DOUBLE(nan), 1, solves, fails, NMPCMC_DOMAIN_ERROR};
    } catch (const NotPD&) {  // escapes run_closed_loop; the worker's catch(...) zeroes the record
        *rec = {PORT_TO_DOUBLE(nan), 1, 0, 0, NMPCMC_NOT_POSITIVE_DEFINITE};
    }
}

}  // namespace port

#ifndef PORT_NO_CAPI
extern "C" {

int PFX(run_closed_loop)(const nmpcmc_scenario* sc, uint64_t idx, nmpcmc_sim_record* out, double* traj, int rows) {
    port::closed_loop(*sc, idx, out, traj, rows);
    return 0;
}

int PFX(run_batch)(const nmpcmc_scenario* sc, uint64_t first, int64_t n, int workers, nmpcmc_sim_record* out,
                   double* wall) {
    std::atomic<int64_t> next{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int w = 0; w < std::max(1, static_cast<int>(std::min<int64_t>(workers, n))); ++w)
        pool.emplace_back([&]() {
            for (int64_t i; (i = next.fetch_add(1)) < n;) port::closed_loop(*sc, first + i, &out[i], nullptr, 0);
        });
    for (auto& th : pool) th.join();
    if (wall) *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
}

void PFX(normals)(uint64_t seed, uint64_t stream, int64_t n, double* out) {
    port::Rng r(seed, stream);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
}

void PFX(philox_block)(const uint32_t* in, uint32_t* out) { port::Rng::block(in, in[4], in[5], out); }

}  // extern "C"
#endif  // PORT_NO_CAPI
