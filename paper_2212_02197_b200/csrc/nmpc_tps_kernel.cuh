// nmpc_tps_kernel.cuh -- K3b: NMPC closed loop, one THREAD per sample.
//
// Same restatement of the reference's NMPC branch as nmpc_kernel.cuh (see the
// file:line map there; every per-stage expression is shared or written in the
// same operation order), but each sample is a single thread: the serial
// recursions (Riccati sweeps, ordered reductions, forward shooting) then run
// on 32 samples per warp instruction instead of one, and the per-sample
// workspace moves from shared memory to a coalesced structure-of-arrays in
// global memory:  element (array a, stage k) of resident slot s lives at
// ws[(a * ST + k) * pitch + s], so a warp touches 256 contiguous bytes per
// access. Resident slots = grid threads; each thread walks the samples
// slot, slot + T, ... of the launch (grid-stride), so the workspace is sized
// by the resident thread count, not by the batch.
//
// Lanes of a warp run different samples and diverge in SQP / IPM / line-search
// iteration counts; SIMT serialises the divergent parts. Results do not
// depend on the mapping: everything a sample computes is a function of its
// own (seed, index) only.
#pragma once

#include "nmpc_kernel.cuh"

namespace nmpcmc_dev {

/// Thread-local view of the SoA workspace.
template <int ST>
struct TW {
    double* b;     // ws + slot
    long long p;   // pitch (resident slots)
    __device__ __forceinline__ double* arr(int a) const { return b + (long long)a * ST * p; }
};

#define TA(a, k) (w.arr(a)[(long long)(k) * w.p])

/// eval_objective (ocp.cpp:76-99): phi in k order, gradient on x slots.
template <int ST>
__device__ __noinline__ double t_eval_objective(const Ocp& o, const TW<ST>& w, int xid, int gid) {
    const double ts = o.Ts;
    double phi = 0.0;
    for (int k = 0; k < o.N; ++k) {
        const double res = TA(xid, k) / o.p.V - TA(A_SP, k);
        const double qres = epi0(dot1(o.Qz, res));
        phi += ts * dot1(res, qres);
        const double gx = epi0(dot1(o.inv_V, qres));
        TA(gid, k) = 0.0 + 2.0 * ts * gx;
    }
    return phi;
}

/// eval_constraints (ocp.cpp:101-135): stops at the first failing shoot, like
/// the exception in the reference. Block (g, Jx, Ju) at ids (gid, gid+1, gid+2).
template <int ST>
__device__ __noinline__ int t_eval_constraints(const Ocp& o, const TW<ST>& w, int uid, int xid, int gid,
                                               Cnt* cnt) {
    double xk = o.x0;
    for (int k = 0; k < o.N; ++k) {
        double F, Sx, Su;
        const int st = shoot1<true>(o.p, xk, TA(uid, k), o.h, o.Nc, F, Sx, Su);
        if (st) {
            cnt->shoot_full += k + 1;
            return st;
        }
        const double next = TA(xid, k);
        TA(gid, k) = next - F;
        TA(gid + 1, k) = Sx;
        TA(gid + 2, k) = Su;
        xk = next;
    }
    cnt->shoot_full += o.N;
    return ST_OK;
}

/// xi_from_inputs (ocp.cpp:137-154).
template <int ST>
__device__ __noinline__ int t_xi_from_inputs(const Ocp& o, const TW<ST>& w, int uid, int xid, Cnt* cnt) {
    double xk = o.x0;
    for (int k = 0; k < o.N; ++k) {
        double F, Sx, Su;
        const int st = shoot1<false>(o.p, xk, TA(uid, k), o.h, o.Nc, F, Sx, Su);
        if (st) {
            cnt->shoot_fonly += k + 1;
            return st;
        }
        TA(xid, k) = F;
        xk = F;
    }
    cnt->shoot_fonly += o.N;
    return ST_OK;
}

/// expand (qp.cpp:308-317) of stage k from the step in DDU.
template <int ST>
__device__ __forceinline__ Dir t_expand(const TW<ST>& w, int k, bool fl, bool fu, double rl, double ru) {
    const double dv = TA(A_DDU, k);
    Dir d;
    d.dsl = fl ? dv + rl : 0.0;
    d.dsu = fu ? ru - dv : 0.0;
    d.dnl = fl ? (TA(A_RCL, k) - TA(A_NL, k) * d.dsl) / TA(A_SL, k) : 0.0;
    d.dnu = fu ? (TA(A_RCU, k) - TA(A_NU, k) * d.dsu) / TA(A_SU, k) : 0.0;
    return d;
}

/// Forward rollout (qp.cpp:142-155) into DDU, DDX, DDMU.
template <int ST>
__device__ __noinline__ void t_rollout(const TW<ST>& w, int N, int jxid, int juid) {
    double dx = 0.0;
    for (int k = 0; k < N; ++k) {
        double du = TA(A_DFF, k);
        if (k >= 1) du = epi1(dot1(TA(A_GAIN, k), dx), du);
        TA(A_DDU, k) = du;
        double dxn = -TA(A_RDYN, k);
        if (k >= 1) dxn = epi1(dot1(TA(jxid, k), dx), dxn);
        dxn = epi1(dot1(TA(juid, k), du), dxn);
        dx = dxn;
        TA(A_DDX, k) = dx;
        const double mm = epi1(dot1(TA(A_VAL, k + 1), dx), TA(A_PVEC, k + 1));
        TA(A_DDMU, k) = -mm;
    }
}

/// Backward vector sweep of riccati_solve_vectors (qp.cpp:122-141) with the
/// cached factor; FACTOR = true also computes riccati_factor (qp.cpp:73-110)
/// on the way (fused, same per-stage operation order). Returns true on
/// NotPositiveDefinite.
template <int ST, bool FACTOR>
__device__ __noinline__ bool t_sweep(const TW<ST>& w, int N, int jxid, int juid) {
    double P = TA(A_WQ, N);
    double pv = TA(A_RSX, N - 1);
    if (FACTOR) TA(A_VAL, N) = P;
    TA(A_PVEC, N) = pv;
    for (int k = N - 1; k >= 0; --k) {
        const double ju = TA(juid, k);
        double l;
        if (FACTOR) {
            const double pju = epi0(dot1(P, ju));
            double hh = epi0(dot1(ju, pju));
            hh = hh + TA(A_WR, k);
            hh = hh + TA(A_BAR, k);
            if (hh <= 0.0 || !dfinite(hh)) return true;
            l = sqrt(hh);
            TA(A_CHOLH, k) = l;
        } else {
            P = TA(A_VAL, k + 1);
            l = TA(A_CHOLH, k);
        }
        const double tmpv = epi1(dot1(P, -TA(A_RDYN, k)), pv);
        double hv = epi1(dot1(ju, tmpv), TA(A_RHAT, k));
        hv = hv / l;
        hv = hv / l;
        hv = -hv;
        TA(A_DFF, k) = hv;
        if (k >= 1) {
            const double jx = TA(jxid, k);
            double gg;
            if (FACTOR) {
                const double pjx = epi0(dot1(P, jx));
                gg = epi0(dot1(ju, pjx));
                gg = gg + TA(A_WM, k);
                double gn = gg / l;
                gn = gn / l;
                const double gk = -gn;
                double pn = epi0(dot1(jx, pjx));
                pn = pn + TA(A_WQ, k);
                pn = epi1(dot1(gg, gk), pn);
                TA(A_VAL, k) = pn;
                TA(A_GAIN, k) = gk;
                TA(A_GMAT, k) = gg;
                P = pn;
            } else {
                gg = TA(A_GMAT, k);
            }
            double pvn = epi1(dot1(jx, tmpv), TA(A_RSX, k - 1));
            pvn = epi1(dot1(gg, hv), pvn);
            TA(A_PVEC, k) = pvn;
            pv = pvn;
        }
    }
    return false;
}

/// solve_qp (qp.cpp:173-423), one thread; data as in nmpc_kernel.cuh solve_qp.
/// (gxid, gid, jxid, juid) = current evaluation block.
template <int ST>
__device__ __noinline__ int t_solve_qp(const Ocp& o, const TW<ST>& w, int gxid, int gid, int jxid, int juid,
                                       double tol, int max_iter, Cnt* cnt) {
    const int N = o.N;
    const double tau = 0.995;
    double ds = 1.0;
    int m = 0;
    for (int k = 0; k < N; ++k) {
        const double u = TA(A_U, k);
        const double lb = o.umin - u, ub = o.umax - u;
        if (lb > ub) return QP_DOMAIN;
        const bool fl = dfinite(lb), fu = dfinite(ub);
        if (fl) {
            ++m;
            ds = smax(ds, fabs(lb));
        }
        if (fu) {
            ++m;
            ds = smax(ds, fabs(ub));
        }
        ds = smax(ds, fold_absmax(0.0, 0.0));
        ds = smax(ds, fold_absmax(0.0, bneg(TA(gid, k))));
        TA(A_DU, k) = 0.0;
        TA(A_DX, k) = 0.0;
        TA(A_MU, k) = 0.0;
        TA(A_SL, k) = fl ? smax(1.0, fabs(lb)) : 0.0;
        TA(A_NL, k) = fl ? 1.0 : 0.0;
        TA(A_SU, k) = fu ? smax(1.0, fabs(ub)) : 0.0;
        TA(A_NU, k) = fu ? 1.0 : 0.0;
        TA(A_RCL, k) = 0.0;
        TA(A_RCU, k) = 0.0;
    }
    for (int k = 0; k < N; ++k) ds = smax(ds, fold_absmax(0.0, TA(gxid, k)));
    const double eps = tol * ds;

    auto rlru = [&](int k, double u, bool fl, bool fu, double& rl, double& ru) {
        const double v = TA(A_DU, k);
        rl = fl ? v - TA(A_SL, k) - (o.umin - u) : 0.0;
        ru = fu ? (o.umax - u) - v - TA(A_SU, k) : 0.0;
    };

    int status = QP_MAXITER;
    for (int iter = 0;; ++iter) {
        // residuals() (qp.cpp:237-284); r_stat norm covers u rows and x rows
        double ninf = 0.0, dinf = 0.0, linf = 0.0, uinf = 0.0;
        double dl = 0.0, du_ = 0.0;  // gap chains: dot(sl, nl), dot(su, nu)
        for (int k = 0; k < N; ++k) {
            const double ju = TA(juid, k);
            const double vk = TA(A_DU, k), muk = TA(A_MU, k);
            double r = epi1(dot1(TA(A_WR, k), vk), 0.0);
            if (k >= 1) r = epi1(dot1(TA(A_WM, k), TA(A_DX, k - 1)), r);
            r = epim1(dot1(ju, muk), r);
            r += TA(A_NU, k) - TA(A_NL, k);
            TA(A_RSU, k) = r;
            double rd = TA(A_DX, k) + -1.0 * bneg(TA(gid, k));
            if (k >= 1) rd = epim1(dot1(TA(jxid, k), TA(A_DX, k - 1)), rd);
            rd = epim1(dot1(ju, vk), rd);
            TA(A_RDYN, k) = rd;
            const int kk = k + 1;
            double rx = epi1(dot1(TA(A_WQ, kk), TA(A_DX, k)), TA(gxid, k));
            if (kk < N) {
                rx = epi1(dot1(TA(A_WM, kk), TA(A_DU, kk)), rx);
                rx = epim1(dot1(TA(jxid, kk), TA(A_MU, kk)), rx);
            }
            rx += muk;
            TA(A_RSX, k) = rx;
            const double u = TA(A_U, k);
            const bool fl = dfinite(o.umin - u), fu = dfinite(o.umax - u);
            double rl, ru;
            rlru(k, u, fl, fu, rl, ru);
            ninf = fold_absmax(fold_absmax(ninf, r), rx);
            dinf = fold_absmax(dinf, rd);
            linf = fold_absmax(linf, rl);
            uinf = fold_absmax(uinf, ru);
            dl += TA(A_SL, k) * TA(A_NL, k);
            du_ += TA(A_SU, k) * TA(A_NU, k);
        }
        const double gap = m > 0 ? (dl + du_) / m : 0.0;
        if (ninf <= eps && dinf <= eps && linf <= eps && uinf <= eps && gap <= eps) {
            status = QP_OPTIMAL;
            break;
        }
        if (iter >= max_iter) {
            status = QP_MAXITER;
            break;
        }
        for (int k = 0; k < N; ++k) {
            const double u = TA(A_U, k);
            const bool fl = dfinite(o.umin - u), fu = dfinite(o.umax - u);
            const double sl = TA(A_SL, k), su = TA(A_SU, k), nl = TA(A_NL, k), nu = TA(A_NU, k);
            double bk = 0.0;
            if (fl) bk += nl / sl;
            if (fu) bk += nu / su;
            TA(A_BAR, k) = bk;
            const double cl = fl ? -sl * nl : 0.0;
            const double cu = fu ? -su * nu : 0.0;
            TA(A_RCL, k) = cl;
            TA(A_RCU, k) = cu;
            double rl, ru;
            rlru(k, u, fl, fu, rl, ru);
            double v = TA(A_RSU, k);
            if (fl) v -= (cl - nl * rl) / sl;
            if (fu) v += (cu - nu * ru) / su;
            TA(A_RHAT, k) = v;
        }
        if (t_sweep<ST, true>(w, N, jxid, juid)) {
            status = QP_FAILED;
            break;
        }
        t_rollout<ST>(w, N, jxid, juid);
        double sigma = 0.0;
        {
            double alpha_aff = 1.0;
            for (int k = 0; k < N; ++k) {
                const double u = TA(A_U, k);
                const bool fl = dfinite(o.umin - u), fu = dfinite(o.umax - u);
                double rl, ru;
                rlru(k, u, fl, fu, rl, ru);
                const Dir d = t_expand<ST>(w, k, fl, fu, rl, ru);
                if (fl) {
                    if (d.dsl < 0.0) alpha_aff = smin(alpha_aff, -1.0 * TA(A_SL, k) / d.dsl);
                    if (d.dnl < 0.0) alpha_aff = smin(alpha_aff, -1.0 * TA(A_NL, k) / d.dnl);
                }
                if (fu) {
                    if (d.dsu < 0.0) alpha_aff = smin(alpha_aff, -1.0 * TA(A_SU, k) / d.dsu);
                    if (d.dnu < 0.0) alpha_aff = smin(alpha_aff, -1.0 * TA(A_NU, k) / d.dnu);
                }
            }
            if (m > 0 && gap > 0.0) {
                double gap_aff = 0.0;
                for (int k = 0; k < N; ++k) {
                    const double u = TA(A_U, k);
                    const bool fl = dfinite(o.umin - u), fu = dfinite(o.umax - u);
                    double rl, ru;
                    rlru(k, u, fl, fu, rl, ru);
                    const Dir d = t_expand<ST>(w, k, fl, fu, rl, ru);
                    if (fl) gap_aff += (TA(A_SL, k) + alpha_aff * d.dsl) * (TA(A_NL, k) + alpha_aff * d.dnl);
                    if (fu) gap_aff += (TA(A_SU, k) + alpha_aff * d.dsu) * (TA(A_NU, k) + alpha_aff * d.dnu);
                }
                gap_aff /= m;
                const double ratio = smax(0.0, gap_aff / gap);
                sigma = smin(1.0, ratio * ratio * ratio);
            }
        }
        for (int k = 0; k < N; ++k) {
            const double u = TA(A_U, k);
            const bool fl = dfinite(o.umin - u), fu = dfinite(o.umax - u);
            double rl, ru;
            rlru(k, u, fl, fu, rl, ru);
            const Dir d = t_expand<ST>(w, k, fl, fu, rl, ru);
            const double sl = TA(A_SL, k), su = TA(A_SU, k), nl = TA(A_NL, k), nu = TA(A_NU, k);
            double cl = TA(A_RCL, k), cu = TA(A_RCU, k);
            if (fl) cl = sigma * gap - sl * nl - d.dsl * d.dnl;
            if (fu) cu = sigma * gap - su * nu - d.dsu * d.dnu;
            TA(A_RCL, k) = cl;
            TA(A_RCU, k) = cu;
            double v = TA(A_RSU, k);
            if (fl) v -= (cl - nl * rl) / sl;
            if (fu) v += (cu - nu * ru) / su;
            TA(A_RHAT, k) = v;
        }
        t_sweep<ST, false>(w, N, jxid, juid);
        t_rollout<ST>(w, N, jxid, juid);
        double alpha = 1.0;
        for (int k = 0; k < N; ++k) {
            const double u = TA(A_U, k);
            const bool fl = dfinite(o.umin - u), fu = dfinite(o.umax - u);
            double rl, ru;
            rlru(k, u, fl, fu, rl, ru);
            const Dir d = t_expand<ST>(w, k, fl, fu, rl, ru);
            if (fl) {
                if (d.dsl < 0.0) alpha = smin(alpha, -tau * TA(A_SL, k) / d.dsl);
                if (d.dnl < 0.0) alpha = smin(alpha, -tau * TA(A_NL, k) / d.dnl);
            }
            if (fu) {
                if (d.dsu < 0.0) alpha = smin(alpha, -tau * TA(A_SU, k) / d.dsu);
                if (d.dnu < 0.0) alpha = smin(alpha, -tau * TA(A_NU, k) / d.dnu);
            }
            TA(A_BAR, k) = d.dsl;  // stash the corrector directions
            TA(A_RHAT, k) = d.dnl;
            TA(A_RCL, k) = d.dsu;
            TA(A_RCU, k) = d.dnu;
        }
        for (int k = 0; k < N; ++k) {
            const double u = TA(A_U, k);
            const bool fl = dfinite(o.umin - u), fu = dfinite(o.umax - u);
            TA(A_DU, k) = TA(A_DU, k) + alpha * TA(A_DDU, k);
            TA(A_DX, k) = TA(A_DX, k) + alpha * TA(A_DDX, k);
            TA(A_MU, k) = TA(A_MU, k) + alpha * TA(A_DDMU, k);
            if (fl) {
                TA(A_SL, k) += alpha * TA(A_BAR, k);
                TA(A_NL, k) += alpha * TA(A_RHAT, k);
            }
            if (fu) {
                TA(A_SU, k) += alpha * TA(A_RCL, k);
                TA(A_NU, k) += alpha * TA(A_RCU, k);
            }
        }
        cnt->ipm_stage += N;
    }
    for (int k = 0; k < N; ++k) {
        const double u = TA(A_U, k);
        const double lb = o.umin - u, ub = o.umax - u;
        TA(A_DU, k) = smin(smax(TA(A_DU, k), lb), ub);
    }
    return status;
}

/// check_convergence (sqp.cpp:86-96) of the Lagrangian gradient at the
/// evaluation block (gxid, gid, jxid, juid) with multipliers (lid, plid, puid).
template <int ST>
__device__ __noinline__ bool t_kkt_check(const TW<ST>& w, int N, int gxid, int gid, int jxid, int juid, int lid,
                                         int plid, int puid, int m, double eps) {
    double gl = 0.0, gi = 0.0, n1 = 0.0, n2 = 0.0, n3 = 0.0;
    double lam_k = TA(lid, 0);
    for (int k = 0; k < N; ++k) {
        const double lam_n = (k + 1 < N) ? TA(lid, k + 1) : 0.0;
        const double pl = TA(plid, k), pu = TA(puid, k);
        const double hu = (0.0 - TA(juid, k) * lam_k) + (pu - pl);
        double hx = TA(gxid, k) + lam_k;
        if (k + 1 < N) hx -= TA(jxid, k + 1) * lam_n;
        gl = fold_absmax(fold_absmax(gl, hu), hx);
        gi = fold_absmax(gi, TA(gid, k));
        n1 += fabs(lam_k);
        n2 += fabs(pl);
        n3 += fabs(pu);
        lam_k = lam_n;
    }
    double s_d = 1.0;
    if (m > 0) {
        const double mults = n1 + n2 + n3;
        s_d = smax(100.0, mults / m) / 100.0;
    }
    return gl / s_d <= eps && gi <= eps;
}

template <int ST>
__device__ __forceinline__ void t_reset_blocks(const TW<ST>& w, int N) {
    for (int k = 0; k <= N; ++k) {
        TA(A_WQ, k) = 1.0;
        TA(A_WM, k) = 0.0;
        TA(A_WR, k) = 1.0;
    }
}

/// add_constraint_term pieces (sqp.cpp:102-116) at stage k for eval block (gx, jx, ju).
template <int ST>
__device__ __forceinline__ double t_lag_u(const TW<ST>& w, int juid, int k) {
    return 0.0 - TA(juid, k) * TA(A_LAM, k);
}
template <int ST>
__device__ __forceinline__ double t_lag_x(const TW<ST>& w, int gxid, int jxid, int k, int N) {
    double h = TA(gxid, k) + TA(A_LAM, k);
    if (k + 1 < N) h -= TA(jxid, k + 1) * TA(A_LAM, k + 1);
    return h;
}

/// One SQP iteration after the QP: merit weights, line search, acceptance,
/// BFGS (sqp.cpp:312-406). cur/trial = evaluation block base ids (gX first,
/// then g, Jx, Ju consecutively... see EvalIds). Returns 0 continue, 1 break,
/// ST_DOMAIN << 4 DomainError.
struct EvalIds {
    int gx, g;  // g, g+1 (Jx), g+2 (Ju)
};

template <int ST>
__device__ __noinline__ int t_sqp_step(const Ocp& o, const TW<ST>& w, const nmpcmc_sqp_options& opt, double* f,
                                       bool first_merit, EvalIds* cur, EvalIds* trial, Cnt* cnt) {
    const int N = o.N;
    const int gxc = cur->gx, gc = cur->g, jxc = gc + 1, juc = gc + 2;
    const int gxt = trial->gx, gt = trial->g, jxt = gt + 1, jut = gt + 2;
    double penalty0 = 0.0, dot_gd = 0.0;
    bool du_bad = false;
    for (int k = 0; k < N; ++k) {
        const double am = fabs(TA(A_MU, k));
        const double sg = first_merit ? am : smax(am, 0.5 * (TA(A_SIG, k) + am));
        TA(A_SIG, k) = sg;
        penalty0 += sg * fabs(TA(gc, k));
        const double duk = TA(A_DU, k);
        du_bad |= !dfinite(duk);
        dot_gd += TA(gxc, k) * TA(A_DX, k);
    }
    if (du_bad) dot_gd = kNaN;
    const double dd = dot_gd - penalty0;
    const double merit_before = *f + penalty0;
    double alpha = 1.0, merit = 0.0, f_trial = 0.0;
    bool ok = false;
    for (int bt = 0;; ++bt) {
        for (int k = 0; k < N; ++k) {
            TA(A_DDU, k) = TA(A_U, k) + alpha * TA(A_DU, k);
            TA(A_DDX, k) = TA(A_X, k) + alpha * TA(A_DX, k);
        }
        f_trial = t_eval_objective<ST>(o, w, A_DDX, gxt);
        const int st = t_eval_constraints<ST>(o, w, A_DDU, A_DDX, gt, cnt);
        if (st == ST_DOMAIN) return ST_DOMAIN << 4;
        merit = HUGE_VAL;
        if (st == ST_OK) {
            merit = f_trial;
            for (int k = 0; k < N; ++k) merit += TA(A_SIG, k) * fabs(TA(gt, k));
        }
        cnt->ls += 1;
        ok = dfinite(merit) && merit <= merit_before + opt.c1 * alpha * dd;
        if (ok || bt >= opt.max_backtracks) break;
        alpha *= opt.backtrack_factor;
    }
    if (!ok && !dfinite(merit)) return 1;
    const double a = alpha;
    for (int k = 0; k < N; ++k) {
        TA(A_U, k) = TA(A_DDU, k);
        TA(A_X, k) = TA(A_DDX, k);
        TA(A_LAM, k) += a * (TA(A_MU, k) - TA(A_LAM, k));
        TA(A_PIL, k) += a * (TA(A_NL, k) - TA(A_PIL, k));
        TA(A_PIU, k) += a * (TA(A_NU, k) - TA(A_PIU, k));
    }
    bool lost = false;
    for (int blk = 0; blk <= N && !lost; ++blk) {
        double s[2], y[2];
        int n;
        bool uonly = false;
        if (blk == 0) {
            n = 1;
            uonly = true;
            s[0] = a * TA(A_DU, 0);
            y[0] = t_lag_u<ST>(w, jut, 0) - t_lag_u<ST>(w, juc, 0);
        } else if (blk < N) {
            n = 2;
            s[0] = a * TA(A_DX, blk - 1);
            s[1] = a * TA(A_DU, blk);
            y[0] = t_lag_x<ST>(w, gxt, jxt, blk - 1, N) - t_lag_x<ST>(w, gxc, jxc, blk - 1, N);
            y[1] = t_lag_u<ST>(w, jut, blk) - t_lag_u<ST>(w, juc, blk);
        } else {
            n = 1;
            s[0] = a * TA(A_DX, N - 1);
            y[0] = t_lag_x<ST>(w, gxt, jxt, N - 1, N) - t_lag_x<ST>(w, gxc, jxc, N - 1, N);
        }
        double q = TA(A_WQ, blk), mm = TA(A_WM, blk), r = TA(A_WR, blk);
        const int res = bfgs_block(q, mm, r, n, s, y, uonly);
        if (res < 0) lost = true;
        if (res > 0) {
            TA(A_WQ, blk) = q;
            TA(A_WM, blk) = mm;
            TA(A_WR, blk) = r;
        }
    }
    if (lost) t_reset_blocks<ST>(w, N);
    // the trial evaluation becomes the current one: swap the block ids
    const EvalIds t = *cur;
    *cur = *trial;
    *trial = t;
    *f = f_trial;
    cnt->sqp += 1;
    return 0;
}

/// sqp_solve (sqp.cpp:182-411).
template <int ST>
__device__ __noinline__ SqpOut t_sqp_solve(const Ocp& o, const TW<ST>& w, const nmpcmc_sqp_options& opt,
                                           Cnt* cnt) {
    const int N = o.N;
    SqpOut out{false, ST_OK};
    const int m = N + (dfinite(o.umin) ? N : 0) + (dfinite(o.umax) ? N : 0);
    t_reset_blocks<ST>(w, N);
    bool first_merit = true;
    EvalIds cur{A_GX, A_G}, trial{A_TGX, A_TG};
    double f = t_eval_objective<ST>(o, w, A_X, cur.gx);
    const int st = t_eval_constraints<ST>(o, w, A_U, A_X, cur.g, cnt);
    if (st == ST_DOMAIN) return SqpOut{false, ST_DOMAIN};
    if (st == ST_NONFINITE) return out;
    for (int iter = 0;; ++iter) {
        if (t_kkt_check<ST>(w, N, cur.gx, cur.g, cur.g + 1, cur.g + 2, A_LAM, A_PIL, A_PIU, m, opt.eps)) {
            out.converged = true;
            break;
        }
        if (iter >= opt.max_iter) break;
        cnt->sqp_stage += N;
        int qs = QP_FAILED;
        for (int attempt = 0; attempt < 2; ++attempt) {
            if (attempt == 1) t_reset_blocks<ST>(w, N);
            qs = t_solve_qp<ST>(o, w, cur.gx, cur.g, cur.g + 1, cur.g + 2, opt.qp_tol, opt.qp_max_iter, cnt);
            cnt->qp += 1;
            if (qs != QP_FAILED) break;
        }
        if (qs == QP_DOMAIN) return SqpOut{false, ST_DOMAIN};
        if (qs == QP_FAILED) break;
        if (t_kkt_check<ST>(w, N, cur.gx, cur.g, cur.g + 1, cur.g + 2, A_MU, A_NL, A_NU, m, opt.eps)) {
            for (int k = 0; k < N; ++k) {
                TA(A_LAM, k) = TA(A_MU, k);
                TA(A_PIL, k) = TA(A_NL, k);
                TA(A_PIU, k) = TA(A_NU, k);
            }
            out.converged = true;
            break;
        }
        const int r = t_sqp_step<ST>(o, w, opt, &f, first_merit, &cur, &trial, cnt);
        first_merit = false;
        if (r == (ST_DOMAIN << 4)) return SqpOut{false, ST_DOMAIN};
        if (r == 1) break;
    }
    return out;
}

/// Warm/cold start (controllers.cpp:147-186).
template <int ST>
__device__ __noinline__ int t_start_iterate(const Ocp& o, const TW<ST>& w, bool warm, Cnt* cnt) {
    const int N = o.N;
    const bool fl = dfinite(o.umin), fh = dfinite(o.umax);
    const double u_nom = fl && fh ? 0.5 * (o.umin + o.umax) : smax(o.umin, smin(o.umax, 0.0));
    for (int k = 0; k < N; ++k)
        TA(A_DDU, k) = warm ? smax(o.umin, smin(o.umax, TA(A_U, min(k + 1, N - 1)))) : u_nom;
    const int st = t_xi_from_inputs<ST>(o, w, A_DDU, A_DDX, cnt);
    if (st == ST_DOMAIN) return ST_DOMAIN;
    if (st == ST_OK) {
        for (int k = 0; k < N; ++k) {
            TA(A_U, k) = TA(A_DDU, k);
            TA(A_X, k) = TA(A_DDX, k);
        }
    } else if (warm) {
        for (int k = 0; k < N; ++k) {  // shifted_warm_start, in place (reads ahead)
            TA(A_U, k) = TA(A_DDU, k);
            TA(A_X, k) = TA(A_X, min(k + 1, N - 1));
        }
    } else {
        for (int k = 0; k < N; ++k) {
            TA(A_U, k) = u_nom;
            TA(A_X, k) = o.x0;
        }
    }
    if (warm) {
        if (N >= 2)
            for (int k = 0; k < N; ++k) {  // shifted_multipliers, in place (reads ahead)
                const int src = min(k + 1, N - 1);
                TA(A_LAM, k) = TA(A_LAM, src);
                TA(A_PIL, k) = TA(A_PIL, src);
                TA(A_PIU, k) = TA(A_PIU, src);
            }
        for (int k = 0; k < N; ++k) {
            TA(A_PIL, k) = smax(0.0, TA(A_PIL, k));
            TA(A_PIU, k) = smax(0.0, TA(A_PIU, k));
        }
    } else {
        for (int k = 0; k < N; ++k) {
            TA(A_LAM, k) = 0.0;
            TA(A_PIL, k) = 0.0;
            TA(A_PIU, k) = 0.0;
        }
    }
    return ST_OK;
}

/// run_closed_loop NMPC branch for one sample on one thread.
template <int NX, int ST>
__device__ __noinline__ void t_closed_loop(const nmpcmc_scenario& sc, uint64_t sim_index, int nbar,
                                           const TW<ST>& w, nmpcmc_sim_record* rec, nmpcmc_work_counters* cntp,
                                           double* traj) {
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
    const int N = o.N;
    Cnt cnt = {};
    double xhat = sc.x0_hat[0], Pf = sc.P0[0];
    bool have_last = false;
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
        if (!dfinite(y)) {
            status = ST_NONFINITE;
            break;
        }
        for (int k = 0; k < N; ++k) TA(A_SP, k) = setpoint_at(sc, t + (k + 1) * sc.Ts);
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
        if (t_start_iterate<ST>(o, w, have_last, &cnt) == ST_DOMAIN) {
            status = ST_DOMAIN;
            break;
        }
        const SqpOut so = t_sqp_solve<ST>(o, w, sc.sqp, &cnt);
        if (so.status != ST_OK) {
            status = so.status;
            break;
        }
        const double u = smax(o.umin, smin(o.umax, TA(A_U, 0)));
        have_last = true;
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
        if (record && i % stride == 0) {
            double* rw = traj + (size_t)row * 5;
            rw[0] = t;
            rw[1] = z;
            rw[2] = zbar;
            rw[3] = u;
            rw[4] = y;
            ++row;
        }
        status = simulate_interval<NX>(p, pl, t, t + sc.Ts, u, sc.Ns, rng);
        if (status != ST_OK) break;
        t = sc.t0 + (i + 1) * sc.Ts;
        z = pl.x[NX - 1] / p.V;
        zbar = setpoint_at(sc, t);
        const double r = z - zbar;
        acc += r * r;
    }
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

/// Grid-stride over the launch's samples; thread = resident slot.
template <int NX, int ST>
__global__ void __launch_bounds__(64) nmpc_tps_kernel(const __grid_constant__ nmpcmc_scenario sc, uint64_t first_sim,
                                                      int64_t n_sims, int nbar, nmpcmc_sim_record* records,
                                                      nmpcmc_work_counters* counters, double* traj, int traj_rows,
                                                      double* ws, int64_t pitch) {
    const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (slot >= pitch) return;
    const TW<ST> w{ws + slot, pitch};
    for (int64_t i = slot; i < n_sims; i += pitch)
        t_closed_loop<NX, ST>(sc, first_sim + (uint64_t)i, nbar, w, records + i, counters ? counters + i : nullptr,
                              traj ? traj + (size_t)i * traj_rows * 5 : nullptr);
}

/// Workspace bytes for `slots` resident threads.
inline size_t tps_ws_bytes(int N, int64_t slots) {
    return (size_t)kWsArrays * ws_stride_for(N) * sizeof(double) * (size_t)slots;
}

template <int NX, int ST>
inline void launch_tps_t(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
                         nmpcmc_work_counters* d_cnt, double* d_traj, int rows, double* ws, int64_t slots,
                         cudaStream_t stream) {
    const int block = 64;
    const unsigned grid = (unsigned)((slots + block - 1) / block);
    nmpc_tps_kernel<NX, ST><<<grid, block, 0, stream>>>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, ws, slots);
}

inline int launch_nmpc_tps(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
                           nmpcmc_work_counters* d_cnt, double* d_traj, int rows, double* ws, int64_t slots,
                           cudaStream_t stream) {
    if (sc.ctrl_variant != NMPCMC_ONE_STATE) return NMPCMC_UNSUPPORTED;
    if (sc.N < 1 || sc.N > 255) return NMPCMC_UNSUPPORTED;
    const int ST = ws_stride_for(sc.N);
    const bool three = sc.truth_variant == NMPCMC_THREE_STATE;
#define NMPCMC_TPS_CASE(S)                                                                             \
    if (ST == S) {                                                                                    \
        if (three) launch_tps_t<3, S>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, ws, slots, stream); \
        else launch_tps_t<1, S>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, ws, slots, stream);      \
        return NMPCMC_OK;                                                                             \
    }
    NMPCMC_TPS_CASE(32)
    NMPCMC_TPS_CASE(64)
    NMPCMC_TPS_CASE(128)
    NMPCMC_TPS_CASE(256)
#undef NMPCMC_TPS_CASE
    return NMPCMC_UNSUPPORTED;
}

#undef TA

}  // namespace nmpcmc_dev
