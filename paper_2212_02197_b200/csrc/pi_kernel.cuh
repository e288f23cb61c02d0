// pi_kernel.cuh -- K2: PI closed loop, one thread per sample.
//
// Restates run_closed_loop's PI branch (montecarlo.cpp:80-157) with pi_step
// (controllers.cpp:12-23), measure / simulate_interval (model.cpp:26-48) and
// phi_metric (montecarlo.cpp:65-78; accumulated on the fly in the same index
// order). The whole 720-step loop lives in registers; per-sample I/O is one
// 24-byte record. Parallelism is across samples only: each sample is a serial
// recursion in time. The state-independent normals (31 per
// control step: Philox + log + sincos, the bulk of the arithmetic) are
// generated a window of 16 Box-Muller pairs at a time into shared memory --
// 16 independent chains the scheduler overlaps -- so only the Euler-Maruyama
// recursion itself stays serial.
#pragma once

#include "certified_math.cuh"
#include "device_common.cuh"

namespace nmpcmc_dev {

/// pi_step (controllers.cpp:12-23) in the documented order:
///   e = ybar - y, P = kP e, I = I_hat + Ts kI e, u_hat = u_bar + P + I,
///   u = max(u_min, min(u_max, u_hat)), I_aw = Ts kaw (u_hat - u),
///   next.I_hat = I + I_aw.
__device__ __forceinline__ nmpcmc_pi_step_result pi_law(const nmpcmc_pi_state& s, double y, double ybar) {
    nmpcmc_pi_step_result r;
    r.e = ybar - y;
    r.P = s.kP * r.e;
    r.I = s.I_hat + s.Ts * s.kI * r.e;
    r.u_hat = s.u_bar + r.P + r.I;
    r.u = smax(s.u_min, smin(s.u_max, r.u_hat));
    r.I_aw = s.Ts * s.kaw * (r.u_hat - r.u);
    r.next_I_hat = r.I + r.I_aw;
    return r;
}

/// Batched pi_step: instance i maps (states[i], y[i], ybar[i]) to
/// results[i] (may be null) and adopts result.next into states[i].
__global__ void pi_step_kernel(nmpcmc_pi_state* states, const double* y, const double* ybar, int64_t n,
                               nmpcmc_pi_step_result* results) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        nmpcmc_pi_state s = states[i];
        const nmpcmc_pi_step_result r = pi_law(s, y[i], ybar[i]);
        if (results != nullptr) results[i] = r;
        s.I_hat = r.next_I_hat;
        states[i] = s;
    }
}

/// Pairs of normals generated ahead per window refill (one control step
/// consumes 1 + Ns * NX normals: 31 in every BASELINE config, one refill).
constexpr int kPiPairs = 16;
constexpr int kPiBlock = 128;
/// Lanes per sample: the group splits each window refill (Philox + log +
/// sincos, the bulk of the work) and runs the Euler-Maruyama recursion in
/// lockstep, so a batch of n samples fills n * kPiLanes threads.
#ifndef NMPCMC_PI_LANES
#define NMPCMC_PI_LANES 4
#endif
#ifndef NMPCMC_PI_MINB
#define NMPCMC_PI_MINB 1
#endif
constexpr int kPiLanes = NMPCMC_PI_LANES;

template <int NX, int G>
__device__ void pi_closed_loop(const nmpcmc_scenario& sc, uint64_t sim_index, int nbar,
                               nmpcmc_sim_record* rec, nmpcmc_work_counters* cnt, double* traj,
                               int traj_rows, double* win_buf, int win_stride) {
    const Cstr p = sample_truth(sc, sim_index);
    NormalWindow<kPiPairs, G> rng;
    // writes the outputs (rec == nullptr: a tail group's stand-in)
    const bool lead = (G == 1 || (threadIdx.x & (G - 1)) == 0) && rec != nullptr;
    rng.init(win_buf, win_stride, sc.base_seed, sim_index);
    const int per_step = (sc.has_noise_R != 0 ? 1 : 0) + sc.Ns * NX;
    Plant<NX> pl;
#pragma unroll
    for (int i = 0; i < NX; ++i) pl.x[i] = sc.x0[i];
    const bool has_R = sc.has_noise_R != 0;
    const double lR = has_R ? chol_semidef_1x1(sc.noise_R) : 0.0;
    // run_closed_loop copies the gains and takes Ts/bounds from the scenario
    // (montecarlo.cpp:97-100)
    const double kP = sc.pi.kP, kI = sc.pi.kI, kaw = sc.pi.kaw, u_bar = sc.pi.u_bar;
    const double Ts = sc.Ts, u_min = sc.u_min, u_max = sc.u_max;
    double I_hat = sc.pi.I_hat;
    const int stride = sc.record_stride < 1 ? 1 : sc.record_stride;
    const bool record = traj != nullptr;

    double t = sc.t0;
    double z = pl.x[NX - 1] / p.V;        // output (model.cpp:50-52)
    double zbar = setpoint_at(sc, t);
    double acc = 0.0;
    {
        const double r = z - zbar;
        acc += r * r;
    }
    int status = ST_OK;
    int row = 0;
    int steps = 0;  // control steps entered (a failing step counts: its work ran)
    // only the measurement and temperature normals are read when the plant
    // has no diffusion on c_A, c_B (simulate_interval<.., true>)
    const bool sparse = NX == 3 && p.sigmaA == 0.0 && p.sigmaB == 0.0 && per_step < 2 * kPiPairs;
    for (int i = 0; i < nbar; ++i) {
        if (sparse) {
            // a live sample's stream position at the start of step i is
            // exactly i * per_step (warp-uniform, as below)
            if (G > 1 && __all_sync(0xffffffffu, status != ST_OK)) break;
            rng.fill_sparse((uint64_t)i * (uint64_t)per_step, has_R ? 1 : 0, sc.Ns);
            if (status != ST_OK) continue;
        } else if (G > 1) {
            // lockstep over the warp: a live sample's stream position at the
            // start of step i is exactly i * per_step, so every group refills
            // at the same steps; a failed sample idles until its warp is done
            if (__all_sync(0xffffffffu, status != ST_OK)) break;
            rng.k = (uint64_t)i * (uint64_t)per_step;
            rng.reserve(per_step);
            if (status != ST_OK) continue;
        } else if (per_step < 2 * kPiPairs) {
            rng.reserve(per_step);  // this step's normals in one refill
        }
        ++steps;
        const double y = measure<NX>(p, pl, has_R, lR, rng);
        // pi_step (controllers.cpp:12-23), evaluated in the documented order
        const double ybar = setpoint_at(sc, t);
        const nmpcmc_pi_state ps{kP, kI, kaw, Ts, u_bar, u_min, u_max, I_hat};
        const nmpcmc_pi_step_result pr = pi_law(ps, y, ybar);
        const double u = pr.u;
        I_hat = pr.next_I_hat;
        if (record && i % stride == 0) {
            if (lead) {
                double* rw = traj + (size_t)row * 5;
                rw[0] = t;
                rw[1] = z;
                rw[2] = zbar;
                rw[3] = u;
                rw[4] = y;
            }
            ++row;
        }
        status = sparse ? simulate_interval<NX, NormalWindow<kPiPairs, G>, true>(p, pl, t, t + sc.Ts, u, sc.Ns, rng)
                        : simulate_interval<NX>(p, pl, t, t + sc.Ts, u, sc.Ns, rng);
        if (status != ST_OK) {
            if (G == 1) break;
            continue;
        }
        t = sc.t0 + (i + 1) * sc.Ts;
        z = pl.x[NX - 1] / p.V;
        zbar = setpoint_at(sc, t);
        const double r = z - zbar;
        acc += r * r;
    }
    if (!lead) return;
    if (status == ST_OK) {
        rec->phi = acc / (double)(nbar + 1);
        rec->failed = 0;
        if (record) {
            double* rw = traj + (size_t)row * 5;
            rw[0] = t;
            rw[1] = z;
            rw[2] = zbar;
            rw[3] = __longlong_as_double(0x7ff8000000000000LL);
            rw[4] = __longlong_as_double(0x7ff8000000000000LL);
        }
    } else {
        rec->phi = __longlong_as_double(0x7ff8000000000000LL);
        rec->failed = 1;
    }
    rec->ocp_solves = 0;
    rec->ocp_failures = 0;
    rec->status = status;
    if (cnt != nullptr) {
        nmpcmc_work_counters c = {};
        c.control_steps = steps;
        *cnt = c;
    }
    (void)traj_rows;
}

/// G consecutive threads per sample (a group of one warp); the group's normal
/// window lives in shared memory, element j of group q at
/// win[j * (kPiBlock / G) + q] (conflict-free across groups, a broadcast
/// within one).
template <int NX, int G>
__global__ void __launch_bounds__(kPiBlock, NMPCMC_PI_MINB) pi_kernel(const __grid_constant__ nmpcmc_scenario sc,
                                                      uint64_t first_sim, int64_t n_sims, int nbar,
                                                      nmpcmc_sim_record* records,
                                                      nmpcmc_work_counters* counters, double* traj,
                                                      int traj_rows) {
    constexpr int kGroups = kPiBlock / G;
    __shared__ double win[2 * kPiPairs * kGroups];
    const int q = threadIdx.x / G;
    const int64_t i = (int64_t)blockIdx.x * kGroups + q;
    if (G == 1) {
        if (i >= n_sims) return;
    } else {
        // a warp runs its groups in lockstep: warps past the end leave, the
        // tail groups of the last warp run a copy of the last sample unseen
        const int64_t w0 = (int64_t)blockIdx.x * kGroups + (threadIdx.x & ~31) / G;
        if (w0 >= n_sims) return;
    }
    const bool real = i < n_sims;
    const int64_t ii = real ? i : n_sims - 1;
    pi_closed_loop<NX, G>(sc, first_sim + (uint64_t)ii, nbar, real ? records + ii : nullptr,
                          counters && real ? counters + ii : nullptr,
                          traj && real ? traj + (size_t)ii * traj_rows * 5 : nullptr, traj_rows, win + q, kGroups);
}

// ---------------------------------------------- warp-specialised PI (K2ws)
// One consumer warp runs 32 samples' closed loops (one thread per sample,
// the serial Euler-Maruyama chain); P producer warps of the same block
// generate the normals those 32 samples read, one control step at a time,
// into a ring of kPiWsSlots shared-memory slots. The normals do not depend
// on the state (a live sample's stream position at step i is i * per_step),
// so producers run ahead of the consumer by up to kPiWsSlots steps and the
// Philox + log + sincos work, the bulk of the arithmetic, overlaps the
// latency-bound recursion instead of sitting on it. Slot s of step i holds
// normal m of sample l at [m * 32 + l]: the consumer's reads are
// conflict-free, and a producer warp writes one m for 32 samples.
// Handshake: named barriers FULL(s) = 1 + s (producers arrive, consumer
// syncs) and EMPTY(s) = 1 + kPiWsSlots + s (consumer arrives, producers sync).
constexpr int kPiWsSlots = 3;
constexpr int kPiWsMaxPerStep = 40;  // normals read per control step (40 KB ring)

/// Normal source of one consumer lane: the current slot's column.
struct SlotRng {
    const double* p;
    __device__ __forceinline__ double normal() {
        const double z = *p;
        p += 32;
        return z;
    }
    __device__ __forceinline__ void skip() {}
};

// Barrier ids are immediates (a switch over the slot), so ptxas reserves only
// the 2 kPiWsSlots + 1 barriers in use: a register id makes it reserve all
// 16, and the SM's barrier budget then caps residency at 4 blocks per SM
// (measured: 1.58 waves at config 1 instead of one).
template <int ID>
__device__ __forceinline__ void bar_sync_id(int n) {
    asm volatile("bar.sync %0, %1;" ::"n"(ID), "r"(n) : "memory");
}
template <int ID>
__device__ __forceinline__ void bar_arrive_id(int n) {
    asm volatile("bar.arrive %0, %1;" ::"n"(ID), "r"(n) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
    static_assert(kPiWsSlots == 3, "one case per barrier id");
    switch (id) {
        case 1: bar_sync_id<1>(n); break;
        case 2: bar_sync_id<2>(n); break;
        case 3: bar_sync_id<3>(n); break;
        case 4: bar_sync_id<4>(n); break;
        case 5: bar_sync_id<5>(n); break;
        default: bar_sync_id<6>(n); break;
    }
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    switch (id) {
        case 1: bar_arrive_id<1>(n); break;
        case 2: bar_arrive_id<2>(n); break;
        case 3: bar_arrive_id<3>(n); break;
        case 4: bar_arrive_id<4>(n); break;
        case 5: bar_arrive_id<5>(n); break;
        default: bar_arrive_id<6>(n); break;
    }
}

/// Normals a control step reads (SPARSE: the measurement one and the c_T
/// increment of every substep; else all per_step of them).
__host__ __device__ inline int pi_ws_reads(const nmpcmc_scenario& sc, bool sparse) {
    const int nx = sc.truth_variant == NMPCMC_THREE_STATE ? 3 : 1;
    const int has_R = sc.has_noise_R != 0 ? 1 : 0;
    return sparse ? has_R + sc.Ns : has_R + sc.Ns * nx;
}

/// The plant drift (cstr.cpp:36-53) with the divisions by the constant
/// volume V as Markstein corrections on the per-sample reciprocal
/// yV = RN(1/V) (3 dependent operations instead of an IEEE division on the
/// Euler-Maruyama chain). Each quotient's certificate (cert_div: the exact
/// fma residual proves it is RN(n / V)) is folded into ok; the caller
/// replays the control step with IEEE divisions unless every one held, so
/// the states are bitwise those of drift3 / drift1.
template <int NX>
__device__ __forceinline__ int drift_fv(const Cstr& p, const double* n, double u, double* dn, double yV, bool& ok) {
    const double f = u * kMlMinToLs;
    if (NX == 3) {
        const double c0 = fast_div(n[0], p.V, yV), c1 = fast_div(n[1], p.V, yV), c2 = fast_div(n[2], p.V, yV);
        ok &= cert_div_bf(n[0], p.V, c0) & cert_div_bf(n[1], p.V, c1) & cert_div_bf(n[2], p.V, c2);
        if (c2 <= 0.0) return ST_DOMAIN;
        const double r = p.k0 * xlibm_exp(-p.EaR / c2) * c0 * c1;
        dn[0] = p.cA_in * f - c0 * f + -1.0 * r * p.V;
        dn[1] = p.cB_in * f - c1 * f + -2.0 * r * p.V;
        dn[2] = p.cT_in * f - c2 * f + p.beta * r * p.V;
        return ST_OK;
    }
    const double c = fast_div(n[0], p.V, yV);
    ok &= cert_div_bf(n[0], p.V, c);
    const Conc1 cc = conc1(p, c);
    if (cc.cT <= 0.0) return ST_DOMAIN;
    const double r = p.k0 * xlibm_exp(-p.EaR / cc.cT) * cc.cA * cc.cB;
    dn[0] = p.cT_in * f - c * f + p.beta * r * p.V;
    return ST_OK;
}

template <int NX, int P, bool SPARSE>
__global__ void __launch_bounds__(32 * (1 + P), P == 3 ? 7 : 3) pi_ws_kernel(const __grid_constant__ nmpcmc_scenario sc,
                                                             uint64_t first_sim, int64_t n_sims, int nbar,
                                                             nmpcmc_sim_record* records,
                                                             nmpcmc_work_counters* counters, double* traj,
                                                             int traj_rows) {
    extern __shared__ double ring[];
    __shared__ int stop;
    constexpr int kThreads = 32 * (1 + P);
    const int lane = threadIdx.x & 31;
    const int64_t base = (int64_t)blockIdx.x * 32;
    const int has_R = sc.has_noise_R != 0 ? 1 : 0;
    const int per_step = has_R + sc.Ns * NX;
    const int reads = SPARSE ? has_R + sc.Ns : per_step;
    const int items = reads * 32;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();

    if (threadIdx.x >= 32) {
        // ---- producers: item j of a slot is normal j >> 5 of sample j & 31
        const int t = threadIdx.x - 32;
        for (int i = 0; i < nbar; ++i) {
            const int s = i % kPiWsSlots;
            if (i >= kPiWsSlots) named_sync(1 + kPiWsSlots + s, kThreads);
            if (*(volatile int*)&stop == 0) {
                double* slot = ring + s * items;
                const uint64_t k0 = (uint64_t)i * (uint64_t)per_step;
                for (int j = t; j < items; j += 32 * P) {
                    const int m = j >> 5;
                    int64_t idx = base + (j & 31);
                    if (idx >= n_sims) idx = n_sims - 1;  // tail lanes run a copy, unseen
                    const uint64_t nn =
                        SPARSE ? (has_R && m == 0 ? k0 : k0 + (uint64_t)(has_R + 3 * (m - has_R) + 2)) : k0 + m;
                    slot[j] = normal_one(sc.base_seed, first_sim + (uint64_t)idx, nn);
                }
            }
            named_arrive(1 + s, kThreads);
        }
        return;
    }

    // ---- consumer: run_closed_loop's PI branch, as pi_closed_loop<NX, 1>
    const int64_t ig = base + lane;
    const bool real = ig < n_sims;
    const int64_t ii = real ? ig : n_sims - 1;
    const uint64_t sim_index = first_sim + (uint64_t)ii;
    const Cstr p = sample_truth(sc, sim_index);
    Plant<NX> pl;
#pragma unroll
    for (int q = 0; q < NX; ++q) pl.x[q] = sc.x0[q];
    const bool hasR = has_R != 0;
    const double lR = hasR ? chol_semidef_1x1(sc.noise_R) : 0.0;
    const double yV = 1.0 / p.V;
    const double kP = sc.pi.kP, kI = sc.pi.kI, kaw = sc.pi.kaw, u_bar = sc.pi.u_bar;
    const double Ts = sc.Ts, u_min = sc.u_min, u_max = sc.u_max;
    double I_hat = sc.pi.I_hat;
    const int stride = sc.record_stride < 1 ? 1 : sc.record_stride;
    double* tr = (traj != nullptr && real) ? traj + (size_t)ii * traj_rows * 5 : nullptr;

    double t = sc.t0;
    double z = pl.x[NX - 1] / p.V;
    double zbar = setpoint_at(sc, t);
    double acc = 0.0;
    {
        const double r = z - zbar;
        acc += r * r;
    }
    int status = ST_OK;
    int row = 0;
    int steps = 0;
    for (int i = 0; i < nbar; ++i) {
        const int s = i % kPiWsSlots;
        named_sync(1 + s, kThreads);
        if (status == ST_OK) {
            SlotRng rng{ring + s * items + lane};
            ++steps;
            const double y = measure<NX>(p, pl, hasR, lR, rng);
            const double ybar = setpoint_at(sc, t);
            const nmpcmc_pi_state ps{kP, kI, kaw, Ts, u_bar, u_min, u_max, I_hat};
            const nmpcmc_pi_step_result pr = pi_law(ps, y, ybar);
            const double u = pr.u;
            I_hat = pr.next_I_hat;
            if (tr != nullptr && i % stride == 0) {
                double* rw = tr + (size_t)row * 5;
                rw[0] = t;
                rw[1] = z;
                rw[2] = zbar;
                rw[3] = u;
                rw[4] = y;
                ++row;
            }
            // fast divisions by V; the step is replayed with IEEE ones from
            // the saved state unless every quotient was certified
            const Plant<NX> pl0 = pl;
            const SlotRng rng0 = rng;
            bool ok = true;
            status = simulate_interval_d<NX, SlotRng, SPARSE>(
                p, pl, t, t + sc.Ts, u, sc.Ns, rng,
                [&](const double* x, double uu, double* dn) -> int { return drift_fv<NX>(p, x, uu, dn, yV, ok); });
            if (!ok) {
                pl = pl0;
                rng = rng0;
                status = simulate_interval<NX, SlotRng, SPARSE>(p, pl, t, t + sc.Ts, u, sc.Ns, rng);
            }
            if (status == ST_OK) {
                t = sc.t0 + (i + 1) * sc.Ts;
                z = pl.x[NX - 1] / p.V;
                zbar = setpoint_at(sc, t);
                const double r = z - zbar;
                acc += r * r;
            }
        }
        // producers stop generating once every sample of the warp has failed
        // (they still keep the handshake going to the end)
        const bool done = __all_sync(0xffffffffu, status != ST_OK);
        if (done && lane == 0) *(volatile int*)&stop = 1;
        if (i + kPiWsSlots < nbar) named_arrive(1 + kPiWsSlots + s, kThreads);
    }
    if (!real) return;
    nmpcmc_sim_record* rec = records + ii;
    if (status == ST_OK) {
        rec->phi = acc / (double)(nbar + 1);
        rec->failed = 0;
        if (tr != nullptr) {
            double* rw = tr + (size_t)row * 5;
            rw[0] = t;
            rw[1] = z;
            rw[2] = zbar;
            rw[3] = __longlong_as_double(0x7ff8000000000000LL);
            rw[4] = __longlong_as_double(0x7ff8000000000000LL);
        }
    } else {
        rec->phi = __longlong_as_double(0x7ff8000000000000LL);
        rec->failed = 1;
    }
    rec->ocp_solves = 0;
    rec->ocp_failures = 0;
    rec->status = status;
    if (counters != nullptr) {
        nmpcmc_work_counters c = {};
        c.control_steps = steps;
        counters[ii] = c;
    }
}

}  // namespace nmpcmc_dev
