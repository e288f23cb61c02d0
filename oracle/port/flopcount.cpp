// flopcount.cpp -- op-counting build of the port (oracle/port/nmpcmc_port.cpp).
// MEASUREMENT INFRASTRUCTURE ONLY: derives the per-unit FP64 work constants of
// the roofline (paper_2212_02197_b200/workmodel.py) by running the reference's
// algorithm, restated by the port, on a counting double. This is the
// cross-check that SURVEY.md §8(d) asks for ("template the restatement on its scalar
// type, run it with an op-counting double wrapper").
//
// Convention: +, -, *, / and sqrt are 1 flop each; exp = log = 20;
// sincos = 40. Negation, abs and comparisons count 0. Every executed operation of the
// reference's expressions counts, gemm/gemv epilogues (1.0*s + 0.0) included.
//
// Build + run: make -C oracle flops && oracle/_build/flopcount
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <limits>
#include <thread>
#include <vector>

#include "nmpcmc_gpu.h"

extern "C" {
double nmx_exp(double);
double nmx_log(double);
void nmx_sincos(double, double*, double*);
}

namespace fc {

enum Phase { OTHER, PLANT, EKF, SHOOT, XI, XISHOOT, QP, SQP, STEP, IPM, NPH };
const char* kNames[NPH] = {"other", "plant", "ekf", "shoot", "xi", "xishoot", "qp", "sqp", "step", "ipm"};
int g_phase = OTHER;
double g_flops[NPH];
double g_units[NPH];

inline void count(double f) { g_flops[g_phase] += f; }

struct PhaseScope {
    int prev;
    explicit PhaseScope(int ph) : prev(g_phase) { g_phase = (ph == SHOOT && prev == XI) ? XISHOOT : ph; }
    ~PhaseScope() { g_phase = prev; }
};
inline void add_unit(int u, double n) {
    if (u == SHOOT && g_phase == XISHOOT) u = XISHOOT;
    g_units[u] += n;
}

/// Counting double: every arithmetic operation adds one flop to the current
/// phase. Mixed overloads (Flop op double/int) are exact matches, so the
/// implicit conversion back to double never makes an operator ambiguous.
struct Flop {
    double v;
    constexpr Flop() : v(0.0) {}
    constexpr Flop(double x) : v(x) {}  // NOLINT: implicit on purpose (literals)
    explicit operator double() const { return v; }
    Flop operator-() const { return Flop(-v); }
};

#define FC_ARITH(op)                                                                      \
    inline Flop operator op(Flop a, Flop b) { return count(1), Flop(a.v op b.v); }        \
    inline Flop operator op(Flop a, double b) { return count(1), Flop(a.v op b); }        \
    inline Flop operator op(double a, Flop b) { return count(1), Flop(a op b.v); }        \
    inline Flop operator op(Flop a, int b) { return count(1), Flop(a.v op b); }           \
    inline Flop operator op(int a, Flop b) { return count(1), Flop(a op b.v); }           \
    inline Flop operator op(Flop a, long b) { return count(1), Flop(a.v op b); }          \
    inline Flop operator op(Flop a, unsigned long b) { return count(1), Flop(a.v op b); } \
    inline Flop& operator op##=(Flop & a, Flop b) { return count(1), a.v = a.v op b.v, a; } \
    inline Flop& operator op##=(Flop & a, double b) { return count(1), a.v = a.v op b, a; }
FC_ARITH(+)
FC_ARITH(-)
FC_ARITH(*)
FC_ARITH(/)
#undef FC_ARITH

#define FC_CMP(op)                                                        \
    inline bool operator op(Flop a, Flop b) { return a.v op b.v; }       \
    inline bool operator op(Flop a, double b) { return a.v op b; }        \
    inline bool operator op(double a, Flop b) { return a op b.v; }        \
    inline bool operator op(Flop a, int b) { return a.v op b; }           \
    inline bool operator op(int a, Flop b) { return a op b.v; }
FC_CMP(<)
FC_CMP(<=)
FC_CMP(>)
FC_CMP(>=)
FC_CMP(==)
FC_CMP(!=)
#undef FC_CMP

}  // namespace fc

namespace std {
inline fc::Flop sqrt(fc::Flop x) { return fc::count(1), fc::Flop(std::sqrt(x.v)); }
inline fc::Flop abs(fc::Flop x) { return fc::Flop(std::fabs(x.v)); }
inline fc::Flop fabs(fc::Flop x) { return fc::Flop(std::fabs(x.v)); }
inline bool isfinite(fc::Flop x) { return std::isfinite(x.v); }
inline const fc::Flop& max(const fc::Flop& a, const fc::Flop& b) { return (a < b) ? b : a; }
inline const fc::Flop& min(const fc::Flop& a, const fc::Flop& b) { return (b < a) ? b : a; }
inline fc::Flop max(double a, fc::Flop b) { return max(fc::Flop(a), b); }
inline fc::Flop max(fc::Flop a, double b) { return max(a, fc::Flop(b)); }
inline fc::Flop min(double a, fc::Flop b) { return min(fc::Flop(a), b); }
inline fc::Flop min(fc::Flop a, double b) { return min(a, fc::Flop(b)); }
template <>
struct numeric_limits<fc::Flop> : numeric_limits<double> {};
}  // namespace std

static inline fc::Flop P_EXP(fc::Flop x) { return fc::count(20), fc::Flop(nmx_exp(x.v)); }
static inline fc::Flop P_LOG(fc::Flop x) { return fc::count(20), fc::Flop(nmx_log(x.v)); }
static inline void P_SINCOS(fc::Flop x, fc::Flop* s, fc::Flop* c) {
    fc::count(40);
    double a, b;
    nmx_sincos(x.v, &a, &b);
    *s = a;
    *c = b;
}

#define PORT_CUSTOM_LIBM
#define PORT_NO_CAPI
#define PORT_PHASE(ph) fc::PhaseScope fc_scope_(fc::ph)
#define PORT_UNIT(u, n) fc::add_unit(fc::u, (n))
#define PORT_TO_DOUBLE(x) ((x).v)
typedef double port_real_t;
#define PORT_REAL port_real_t
#define double fc::Flop
#include "nmpcmc_port.cpp"
#undef double

namespace {

/// One state-only shooting interval as the device computes it for
/// xi_from_inputs (F only, no sensitivities): Nc RK4 steps of the drift.
double fonly_interval(const port::Cstr& m, int nc, double Ts) {
    const double f0 = fc::g_flops[fc::OTHER];
    std::vector<fc::Flop> x(m.nx);
    for (int i = 0; i < m.nx; ++i) x[i] = (m.nx == 3 ? 11.0 : 35.0) + i;
    if (m.nx == 3) x = {0.0358, 0.0297, 35.175};
    else x = {35.175};
    const fc::Flop h = fc::Flop(Ts) / nc;
    for (int st = 0; st < nc; ++st) {
        auto a = m.drift(x, 600.0);
        std::vector<fc::Flop> t(m.nx);
        for (int i = 0; i < m.nx; ++i) t[i] = x[i] + 0.5 * h * a[i];
        auto b = m.drift(t, 600.0);
        for (int i = 0; i < m.nx; ++i) t[i] = x[i] + 0.5 * h * b[i];
        auto c = m.drift(t, 600.0);
        for (int i = 0; i < m.nx; ++i) t[i] = x[i] + 1.0 * h * c[i];
        auto d = m.drift(t, 600.0);
        for (int i = 0; i < m.nx; ++i) x[i] += (h / 6.0) * (a[i] + 2.0 * b[i] + 2.0 * c[i] + d[i]);
    }
    return fc::g_flops[fc::OTHER] - f0;
}

/// A scenario as configs.make_scenario builds it (BASELINE config 2/3).
nmpcmc_scenario make(int ctrl_variant, int N, int steps) {
    nmpcmc_scenario sc{};
    sc.controller = NMPCMC_CTRL_NMPC;
    sc.truth_variant = NMPCMC_THREE_STATE;
    sc.ctrl_variant = ctrl_variant;
    nmpcmc_cstr_params p{0.105, 0x1.679cb6b1d419cp+35, 8500.0, 560.0 / 4.186, 0.8, 1.2, 273.65,
                         0.0, 0.0, 2.5, 0.0, 1000.0};
    sc.truth = p;
    sc.ctrl = p;
    sc.has_noise_R = 1;
    sc.noise_R = 0.01;
    sc.R_filter = 0.01;
    sc.Qz = 1.0;
    sc.horizon_Ts = 10.0;
    sc.N = N;
    sc.Nc = 5;
    sc.np = 5;
    sc.Ns = 10;
    sc.sqp = {1e-6, 1e-4, 0.5, 1e-12, 20, 30, 50, 0};
    sc.u_min = 0.0;
    sc.u_max = 1000.0;
    sc.t0 = 0.0;
    sc.Ts = 10.0;
    sc.tf = 10.0 * steps;
    sc.n_setpoints = 4;
    const double sp[4] = {335.0, 340.0, 330.0, 340.0};
    for (int i = 0; i < 4; ++i) {
        sc.sp_times[i] = 1800.0 * i;
        sc.sp_values[i] = sp[i];
    }
    const double T0 = 335.0, cA = p.cA_in - (T0 - p.cT_in) / p.beta, cB = p.cB_in - 2.0 * (T0 - p.cT_in) / p.beta;
    const double x0[3] = {cA * p.V, cB * p.V, T0 * p.V};
    for (int i = 0; i < 3; ++i) sc.x0[i] = x0[i];
    const int nxc = ctrl_variant == NMPCMC_THREE_STATE ? 3 : 1;
    for (int i = 0; i < nxc; ++i) {
        sc.x0_hat[i] = x0[3 - nxc + i];
        sc.P0[i * nxc + i] = 1e-6;
    }
    sc.base_seed = 12345;
    sc.perturb = 1;
    sc.perturb_rel_std[0] = sc.perturb_rel_std[1] = sc.perturb_rel_std[2] = 0.05;
    return sc;
}

}  // namespace

int main(int argc, char** argv) {
    const int samples = argc > 1 ? std::atoi(argv[1]) : 6;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 60;
    std::printf("{\n");
    bool first = true;
    for (int cv : {NMPCMC_ONE_STATE, NMPCMC_THREE_STATE}) {
        for (int N : {30, 60, 120}) {
            std::fill(fc::g_flops, fc::g_flops + fc::NPH, 0.0);
            std::fill(fc::g_units, fc::g_units + fc::NPH, 0.0);
            const nmpcmc_scenario sc = make(cv, N, steps);
            int failed = 0;
            for (int i = 0; i < samples; ++i) {
                nmpcmc_sim_record rec;
                port::closed_loop(sc, (uint64_t)i, &rec, nullptr, 0);
                failed += rec.failed;
            }
            const port::Cstr ctrl(sc.ctrl, cv);
            const double fonly = fonly_interval(ctrl, sc.Nc, sc.horizon_Ts);
            using namespace fc;
            const double steps_done = g_units[STEP];
            std::printf("%s \"nx%d_N%d\": {\"samples\": %d, \"failed\": %d, \"control_steps\": %.0f,\n",
                        first ? " " : ",", cv == NMPCMC_THREE_STATE ? 3 : 1, N, samples, failed, steps_done);
            first = false;
            std::printf("   \"shoot_full\": %.2f, \"shoot_fonly\": %.2f, \"ipm_stage\": %.2f, \"sqp_stage\": %.2f,\n",
                        g_flops[SHOOT] / g_units[SHOOT], fonly, g_flops[QP] / g_units[IPM],
                        g_flops[SQP] / g_units[SQP]);
            std::printf("   \"ekf_step\": %.2f, \"plant_step\": %.2f, \"other_per_step\": %.2f,\n",
                        g_flops[EKF] / steps_done, g_flops[PLANT] / steps_done,
                        (g_flops[OTHER] - fonly + g_flops[XI]) / steps_done);
            std::printf("   \"units\": {\"shoot\": %.0f, \"xishoot\": %.0f, \"ipm_stage_iters\": %.0f, "
                        "\"sqp_stage_iters\": %.0f}}\n",
                        g_units[SHOOT], g_units[XISHOOT], g_units[IPM], g_units[SQP]);
        }
    }
    std::printf("}\n");
    return 0;
}
