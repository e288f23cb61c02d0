// controllers_api.cu -- the controller-level C ABI (include/nmpcmc_gpu.h):
// batched pi_step (controllers.cpp:12-23) and batched nmpc_step
// (controllers.cpp:114-212) on device-resident NmpcStates
// (make_nmpc_state, controllers.cpp:25-48). Kernels: pi_step_kernel
// (pi_kernel.cuh, K2's law) and nmpc_step_kernel (nmpc_gen_kernel.cuh, K3w's
// code path with the closed loop's own step function nmpc_step_ws).
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "ctx_internal.h"
#include "launchers.h"
#include "nmpcmc_gpu.h"

using nmpcmc_host::cuda_check;
using nmpcmc_host::ensure;
using nmpcmc_host::fail;

struct nmpcmc_nmpc_batch {
    nmpcmc_gpu_ctx* ctx = nullptr;
    nmpcmc_scenario sc{};
    int64_t batch = 0;
    int nx = 1;
    int64_t stride = 0;  // doubles per state (StateLay)
    double* d_states = nullptr;
    void* d_io = nullptr;  // t, y, setpoints, u, diag staging
    size_t io_cap = 0;
};

namespace {

int nx_of(const nmpcmc_scenario& sc) { return sc.ctrl_variant == NMPCMC_THREE_STATE ? 3 : 1; }

/// StateLay offsets (nmpc_gen_kernel.cuh) for host-side packing.
struct HostLay {
    int64_t XH, P, WARM, XI, LAM, PL, PU, total;
    HostLay(int nx, int N)
        : XH(0), P(nx), WARM(nx + nx * nx), XI(WARM + 1), LAM(XI + (int64_t)N * (1 + nx)),
          PL(LAM + (int64_t)N * nx), PU(PL + N), total(PU + N) {}
};

}  // namespace

extern "C" {

int nmpcmc_gpu_pi_step_device(nmpcmc_gpu_ctx* ctx, nmpcmc_pi_state* states_dev, const double* y_dev,
                              const double* y_bar_dev, int64_t n, nmpcmc_pi_step_result* results_dev) {
    if (ctx == nullptr || n < 0) return NMPCMC_INVALID_ARGUMENT;
    if (n == 0) return NMPCMC_OK;
    if (!states_dev || !y_dev || !y_bar_dev) return NMPCMC_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    nmpcmc_launch::launch_pi_step(states_dev, y_dev, y_bar_dev, n, results_dev, ctx->sm_count, ctx->stream);
    return cuda_check(ctx, cudaGetLastError(), "pi_step_kernel launch");
}

int nmpcmc_gpu_pi_step_batch(nmpcmc_gpu_ctx* ctx, nmpcmc_pi_state* states, const double* y, const double* y_bar,
                             int64_t n, nmpcmc_pi_step_result* results) {
    if (ctx == nullptr || n < 0) return NMPCMC_INVALID_ARGUMENT;
    if (n == 0) return NMPCMC_OK;
    if (!states || !y || !y_bar) return NMPCMC_INVALID_ARGUMENT;
    for (int64_t i = 0; i < n; ++i)  // PiState invariant (controllers.hpp:14)
        if (!(states[i].Ts > 0.0)) return fail(ctx, NMPCMC_DOMAIN_ERROR, "pi_step: Ts must be positive");
    cudaSetDevice(ctx->device);
    auto rnd = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t bs = n * sizeof(nmpcmc_pi_state), by = n * sizeof(double),
                 br = results ? n * sizeof(nmpcmc_pi_step_result) : 0;
    int rc;
    if ((rc = ensure(ctx, &ctx->d_state, &ctx->state_cap, rnd(bs) + 2 * rnd(by) + rnd(br))) != NMPCMC_OK) return rc;
    char* p = static_cast<char*>(ctx->d_state);
    auto* d_s = reinterpret_cast<nmpcmc_pi_state*>(p);
    auto* d_y = reinterpret_cast<double*>(p + rnd(bs));
    auto* d_yb = reinterpret_cast<double*>(p + rnd(bs) + rnd(by));
    auto* d_r = results ? reinterpret_cast<nmpcmc_pi_step_result*>(p + rnd(bs) + 2 * rnd(by)) : nullptr;
    cudaError_t e = cudaMemcpyAsync(d_s, states, bs, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_y, y, by, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_yb, y_bar, by, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaMemcpyAsync");
    if ((rc = nmpcmc_gpu_pi_step_device(ctx, d_s, d_y, d_yb, n, d_r)) != NMPCMC_OK) return rc;
    e = cudaMemcpyAsync(states, d_s, bs, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && results) e = cudaMemcpyAsync(results, d_r, br, cudaMemcpyDeviceToHost, ctx->stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaMemcpyAsync");
    return cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "pi_step_kernel");
}

int nmpcmc_gpu_nmpc_batch_create(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, int64_t batch,
                                 const double* x0_hat, const double* P0, nmpcmc_nmpc_batch** out) {
    if (ctx == nullptr || sc == nullptr || out == nullptr || batch < 1) return NMPCMC_INVALID_ARGUMENT;
    *out = nullptr;
    // make_nmpc_state's checks (controllers.cpp:28-35)
    if (sc->N <= 0 || !(sc->horizon_Ts > 0.0) || sc->Nc <= 0 || sc->np <= 0)
        return fail(ctx, NMPCMC_DOMAIN_ERROR, "make_nmpc_state: horizon and step counts must be positive");
    if (nmpcmc_launch::nmpc_state_doubles(*sc) <= 0 || !nmpcmc_launch::genw_fits(*sc))
        return fail(ctx, NMPCMC_UNSUPPORTED, "nmpc batch: horizon too long for the shared-memory sweep arrays");
    cudaSetDevice(ctx->device);
    auto* st = new nmpcmc_nmpc_batch();
    st->ctx = ctx;
    st->sc = *sc;
    st->batch = batch;
    st->nx = nx_of(*sc);
    const HostLay lay(st->nx, sc->N);
    st->stride = lay.total;
    std::vector<double> h((size_t)(batch * lay.total), 0.0);
    const int nx = st->nx;
    for (int64_t b = 0; b < batch; ++b) {
        double* s = h.data() + b * lay.total;
        for (int i = 0; i < nx; ++i) s[lay.XH + i] = x0_hat ? x0_hat[b * nx + i] : sc->x0_hat[i];
        for (int e = 0; e < nx * nx; ++e) s[lay.P + e] = P0 ? P0[b * nx * nx + e] : sc->P0[e];
        s[lay.WARM] = 0.0;  // last_xi empty: the first step cold-starts
    }
    const size_t bytes = h.size() * sizeof(double);
    cudaError_t e = cudaMalloc(&st->d_states, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(st->d_states, h.data(), bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        const int rc = cuda_check(ctx, e, "nmpc batch states");
        nmpcmc_gpu_nmpc_batch_destroy(st);
        return rc;
    }
    *out = st;
    return NMPCMC_OK;
}

void nmpcmc_gpu_nmpc_batch_destroy(nmpcmc_nmpc_batch* st) {
    if (st == nullptr) return;
    if (st->ctx) cudaSetDevice(st->ctx->device);
    if (st->d_states) cudaFree(st->d_states);
    if (st->d_io) cudaFree(st->d_io);
    delete st;
}

int64_t nmpcmc_gpu_nmpc_batch_size(const nmpcmc_nmpc_batch* st) { return st ? st->batch : 0; }

int nmpcmc_gpu_nmpc_step_batch(nmpcmc_gpu_ctx* ctx, nmpcmc_nmpc_batch* st, const double* t, const double* y,
                               const double* setpoints, double* u_out, nmpcmc_nmpc_diag* diag) {
    if (ctx == nullptr || st == nullptr || !t || !y || !u_out) return NMPCMC_INVALID_ARGUMENT;
    if (st->ctx->device != ctx->device) return fail(ctx, NMPCMC_INVALID_ARGUMENT, "nmpc batch: other device");
    cudaSetDevice(ctx->device);
    const int64_t B = st->batch, N = st->sc.N;
    auto rnd = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t bt = B * sizeof(double), bsp = setpoints ? B * N * sizeof(double) : 0,
                 bd = diag ? B * sizeof(nmpcmc_nmpc_diag) : 0;
    int rc;
    if ((rc = ensure(ctx, &st->d_io, &st->io_cap, 3 * rnd(bt) + rnd(bsp) + rnd(bd))) != NMPCMC_OK) return rc;
    char* p = static_cast<char*>(st->d_io);
    auto* d_t = reinterpret_cast<double*>(p);
    auto* d_y = reinterpret_cast<double*>(p + rnd(bt));
    auto* d_u = reinterpret_cast<double*>(p + 2 * rnd(bt));
    auto* d_sp = setpoints ? reinterpret_cast<double*>(p + 3 * rnd(bt)) : nullptr;
    auto* d_dg = diag ? reinterpret_cast<nmpcmc_nmpc_diag*>(p + 3 * rnd(bt) + rnd(bsp)) : nullptr;
    const int64_t blocks = nmpcmc_launch::genw_blocks(st->sc, ctx->sm_count, B);
    const size_t need = (size_t)blocks * (size_t)nmpcmc_launch::gen_ws_doubles(st->sc) * sizeof(double);
    if ((rc = ensure(ctx, &ctx->d_ws, &ctx->ws_cap, need)) != NMPCMC_OK) return rc;
    if ((rc = ensure(ctx, &ctx->d_counter, &ctx->counter_cap, 256)) != NMPCMC_OK) return rc;
    cudaError_t e = cudaMemcpyAsync(d_t, t, bt, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_y, y, bt, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess && setpoints) e = cudaMemcpyAsync(d_sp, setpoints, bsp, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaMemcpyAsync");
    rc = nmpcmc_launch::launch_nmpc_step(st->sc, B, st->d_states, d_t, d_y, d_sp, d_u, d_dg,
                                         static_cast<double*>(ctx->d_ws), blocks,
                                         static_cast<unsigned long long*>(ctx->d_counter), ctx->stream);
    if (rc != NMPCMC_OK) return fail(ctx, rc, "nmpc_step batch: unsupported configuration");
    if ((rc = cuda_check(ctx, cudaGetLastError(), "nmpc_step_kernel launch")) != NMPCMC_OK) return rc;
    e = cudaMemcpyAsync(u_out, d_u, bt, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && diag) e = cudaMemcpyAsync(diag, d_dg, bd, cudaMemcpyDeviceToHost, ctx->stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaMemcpyAsync");
    return cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "nmpc_step_kernel");
}

int nmpcmc_gpu_nmpc_batch_get(nmpcmc_nmpc_batch* st, double* x_hat, double* P, double* last_xi,
                              double* last_lambda, double* last_pi_l, double* last_pi_u, int32_t* warm) {
    if (st == nullptr) return NMPCMC_INVALID_ARGUMENT;
    cudaSetDevice(st->ctx->device);
    const HostLay lay(st->nx, st->sc.N);
    std::vector<double> h((size_t)(st->batch * lay.total));
    cudaError_t e = cudaStreamSynchronize(st->ctx->stream);
    if (e == cudaSuccess)
        e = cudaMemcpy(h.data(), st->d_states, h.size() * sizeof(double), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_check(st->ctx, e, "nmpc batch read");
    const int nx = st->nx;
    const int64_t N = st->sc.N, L = N * (1 + nx);
    for (int64_t b = 0; b < st->batch; ++b) {
        const double* s = h.data() + b * lay.total;
        if (x_hat)
            for (int i = 0; i < nx; ++i) x_hat[b * nx + i] = s[lay.XH + i];
        if (P)
            for (int i = 0; i < nx * nx; ++i) P[b * nx * nx + i] = s[lay.P + i];
        if (last_xi)
            for (int64_t i = 0; i < L; ++i) last_xi[b * L + i] = s[lay.XI + i];
        if (last_lambda)
            for (int64_t i = 0; i < N * nx; ++i) last_lambda[b * N * nx + i] = s[lay.LAM + i];
        if (last_pi_l)
            for (int64_t i = 0; i < N; ++i) last_pi_l[b * N + i] = s[lay.PL + i];
        if (last_pi_u)
            for (int64_t i = 0; i < N; ++i) last_pi_u[b * N + i] = s[lay.PU + i];
        if (warm) warm[b] = s[lay.WARM] != 0.0 ? 1 : 0;
    }
    return NMPCMC_OK;
}

int64_t nmpcmc_qnlp_doubles(int32_t N, int32_t n_x) {
    if (N < 1 || (n_x != 1 && n_x != 3)) return 0;
    return nmpcmc_launch::qnlp_stride(N, n_x);
}

int nmpcmc_gpu_sqp_solve_qnlp_batch(nmpcmc_gpu_ctx* ctx, const nmpcmc_qnlp_dims* d, int64_t batch,
                                    const double* problems, const double* xi0, double* xi, double* lambda,
                                    double* pi_l, double* pi_u, int32_t* converged, int32_t* iterations,
                                    int32_t* status) {
    if (ctx == nullptr || d == nullptr || batch < 0) return NMPCMC_INVALID_ARGUMENT;
    if (d->N < 1 || (d->n_x != 1 && d->n_x != 3) || d->n_u != 1)
        return fail(ctx, NMPCMC_DIMENSION_MISMATCH, "qnlp batch: N >= 1, n_x in {1, 3}, n_u = 1");
    if (d->sqp.max_iter < 0 || d->sqp.qp_max_iter < 1 || d->sqp.max_backtracks < 0)
        return fail(ctx, NMPCMC_DOMAIN_ERROR, "qnlp batch: bad SqpOptions");
    if (batch == 0) return NMPCMC_OK;
    if (!problems || !xi || !lambda || !pi_l || !pi_u || !converged || !iterations || !status)
        return NMPCMC_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    const int nx = d->n_x, N = d->N;
    const int64_t stride = nmpcmc_launch::qnlp_stride(N, nx), L = (int64_t)N * (1 + nx);
    auto rnd = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t bp = batch * stride * 8, bx = batch * L * 8, bl = batch * (int64_t)N * nx * 8,
                 bpi = batch * (int64_t)N * 8, bi = batch * 4;
    int rc;
    if ((rc = ensure(ctx, &ctx->d_scratch, &ctx->scratch_cap,
                     rnd(bp) + (xi0 ? rnd(bx) : 0) + rnd(bx) + rnd(bl) + 2 * rnd(bpi) + 3 * rnd(bi))) != NMPCMC_OK)
        return rc;
    char* p = static_cast<char*>(ctx->d_scratch);
    auto take = [&](size_t n) {
        char* a = p;
        p += rnd(n);
        return a;
    };
    auto* d_prob = reinterpret_cast<double*>(take(bp));
    auto* d_xi0 = xi0 ? reinterpret_cast<double*>(take(bx)) : nullptr;
    auto* d_xi = reinterpret_cast<double*>(take(bx));
    auto* d_lam = reinterpret_cast<double*>(take(bl));
    auto* d_pil = reinterpret_cast<double*>(take(bpi));
    auto* d_piu = reinterpret_cast<double*>(take(bpi));
    auto* d_conv = reinterpret_cast<int32_t*>(take(bi));
    auto* d_it = reinterpret_cast<int32_t*>(take(bi));
    auto* d_st = reinterpret_cast<int32_t*>(take(bi));
    // one warp per problem, persistent one-warp blocks; the per-warp slabs
    // stay L2-resident (as K3w's)
    int64_t blocks = (int64_t)ctx->sm_count * 16;
    const int64_t slab = nmpcmc_launch::qnlp_ws_doubles(N, nx);
    const int64_t l2_cap = (int64_t)(96ull << 20) / (slab * 8);
    if (blocks > l2_cap) blocks = l2_cap < ctx->sm_count ? ctx->sm_count : l2_cap;
    if (blocks > batch) blocks = batch;
    if ((rc = ensure(ctx, &ctx->d_ws, &ctx->ws_cap, (size_t)(blocks * slab * 8))) != NMPCMC_OK) return rc;
    if ((rc = ensure(ctx, &ctx->d_counter, &ctx->counter_cap, 256)) != NMPCMC_OK) return rc;
    cudaError_t e = cudaMemcpyAsync(d_prob, problems, bp, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess && xi0) e = cudaMemcpyAsync(d_xi0, xi0, bx, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaMemcpyAsync");
    rc = nmpcmc_launch::launch_qnlp_batch(N, nx, d->sqp, batch, d_prob, d_xi0, d_xi, d_lam, d_pil, d_piu, d_conv,
                                          d_it, d_st, static_cast<double*>(ctx->d_ws), blocks,
                                          static_cast<unsigned long long*>(ctx->d_counter), ctx->stream);
    if (rc != NMPCMC_OK) return fail(ctx, rc, "qnlp batch: horizon too long for the shared-memory sweep arrays");
    if ((rc = cuda_check(ctx, cudaGetLastError(), "qnlp_batch_kernel launch")) != NMPCMC_OK) return rc;
    e = cudaMemcpyAsync(xi, d_xi, bx, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(lambda, d_lam, bl, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pi_l, d_pil, bpi, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pi_u, d_piu, bpi, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(converged, d_conv, bi, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(iterations, d_it, bi, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(status, d_st, bi, cudaMemcpyDeviceToHost, ctx->stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaMemcpyAsync");
    return cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "qnlp_batch_kernel");
}

int nmpcmc_gpu_solve_ocp_batch_traced(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, int64_t batch,
                                      const double* x0, const double* t0, const double* xi0, double* xi,
                                      double* lambda, double* pi_l, double* pi_u, int32_t* converged,
                                      int32_t* status, int32_t* iterations, int32_t max_trace,
                                      nmpcmc_sqp_iter_log* trace, int32_t* trace_len) {
    if (ctx == nullptr || sc == nullptr || batch < 0 || max_trace < 0) return NMPCMC_INVALID_ARGUMENT;
    if (batch > 0 && (!x0 || !t0 || !xi || !lambda || !pi_l || !pi_u || !converged || !status || !iterations ||
                      !trace_len || (max_trace > 0 && !trace)))
        return NMPCMC_INVALID_ARGUMENT;
    if (sc->controller != NMPCMC_CTRL_NMPC) return fail(ctx, NMPCMC_INVALID_ARGUMENT, "OCP batch: NMPC scenario");
    int32_t nbar = 0;
    int rc = nmpcmc_gpu_validate(sc, &nbar);
    if (rc != NMPCMC_OK) return fail(ctx, rc, "scenario validation failed");
    if (batch == 0) return NMPCMC_OK;
    if (!nmpcmc_launch::genw_fits(*sc))
        return fail(ctx, NMPCMC_UNSUPPORTED, "OCP batch: horizon too long for the shared-memory sweep arrays");
    cudaSetDevice(ctx->device);
    const int nx = nx_of(*sc);
    const int64_t L = (int64_t)sc->N * (1 + nx), NN = (int64_t)sc->N * nx;
    const size_t b_x0 = batch * nx * 8, b_t0 = batch * 8, b_xi = batch * L * 8, b_lam = batch * NN * 8,
                 b_pi = batch * sc->N * 8, b_i = batch * 4, b_tr = (size_t)batch * max_trace * sizeof(nmpcmc_sqp_iter_log);
    auto rnd = [](size_t n) { return (n + 255) / 256 * 256; };
    const size_t total = rnd(b_x0) + rnd(b_t0) + (xi0 ? rnd(b_xi) : 0) + rnd(b_xi) + rnd(b_lam) + 2 * rnd(b_pi) +
                         4 * rnd(b_i) + rnd(b_tr);
    if ((rc = ensure(ctx, &ctx->d_scratch, &ctx->scratch_cap, total)) != NMPCMC_OK) return rc;
    char* p = static_cast<char*>(ctx->d_scratch);
    auto take = [&](size_t n) {
        char* a = p;
        p += rnd(n);
        return a;
    };
    auto* d_x0 = reinterpret_cast<double*>(take(b_x0));
    auto* d_t0 = reinterpret_cast<double*>(take(b_t0));
    auto* d_xi0 = xi0 ? reinterpret_cast<double*>(take(b_xi)) : nullptr;
    auto* d_xi = reinterpret_cast<double*>(take(b_xi));
    auto* d_lam = reinterpret_cast<double*>(take(b_lam));
    auto* d_pil = reinterpret_cast<double*>(take(b_pi));
    auto* d_piu = reinterpret_cast<double*>(take(b_pi));
    auto* d_conv = reinterpret_cast<int32_t*>(take(b_i));
    auto* d_st = reinterpret_cast<int32_t*>(take(b_i));
    auto* d_it = reinterpret_cast<int32_t*>(take(b_i));
    auto* d_tl = reinterpret_cast<int32_t*>(take(b_i));
    auto* d_tr = max_trace > 0 ? reinterpret_cast<nmpcmc_sqp_iter_log*>(take(b_tr)) : nullptr;
    const int64_t blocks = nmpcmc_launch::genw_blocks(*sc, ctx->sm_count, batch);
    const size_t ws_b = (size_t)blocks * (size_t)nmpcmc_launch::gen_ws_doubles(*sc) * sizeof(double);
    if ((rc = ensure(ctx, &ctx->d_ws, &ctx->ws_cap, ws_b)) != NMPCMC_OK) return rc;
    if ((rc = ensure(ctx, &ctx->d_counter, &ctx->counter_cap, 256)) != NMPCMC_OK) return rc;
    cudaError_t e = cudaMemcpyAsync(d_x0, x0, b_x0, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_t0, t0, b_t0, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess && xi0) e = cudaMemcpyAsync(d_xi0, xi0, b_xi, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaMemcpyAsync");
    // the trace buffer pointer is non-null even when max_trace == 0, so the
    // kernel still counts the records into trace_len
    nmpcmc_sqp_iter_log* tr_arg = d_tr != nullptr ? d_tr : reinterpret_cast<nmpcmc_sqp_iter_log*>(d_tl);
    rc = nmpcmc_launch::launch_ocp_batch(*sc, batch, d_x0, d_t0, d_xi0, d_xi, d_lam, d_pil, d_piu, d_conv, d_st,
                                         static_cast<double*>(ctx->d_ws), blocks,
                                         static_cast<unsigned long long*>(ctx->d_counter), ctx->stream, d_it,
                                         max_trace, tr_arg, d_tl);
    if (rc != NMPCMC_OK) return fail(ctx, rc, "OCP batch: unsupported configuration");
    if ((rc = cuda_check(ctx, cudaGetLastError(), "ocp_batch_kernel launch")) != NMPCMC_OK) return rc;
    e = cudaMemcpyAsync(xi, d_xi, b_xi, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(lambda, d_lam, b_lam, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pi_l, d_pil, b_pi, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pi_u, d_piu, b_pi, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(converged, d_conv, b_i, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(status, d_st, b_i, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(iterations, d_it, b_i, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(trace_len, d_tl, b_i, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && d_tr) e = cudaMemcpyAsync(trace, d_tr, b_tr, cudaMemcpyDeviceToHost, ctx->stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaMemcpyAsync");
    return cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "ocp_batch_kernel");
}

}  // extern "C"
