// nmpcmc_gpu.cu -- device entry points of the C ABI (include/nmpcmc_gpu.h).
//
// One context = one device + one stream. nmpcmc_gpu_run replaces the
// reference's std::thread pool (run_monte_carlo, montecarlo.cpp:213-251):
// the sample range becomes the grid (PI: a thread per sample; NMPC: a warp
// per sample), records land in index order exactly like McResult::sims.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ctx_internal.h"
#include "launchers.h"
#include "nmpcmc_gpu.h"

namespace {

using nmpcmc_host::cuda_check;
using nmpcmc_host::ensure;
using nmpcmc_host::fail;

/// Launch target: a stream and the workspace buffers the launch may use.
struct Target {
    cudaStream_t stream;
    void** d_gws;
    size_t* gws_cap;
    void** d_counter;
    size_t* counter_cap;
    void** d_ws;
    size_t* ws_cap;
};
Target main_target(nmpcmc_gpu_ctx* ctx) {
    return Target{ctx->stream, &ctx->d_gws, &ctx->gws_cap, &ctx->d_counter, &ctx->counter_cap, &ctx->d_ws,
                  &ctx->ws_cap};
}
Target lane_target(Lane& l) {
    return Target{l.stream, &l.d_gws, &l.gws_cap, &l.d_counter, &l.counter_cap, &l.d_ws, &l.ws_cap};
}

/// Enqueue the closed-loop kernel for [first, first+n) on target tg.
int launch(nmpcmc_gpu_ctx* ctx, const Target& tg, const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar,
           nmpcmc_sim_record* d_rec, nmpcmc_work_counters* d_cnt, double* d_traj, int rows) {
    if (n == 0) return NMPCMC_OK;
    if (sc.controller == NMPCMC_CTRL_PI) {
        nmpcmc_launch::launch_pi(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, ctx->sm_count, ctx->pi_kernel, tg.stream);
        return cuda_check(ctx, cudaGetLastError(), "pi_kernel launch");
    }
    int rc;
    // K3 for the one-state model (N <= 255) unless a generic kernel is asked
    // for; THREAD (the retired one-thread-per-sample K3b) selects K3g, the
    // generic one-thread-per-sample kernel
    const bool thread = ctx->nmpc_kernel == NMPCMC_NMPC_KERNEL_GENERIC ||
                        ctx->nmpc_kernel == NMPCMC_NMPC_KERNEL_THREAD;
    const bool generic = sc.ctrl_variant != NMPCMC_ONE_STATE || sc.N > 255 || thread ||
                         ctx->nmpc_kernel == NMPCMC_NMPC_KERNEL_GENERIC_WARP || ctx->ctrl_fd;
    // finite-difference controller jacobians run on K3w only
    if (ctx->ctrl_fd && (thread || !nmpcmc_launch::genw_fits(sc)))
        return fail(ctx, NMPCMC_UNSUPPORTED, "finite-difference jacobians need the one-warp generic kernel (K3w)");
    if (generic && !thread && nmpcmc_launch::genw_fits(sc)) {  // K3w (or K3g when N is too long for it)
        const int64_t blocks = nmpcmc_launch::genw_blocks(sc, ctx->sm_count, n);
        const size_t need = (size_t)blocks * (size_t)nmpcmc_launch::gen_ws_doubles(sc) * sizeof(double);
        if ((rc = ensure(ctx, tg.d_ws, tg.ws_cap, need)) != NMPCMC_OK) return rc;
        if ((rc = ensure(ctx, tg.d_counter, tg.counter_cap, 256)) != NMPCMC_OK) return rc;
        rc = nmpcmc_launch::launch_genw(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows,
                                        static_cast<double*>(*tg.d_ws), blocks,
                                        static_cast<unsigned long long*>(*tg.d_counter), tg.stream, ctx->ctrl_fd);
    } else if (generic) {
        const int64_t slots = nmpcmc_launch::gen_slots(sc, ctx->sm_count, n);
        const size_t need = (size_t)slots * (size_t)nmpcmc_launch::gen_ws_doubles(sc) * sizeof(double);
        if ((rc = ensure(ctx, tg.d_ws, tg.ws_cap, need)) != NMPCMC_OK) return rc;
        if ((rc = ensure(ctx, tg.d_counter, tg.counter_cap, 256)) != NMPCMC_OK) return rc;
        rc = nmpcmc_launch::launch_gen(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows,
                                       static_cast<double*>(*tg.d_ws), slots,
                                       static_cast<unsigned long long*>(*tg.d_counter), tg.stream);
    } else {
        size_t bytes = 0;
        int64_t blocks = 0;
        nmpcmc_launch::nmpc_gws_need(sc, ctx->sm_count, n, &bytes, &blocks);
        if ((rc = ensure(ctx, tg.d_gws, tg.gws_cap, bytes)) != NMPCMC_OK) return rc;
        if ((rc = ensure(ctx, tg.d_counter, tg.counter_cap, 256)) != NMPCMC_OK) return rc;
        rc = nmpcmc_launch::launch_nmpc(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, ctx->sm_count,
                                        static_cast<double*>(*tg.d_gws), blocks,
                                        static_cast<unsigned long long*>(*tg.d_counter), tg.stream);
    }
    if (rc != NMPCMC_OK) return fail(ctx, rc, "nmpc launch: unsupported configuration");
    return cuda_check(ctx, cudaGetLastError(), "nmpc_kernel launch");
}

/// Pick the lane of the next launch (lane mode): NMPC launches alternate
/// between lanes 0 and 1, PI uses lane 2. The lane first waits for all work
/// enqueued so far on ctx->stream.
int lane_begin(nmpcmc_gpu_ctx* ctx, int controller, Lane** out) {
    int rc;
    if (ctx->fork == nullptr &&
        (rc = cuda_check(ctx, cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming), "event")) != NMPCMC_OK)
        return rc;
    const int i = controller == NMPCMC_CTRL_PI ? 2 : (ctx->next_nmpc_lane++ & 1);
    Lane& l = ctx->lane[i];
    if (l.stream == nullptr) {
        if ((rc = cuda_check(ctx, cudaStreamCreateWithFlags(&l.stream, cudaStreamNonBlocking), "lane stream")) !=
            NMPCMC_OK)
            return rc;
        if ((rc = cuda_check(ctx, cudaEventCreateWithFlags(&l.done, cudaEventDisableTiming), "event")) != NMPCMC_OK)
            return rc;
    }
    cudaEventRecord(ctx->fork, ctx->stream);
    cudaStreamWaitEvent(l.stream, ctx->fork, 0);
    *out = &l;
    return NMPCMC_OK;
}
void lane_end(Lane* l) {
    cudaEventRecord(l->done, l->stream);
    l->pending = true;
}

}  // namespace

extern "C" {

int nmpcmc_gpu_device_count(int* count_out) {
    if (count_out == nullptr) return NMPCMC_INVALID_ARGUMENT;
    *count_out = 0;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) return NMPCMC_NO_DEVICE;
    *count_out = count;
    return NMPCMC_OK;
}

int nmpcmc_gpu_ctx_create(int device, nmpcmc_gpu_ctx** out) {
    if (out == nullptr) return NMPCMC_INVALID_ARGUMENT;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return NMPCMC_NO_DEVICE;
    if (device < 0 || device >= count) return NMPCMC_NO_DEVICE;
    auto* ctx = new nmpcmc_gpu_ctx();
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete ctx;
        return NMPCMC_CUDA_ERROR;
    }
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return NMPCMC_CUDA_ERROR;
    }
    ctx->own = ctx->stream;
    *out = ctx;
    return NMPCMC_OK;
}

void nmpcmc_gpu_ctx_destroy(nmpcmc_gpu_ctx* ctx) {
    if (ctx == nullptr) return;
    for (size_t g = 0; g < ctx->comms.size(); ++g)
        if (ctx->comms[g]) nmpcmc_host::nccl().CommDestroy(ctx->comms[g]);
    for (nmpcmc_gpu_ctx* s : ctx->subs) nmpcmc_gpu_ctx_destroy(s);
    if (ctx->comm) nmpcmc_host::nccl().CommDestroy(ctx->comm);
    cudaSetDevice(ctx->device);
    for (Lane& l : ctx->lane) {
        if (l.stream) {
            cudaStreamSynchronize(l.stream);
            cudaStreamDestroy(l.stream);
        }
        if (l.done) cudaEventDestroy(l.done);
        for (void* p : {l.d_gws, l.d_counter, l.d_ws, l.d_rec, l.d_cnt})
            if (p) cudaFree(p);
    }
    if (ctx->fork) cudaEventDestroy(ctx->fork);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    for (void* p : {ctx->d_rec, ctx->d_cnt, ctx->d_traj, ctx->d_scratch, ctx->d_ws, ctx->d_gws, ctx->d_counter,
                    ctx->d_k4, ctx->d_all, ctx->d_state, ctx->d_tot})
        if (p) cudaFree(p);
    delete ctx;
}

const char* nmpcmc_gpu_last_error(const nmpcmc_gpu_ctx* ctx) {
    return ctx ? ctx->err.c_str() : nmpcmc_host::create_error().c_str();
}

int nmpcmc_gpu_set_option(nmpcmc_gpu_ctx* ctx, int32_t option, int64_t value) {
    if (ctx == nullptr) return NMPCMC_INVALID_ARGUMENT;
    for (nmpcmc_gpu_ctx* s : ctx->subs) {
        const int rc = nmpcmc_gpu_set_option(s, option, value);
        if (rc != NMPCMC_OK) return rc;
    }
    switch (option) {
        case NMPCMC_OPT_NMPC_KERNEL:
            if (value < NMPCMC_NMPC_KERNEL_WARP || value > NMPCMC_NMPC_KERNEL_GENERIC_WARP)
                return NMPCMC_INVALID_ARGUMENT;
            ctx->nmpc_kernel = (int)value;
            return NMPCMC_OK;
        case NMPCMC_OPT_LANES:
            if (value != 1 && value != 2) return NMPCMC_INVALID_ARGUMENT;
            nmpcmc_gpu_join(ctx);
            ctx->lanes = (int)value;
            return NMPCMC_OK;
        case NMPCMC_OPT_TPS_WARPS_PER_SM:
            if (value < 1 || value > 64) return NMPCMC_INVALID_ARGUMENT;
            ctx->tps_warps_per_sm = (int)value;
            return NMPCMC_OK;
        case NMPCMC_OPT_PI_KERNEL:
            if (value != NMPCMC_PI_KERNEL_AUTO && value != NMPCMC_PI_KERNEL_LANES && value != NMPCMC_PI_KERNEL_WS3 &&
                value != NMPCMC_PI_KERNEL_WS7)
                return NMPCMC_INVALID_ARGUMENT;
            ctx->pi_kernel = (int)value;
            return NMPCMC_OK;
        case NMPCMC_OPT_CTRL_JACOBIANS:
            if (value != NMPCMC_JACOBIANS_ANALYTIC && value != NMPCMC_JACOBIANS_FD) return NMPCMC_INVALID_ARGUMENT;
            ctx->ctrl_fd = value == NMPCMC_JACOBIANS_FD ? 1 : 0;
            return NMPCMC_OK;
        default:
            return NMPCMC_INVALID_ARGUMENT;
    }
}

int nmpcmc_gpu_set_stream(nmpcmc_gpu_ctx* ctx, void* stream) {
    if (ctx == nullptr) return NMPCMC_INVALID_ARGUMENT;
    if (!ctx->subs.empty()) return fail(ctx, NMPCMC_UNSUPPORTED, "set_stream: one stream per device on a multi-device context");
    cudaStream_t next = static_cast<cudaStream_t>(stream);
    if (next == ctx->stream) return NMPCMC_OK;
    cudaSetDevice(ctx->device);
    nmpcmc_gpu_join(ctx);  // lanes stay ordered before later work on the old stream
    // every launch shares the context's workspace and work counter, so work
    // on the new stream must start after everything on the old one: an event
    // on the old stream after the join, waited on by the new stream
    int rc;
    if (ctx->fork == nullptr &&
        (rc = cuda_check(ctx, cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming), "event")) != NMPCMC_OK)
        return rc;
    if ((rc = cuda_check(ctx, cudaEventRecord(ctx->fork, ctx->stream), "event record")) != NMPCMC_OK) return rc;
    if ((rc = cuda_check(ctx, cudaStreamWaitEvent(next, ctx->fork, 0), "stream wait")) != NMPCMC_OK) return rc;
    ctx->stream = next;
    return NMPCMC_OK;
}

int nmpcmc_gpu_run_device(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first_sim,
                          int64_t n_sims, nmpcmc_sim_record* records_dev,
                          nmpcmc_work_counters* counters_dev) {
    if (ctx == nullptr || sc == nullptr || (records_dev == nullptr && n_sims > 0) || n_sims < 0)
        return NMPCMC_INVALID_ARGUMENT;
    if (!ctx->subs.empty())
        return fail(ctx, NMPCMC_UNSUPPORTED, "run_device: device buffers are per device; use run / run_async");
    int32_t nbar = 0;
    int rc = nmpcmc_gpu_validate(sc, &nbar);
    if (rc != NMPCMC_OK) return fail(ctx, rc, "scenario validation failed");
    cudaSetDevice(ctx->device);
    if (ctx->lanes > 1) {
        Lane* l = nullptr;
        if ((rc = lane_begin(ctx, sc->controller, &l)) != NMPCMC_OK) return rc;
        rc = launch(ctx, lane_target(*l), *sc, first_sim, n_sims, nbar, records_dev, counters_dev, nullptr, 0);
        lane_end(l);
        return rc;
    }
    return launch(ctx, main_target(ctx), *sc, first_sim, n_sims, nbar, records_dev, counters_dev, nullptr, 0);
}

int nmpcmc_gpu_run_async(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first_sim,
                         int64_t n_sims, nmpcmc_sim_record* records_out,
                         nmpcmc_work_counters* counters_out) {
    if (ctx == nullptr || sc == nullptr || records_out == nullptr || n_sims < 1)
        return NMPCMC_INVALID_ARGUMENT;
    if (!ctx->subs.empty()) return nmpcmc_host::multi_run_async(ctx, sc, first_sim, n_sims, records_out, counters_out);
    int32_t nbar = 0;
    int rc = nmpcmc_gpu_validate(sc, &nbar);
    if (rc != NMPCMC_OK) return fail(ctx, rc, "scenario validation failed");
    cudaSetDevice(ctx->device);
    Lane* l = nullptr;
    if (ctx->lanes > 1 && (rc = lane_begin(ctx, sc->controller, &l)) != NMPCMC_OK) return rc;
    const Target tg = l ? lane_target(*l) : main_target(ctx);
    void** rec_buf = l ? &l->d_rec : &ctx->d_rec;
    size_t* rec_cap = l ? &l->rec_cap : &ctx->rec_cap;
    void** cnt_buf = l ? &l->d_cnt : &ctx->d_cnt;
    size_t* cnt_cap = l ? &l->cnt_cap : &ctx->cnt_cap;
    const size_t nrec = (size_t)n_sims * sizeof(nmpcmc_sim_record);
    const size_t ncnt = (size_t)n_sims * sizeof(nmpcmc_work_counters);
    if ((rc = ensure(ctx, rec_buf, rec_cap, nrec)) != NMPCMC_OK) return rc;
    if (counters_out && (rc = ensure(ctx, cnt_buf, cnt_cap, ncnt)) != NMPCMC_OK) return rc;
    auto* d_rec = static_cast<nmpcmc_sim_record*>(*rec_buf);
    auto* d_cnt = counters_out ? static_cast<nmpcmc_work_counters*>(*cnt_buf) : nullptr;
    rc = launch(ctx, tg, *sc, first_sim, n_sims, nbar, d_rec, d_cnt, nullptr, 0);
    if (rc == NMPCMC_OK)
        rc = cuda_check(ctx, cudaMemcpyAsync(records_out, d_rec, nrec, cudaMemcpyDeviceToHost, tg.stream),
                        "D2H records");
    if (rc == NMPCMC_OK && counters_out)
        rc = cuda_check(ctx, cudaMemcpyAsync(counters_out, d_cnt, ncnt, cudaMemcpyDeviceToHost, tg.stream),
                        "D2H counters");
    if (l) lane_end(l);
    return rc;
}

int nmpcmc_gpu_join(nmpcmc_gpu_ctx* ctx) {
    if (ctx == nullptr) return NMPCMC_INVALID_ARGUMENT;
    for (nmpcmc_gpu_ctx* s : ctx->subs) nmpcmc_gpu_join(s);
    for (Lane& l : ctx->lane)
        if (l.pending) {
            cudaStreamWaitEvent(ctx->stream, l.done, 0);
            l.pending = false;
        }
    return NMPCMC_OK;
}

int nmpcmc_gpu_wait(nmpcmc_gpu_ctx* ctx) {
    if (ctx == nullptr) return NMPCMC_INVALID_ARGUMENT;
    for (nmpcmc_gpu_ctx* s : ctx->subs) {
        const int rc = nmpcmc_gpu_wait(s);
        if (rc != NMPCMC_OK) return fail(ctx, rc, s->err);
    }
    cudaSetDevice(ctx->device);
    nmpcmc_gpu_join(ctx);
    return cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "kernel execution");
}

int nmpcmc_gpu_run(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first_sim,
                   int64_t n_sims, nmpcmc_sim_record* records_out,
                   nmpcmc_work_counters* counters_out, nmpcmc_aggregate* agg_out) {
    if (ctx == nullptr || sc == nullptr || records_out == nullptr || n_sims < 1)
        return NMPCMC_INVALID_ARGUMENT;
    if (!ctx->subs.empty())
        return nmpcmc_host::multi_run(ctx, sc, first_sim, n_sims, records_out, counters_out, agg_out);
    // one device: launch, statistics on the device (K4) while the records and
    // counters stream back, one host wait
    nmpcmc_sim_record* dr = nullptr;
    nmpcmc_work_counters* dc = nullptr;
    int rc = nmpcmc_host::run_to_device(ctx, *sc, first_sim, n_sims, n_sims, true, &dr, &dc);
    if (rc != NMPCMC_OK) return rc;
    if ((rc = ensure(ctx, &ctx->d_tot, &ctx->tot_cap, 64)) != NMPCMC_OK) return rc;
    if ((rc = nmpcmc_host::counters_sum(ctx, ctx->stream, dc, n_sims, static_cast<long long*>(ctx->d_tot))) !=
        NMPCMC_OK)
        return rc;
    long long tot[8];
    cudaError_t e = cudaMemcpyAsync(tot, ctx->d_tot, sizeof tot, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(records_out, dr, (size_t)n_sims * sizeof(nmpcmc_sim_record), cudaMemcpyDeviceToHost,
                            ctx->stream);
    if (e == cudaSuccess && counters_out)
        e = cudaMemcpyAsync(counters_out, dc, (size_t)n_sims * sizeof(nmpcmc_work_counters), cudaMemcpyDeviceToHost,
                            ctx->stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaMemcpyAsync");
    if ((rc = cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "kernel execution")) != NMPCMC_OK) return rc;
    ctx->last_totals = nmpcmc_work_counters{tot[0], tot[1], tot[2], tot[3], tot[4], tot[5], tot[6], tot[7]};
    ctx->last_rec = dr;
    ctx->last_n = n_sims;
    if (agg_out) return nmpcmc_host::k4_run(ctx, ctx->stream, dr, n_sims, agg_out, 0, nullptr, nullptr, nullptr);
    return NMPCMC_OK;
}

int nmpcmc_gpu_run_traj(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first_sim,
                        int64_t n_sims, nmpcmc_sim_record* records_out, double* traj_out) {
    if (ctx == nullptr || sc == nullptr || records_out == nullptr || traj_out == nullptr || n_sims < 1)
        return NMPCMC_INVALID_ARGUMENT;
    if (!ctx->subs.empty()) {
        // one host thread per device, each on its contiguous block
        const int G = (int)ctx->subs.size();
        const int64_t rows = nmpcmc_gpu_traj_rows(sc);
        std::vector<int> rcs(G, NMPCMC_OK);
        std::vector<std::thread> pool;
        for (int g = 0; g < G; ++g) {
            int64_t b = 0, cnt = 0;
            nmpcmc_gpu_shard_range(n_sims, g, G, &b, &cnt);
            if (cnt == 0) continue;
            pool.emplace_back([&, g, b, cnt] {
                rcs[g] = nmpcmc_gpu_run_traj(ctx->subs[g], sc, first_sim + (uint64_t)b, cnt, records_out + b,
                                             traj_out + (size_t)b * rows * 5);
            });
        }
        for (std::thread& t : pool) t.join();
        for (int g = 0; g < G; ++g)
            if (rcs[g] != NMPCMC_OK) return fail(ctx, rcs[g], ctx->subs[g]->err);
        return NMPCMC_OK;
    }
    int32_t nbar = 0;
    int rc = nmpcmc_gpu_validate(sc, &nbar);
    if (rc != NMPCMC_OK) return fail(ctx, rc, "scenario validation failed");
    const int rows = nmpcmc_gpu_traj_rows(sc);
    cudaSetDevice(ctx->device);
    const size_t nrec = (size_t)n_sims * sizeof(nmpcmc_sim_record);
    const size_t ntraj = (size_t)n_sims * rows * 5 * sizeof(double);
    if ((rc = ensure(ctx, &ctx->d_rec, &ctx->rec_cap, nrec)) != NMPCMC_OK) return rc;
    if ((rc = ensure(ctx, &ctx->d_traj, &ctx->traj_cap, ntraj)) != NMPCMC_OK) return rc;
    // rows a failed run never reaches stay NaN (0xff.. bytes are a NaN pattern)
    if ((rc = cuda_check(ctx, cudaMemsetAsync(ctx->d_traj, 0xff, ntraj, ctx->stream), "memset")) != NMPCMC_OK) return rc;
    cudaError_t cerr = cudaSuccess;
    auto cp = [&](void* dst, const void* src, size_t n, cudaMemcpyKind kind) {
        if (cerr == cudaSuccess && n > 0) cerr = cudaMemcpyAsync(dst, src, n, kind, ctx->stream);
    };
    auto* d_rec = static_cast<nmpcmc_sim_record*>(ctx->d_rec);
    auto* d_traj = static_cast<double*>(ctx->d_traj);
    if ((rc = launch(ctx, main_target(ctx), *sc, first_sim, n_sims, nbar, d_rec, nullptr, d_traj, rows)) != NMPCMC_OK)
        return rc;
    cp(records_out, d_rec, nrec, cudaMemcpyDeviceToHost);
    cp(traj_out, d_traj, ntraj, cudaMemcpyDeviceToHost);
    if (cerr != cudaSuccess) return cuda_check(ctx, cerr, "cudaMemcpyAsync");
    return cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "kernel execution");
}

}  // extern "C"

namespace nmpcmc_host {

/// Launch [first, first + n) on the context's own stream into its device
/// record / counter buffers, sized for at least `cap` samples (a sharded run
/// sizes every block's buffer for the largest block, so an empty block still
/// owns a buffer the all-gather can read). Enqueued only.
int run_to_device(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario& sc, uint64_t first, int64_t n, int64_t cap,
                  bool want_counters, nmpcmc_sim_record** d_rec, nmpcmc_work_counters** d_cnt) {
    int32_t nbar = 0;
    int rc = nmpcmc_gpu_validate(&sc, &nbar);
    if (rc != NMPCMC_OK) return fail(ctx, rc, "scenario validation failed");
    cudaSetDevice(ctx->device);
    nmpcmc_gpu_join(ctx);
    const int64_t c = std::max<int64_t>(std::max(cap, n), 1);
    if ((rc = ensure(ctx, &ctx->d_rec, &ctx->rec_cap, (size_t)c * sizeof(nmpcmc_sim_record))) != NMPCMC_OK) return rc;
    if (want_counters &&
        (rc = ensure(ctx, &ctx->d_cnt, &ctx->cnt_cap, (size_t)c * sizeof(nmpcmc_work_counters))) != NMPCMC_OK)
        return rc;
    *d_rec = static_cast<nmpcmc_sim_record*>(ctx->d_rec);
    *d_cnt = want_counters ? static_cast<nmpcmc_work_counters*>(ctx->d_cnt) : nullptr;
    return launch(ctx, main_target(ctx), sc, first, n, nbar, *d_rec, *d_cnt, nullptr, 0);
}

}  // namespace nmpcmc_host

// ------------------------------------------------------- unit entry points
namespace {

template <typename T>
int scratch_roundtrip(nmpcmc_gpu_ctx* ctx, const void* in, size_t in_bytes, size_t out_bytes,
                      void* out, T&& kernel_launch) {
    int rc = ensure(ctx, &ctx->d_scratch, &ctx->scratch_cap, in_bytes + out_bytes + 256);
    if (rc != NMPCMC_OK) return rc;
    char* base = static_cast<char*>(ctx->d_scratch);
    char* d_out = base + ((in_bytes + 255) / 256) * 256;
    if (in_bytes &&
        (rc = cuda_check(ctx, cudaMemcpyAsync(base, in, in_bytes, cudaMemcpyHostToDevice, ctx->stream), "H2D")) !=
            NMPCMC_OK)
        return rc;
    kernel_launch(base, d_out);
    if ((rc = cuda_check(ctx, cudaGetLastError(), "unit kernel launch")) != NMPCMC_OK) return rc;
    if ((rc = cuda_check(ctx, cudaMemcpyAsync(out, d_out, out_bytes, cudaMemcpyDeviceToHost, ctx->stream), "D2H")) !=
        NMPCMC_OK)
        return rc;
    return cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "unit kernel");
}

}  // namespace

extern "C" {

int nmpcmc_gpu_philox_blocks(nmpcmc_gpu_ctx* ctx, const uint32_t* in, int64_t n, uint32_t* out) {
    if (ctx == nullptr || in == nullptr || out == nullptr || n < 1) return NMPCMC_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    return scratch_roundtrip(ctx, in, n * 6 * sizeof(uint32_t), n * 4 * sizeof(uint32_t), out,
                             [&](char* din, char* dout) {
                                 nmpcmc_launch::launch_philox(reinterpret_cast<uint32_t*>(din), n,
                                                              reinterpret_cast<uint32_t*>(dout), ctx->stream);
                             });
}

int nmpcmc_gpu_normals(nmpcmc_gpu_ctx* ctx, uint64_t seed, uint64_t stream, int64_t n, double* out) {
    if (ctx == nullptr || out == nullptr || n < 1) return NMPCMC_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    return scratch_roundtrip(ctx, nullptr, 0, n * sizeof(double), out, [&](char*, char* dout) {
        nmpcmc_launch::launch_normals(seed, stream, n, reinterpret_cast<double*>(dout), ctx->stream);
    });
}

int nmpcmc_gpu_libm(nmpcmc_gpu_ctx* ctx, int32_t fn, const double* x, int64_t n, double* out) {
    if (ctx == nullptr || x == nullptr || out == nullptr || n < 1 || fn < 0 || fn > 3)
        return NMPCMC_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    return scratch_roundtrip(ctx, x, n * sizeof(double), n * sizeof(double), out, [&](char* din, char* dout) {
        nmpcmc_launch::launch_libm(fn, reinterpret_cast<double*>(din), n, reinterpret_cast<double*>(dout),
                                   ctx->stream);
    });
}

}  // extern "C"

// --------------------------------------------- FP64 peak (roofline denominator)
// MEASURED_PEAKS.json carries HBM and bf16 only; the closed loop runs on the
// FP64 CUDA cores, so its roofline denominator is measured here: independent
// DFMA chains, grid = 8 x SMs x 256 threads, 2 flops per DFMA (k_misc.cu).
extern "C" int nmpcmc_gpu_fp64_peak(nmpcmc_gpu_ctx* ctx, int use_fma, double* tflops_out) {
    if (ctx == nullptr || tflops_out == nullptr) return NMPCMC_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    const int blocks = ctx->sm_count * 8, threads = 256, iters = 4096;
    int rc = ensure(ctx, &ctx->d_scratch, &ctx->scratch_cap, (size_t)blocks * threads * sizeof(double));
    if (rc != NMPCMC_OK) return rc;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0, ctx->stream);
        nmpcmc_launch::launch_fp64_peak(blocks, threads, static_cast<double*>(ctx->d_scratch), iters, use_fma,
                                        ctx->stream);
        cudaEventRecord(e1, ctx->stream);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)blocks * threads * iters * 64.0 * (use_fma ? 2.0 : 1.0);
        if (rep > 0) best = std::max(best, ops / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *tflops_out = best;
    return cuda_check(ctx, cudaGetLastError(), "fp64 peak");
}

// ------------------------------------------------------------ batched QP
extern "C" int64_t nmpcmc_qp_stage_doubles(int32_t n_x, int32_t n_u) {
    return nmpcmc_launch::qp_stage_doubles(n_x, n_u);
}
extern "C" int64_t nmpcmc_qp_solution_doubles(int32_t N, int32_t n_x, int32_t n_u) {
    return nmpcmc_launch::qp_solution_doubles(N, n_x, n_u);
}

extern "C" int nmpcmc_gpu_solve_qp_batch(nmpcmc_gpu_ctx* ctx, const nmpcmc_qp_dims* dims, int64_t batch,
                                         const double* stages, double* solutions, int32_t* status,
                                         int32_t* iterations) {
    if (ctx == nullptr || dims == nullptr || batch < 0 || (batch > 0 && (!stages || !solutions || !status || !iterations)))
        return NMPCMC_INVALID_ARGUMENT;
    const nmpcmc_qp_dims d = *dims;
    // QP validate (qp.cpp:21-58): at least one input stage and positive blocks
    if (d.N < 1 || d.n_x < 1 || d.n_u < 1) return fail(ctx, NMPCMC_DIMENSION_MISMATCH, "QP dimensions");
    if (d.n_x > nmpcmc_launch::qp_max_nx() || d.n_u > nmpcmc_launch::qp_max_nu())
        return fail(ctx, NMPCMC_UNSUPPORTED, "QP batch: n_x <= 8 and n_u <= 4 on device");
    if (d.mode != 0 && d.mode != 1) return fail(ctx, NMPCMC_INVALID_ARGUMENT, "QP batch: mode");
    if (batch == 0) return NMPCMC_OK;
    cudaSetDevice(ctx->device);
    const int64_t SB = nmpcmc_launch::qp_stage_doubles(d.n_x, d.n_u);
    const int64_t SO = nmpcmc_launch::qp_solution_doubles(d.N, d.n_x, d.n_u);
    const size_t in_b = (size_t)batch * (d.N + 1) * SB * sizeof(double);
    const size_t out_b = (size_t)batch * SO * sizeof(double);
    const size_t st_b = (size_t)batch * 2 * sizeof(int32_t);
    const int64_t slots = nmpcmc_launch::qp_slots(ctx->sm_count, batch);
    const size_t ws_b = (size_t)slots * (size_t)nmpcmc_launch::qp_ws_doubles(d.N, d.n_x, d.n_u) * sizeof(double);
    int rc = ensure(ctx, &ctx->d_scratch, &ctx->scratch_cap, in_b + out_b + st_b + 256);
    if (rc == NMPCMC_OK) rc = ensure(ctx, &ctx->d_ws, &ctx->ws_cap, ws_b);
    if (rc != NMPCMC_OK) return rc;
    char* base = static_cast<char*>(ctx->d_scratch);
    auto* d_in = reinterpret_cast<double*>(base);
    auto* d_out = reinterpret_cast<double*>(base + in_b);
    auto* d_st = reinterpret_cast<int32_t*>(base + in_b + out_b);
    cudaError_t cerr = cudaSuccess;
    auto cp = [&](void* dst, const void* src, size_t n, cudaMemcpyKind kind) {
        if (cerr == cudaSuccess && n > 0) cerr = cudaMemcpyAsync(dst, src, n, kind, ctx->stream);
    };
    cp(d_in, stages, in_b, cudaMemcpyHostToDevice);
    nmpcmc_launch::launch_qp_batch(d, batch, d_in, d_out, d_st, d_st + batch, static_cast<double*>(ctx->d_ws), slots,
                                   ctx->stream);
    if ((rc = cuda_check(ctx, cudaGetLastError(), "qp_batch_kernel launch")) != NMPCMC_OK) return rc;
    cp(solutions, d_out, out_b, cudaMemcpyDeviceToHost);
    cp(status, d_st, (size_t)batch * sizeof(int32_t), cudaMemcpyDeviceToHost);
    cp(iterations, d_st + batch, (size_t)batch * sizeof(int32_t), cudaMemcpyDeviceToHost);
    if (cerr != cudaSuccess) return cuda_check(ctx, cerr, "cudaMemcpyAsync");
    return cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "qp_batch_kernel");
}

// ------------------------------------------------------------ batched OCP
extern "C" int nmpcmc_gpu_solve_ocp_batch(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, int64_t batch,
                                          const double* x0, const double* t0, const double* xi0, double* xi,
                                          double* lambda, double* pi_l, double* pi_u, int32_t* converged,
                                          int32_t* status) {
    if (ctx == nullptr || sc == nullptr || batch < 0) return NMPCMC_INVALID_ARGUMENT;
    if (batch > 0 && (!x0 || !t0 || !xi || !lambda || !pi_l || !pi_u || !converged || !status))
        return NMPCMC_INVALID_ARGUMENT;
    if (sc->controller != NMPCMC_CTRL_NMPC) return fail(ctx, NMPCMC_INVALID_ARGUMENT, "OCP batch: NMPC scenario");
    int32_t nbar = 0;
    int rc = nmpcmc_gpu_validate(sc, &nbar);
    if (rc != NMPCMC_OK) return fail(ctx, rc, "scenario validation failed");
    if (batch == 0) return NMPCMC_OK;
    cudaSetDevice(ctx->device);
    const int nx = sc->ctrl_variant == NMPCMC_THREE_STATE ? 3 : 1;
    const int64_t L = (int64_t)sc->N * (1 + nx), NN = (int64_t)sc->N * nx;
    const size_t b_x0 = batch * nx * 8, b_t0 = batch * 8, b_xi = batch * L * 8, b_lam = batch * NN * 8,
                 b_pi = batch * sc->N * 8, b_i = batch * 4;
    auto rnd = [](size_t n) { return (n + 255) / 256 * 256; };
    const size_t total =
        rnd(b_x0) + rnd(b_t0) + (xi0 ? rnd(b_xi) : 0) + rnd(b_xi) + rnd(b_lam) + 2 * rnd(b_pi) + 2 * rnd(b_i);
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
    // one-state OCPs with N <= 255 run on K3's phases (shared-memory Riccati
    // sweeps, certified sqrt/division); the rest on K3w's generic path
    const bool k3 = sc->ctrl_variant == NMPCMC_ONE_STATE && sc->N <= 255;
    int64_t blocks = 0;
    if (k3) {
        size_t gbytes = 0;
        nmpcmc_launch::nmpc_gws_need(*sc, ctx->sm_count, batch, &gbytes, &blocks);
        if ((rc = ensure(ctx, &ctx->d_gws, &ctx->gws_cap, gbytes)) != NMPCMC_OK) return rc;
    } else {
        blocks = nmpcmc_launch::genw_blocks(*sc, ctx->sm_count, batch);
        const size_t ws_b = (size_t)blocks * (size_t)nmpcmc_launch::gen_ws_doubles(*sc) * sizeof(double);
        if ((rc = ensure(ctx, &ctx->d_ws, &ctx->ws_cap, ws_b)) != NMPCMC_OK) return rc;
    }
    if ((rc = ensure(ctx, &ctx->d_counter, &ctx->counter_cap, 256)) != NMPCMC_OK) return rc;
    cudaError_t cerr = cudaSuccess;
    auto cp = [&](void* dst, const void* src, size_t n, cudaMemcpyKind kind) {
        if (cerr == cudaSuccess && n > 0) cerr = cudaMemcpyAsync(dst, src, n, kind, ctx->stream);
    };
    cp(d_x0, x0, b_x0, cudaMemcpyHostToDevice);
    cp(d_t0, t0, b_t0, cudaMemcpyHostToDevice);
    if (xi0) cp(d_xi0, xi0, b_xi, cudaMemcpyHostToDevice);
    rc = k3 ? nmpcmc_launch::launch_ocp1(*sc, batch, d_x0, d_t0, d_xi0, d_xi, d_lam, d_pil, d_piu, d_conv, d_st,
                                      ctx->sm_count, static_cast<double*>(ctx->d_gws), blocks,
                                      static_cast<unsigned long long*>(ctx->d_counter), ctx->stream)
            : nmpcmc_launch::launch_ocp_batch(*sc, batch, d_x0, d_t0, d_xi0, d_xi, d_lam, d_pil, d_piu, d_conv,
                                                d_st, static_cast<double*>(ctx->d_ws), blocks,
                                                static_cast<unsigned long long*>(ctx->d_counter), ctx->stream);
    if (rc != NMPCMC_OK)
        return fail(ctx, rc, "OCP batch: horizon too long for the shared-memory sweep arrays");
    if ((rc = cuda_check(ctx, cudaGetLastError(), "ocp_batch_kernel launch")) != NMPCMC_OK) return rc;
    cp(xi, d_xi, b_xi, cudaMemcpyDeviceToHost);
    cp(lambda, d_lam, b_lam, cudaMemcpyDeviceToHost);
    cp(pi_l, d_pil, b_pi, cudaMemcpyDeviceToHost);
    cp(pi_u, d_piu, b_pi, cudaMemcpyDeviceToHost);
    cp(converged, d_conv, b_i, cudaMemcpyDeviceToHost);
    cp(status, d_st, b_i, cudaMemcpyDeviceToHost);
    if (cerr != cudaSuccess) return cuda_check(ctx, cerr, "cudaMemcpyAsync");
    return cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "ocp_batch_kernel");
}
