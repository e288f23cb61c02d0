// ctx_internal.h -- the context object behind the opaque nmpcmc_gpu_ctx
// handle, shared by the translation units of libnmpcmc_gpu.so (not installed).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "nccl_dl.h"
#include "nmpcmc_gpu.h"

/// Where one launch runs and the workspace it owns. The context's own target
/// uses ctx->stream; with NMPCMC_OPT_LANES = 2, NMPC launches alternate
/// between two lanes and PI launches use a third, each lane with its own
/// stream and workspace, so a batch's drain overlaps the next batch.
struct Lane {
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    bool pending = false;
    void* d_gws = nullptr;
    size_t gws_cap = 0;
    void* d_counter = nullptr;
    size_t counter_cap = 0;
    void* d_ws = nullptr;
    size_t ws_cap = 0;
    void* d_rec = nullptr;
    size_t rec_cap = 0;
    void* d_cnt = nullptr;
    size_t cnt_cap = 0;
};

struct nmpcmc_gpu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    void* d_rec = nullptr;
    size_t rec_cap = 0;
    void* d_cnt = nullptr;
    size_t cnt_cap = 0;
    void* d_traj = nullptr;
    size_t traj_cap = 0;
    void* d_scratch = nullptr;
    size_t scratch_cap = 0;
    void* d_ws = nullptr;  // generic-kernel / K5 workspace
    size_t ws_cap = 0;
    void* d_gws = nullptr;  // K3 per-block global workspace
    size_t gws_cap = 0;
    void* d_counter = nullptr;  // K3 work counter
    size_t counter_cap = 0;
    void* d_k4 = nullptr;  // K4 statistics workspace
    size_t k4_cap = 0;
    void* d_all = nullptr;  // gathered records of a sharded run
    size_t all_cap = 0;
    void* d_state = nullptr;  // controller-level API staging
    size_t state_cap = 0;
    void* d_tot = nullptr;  // summed work counters (8 x int64)
    size_t tot_cap = 0;
    int sm_count = 0;
    int nmpc_kernel = NMPCMC_NMPC_KERNEL_WARP;  // which NMPC kernel to launch
    int tps_warps_per_sm = 8;                   // K3b resident warps per SM
    int ctrl_fd = 0;                            // NMPCMC_OPT_CTRL_JACOBIANS: 1 = finite differences
    cudaStream_t own = nullptr;                 // the stream ctx_create made (set_stream may replace ctx->stream)
    int lanes = 1;                              // NMPCMC_OPT_LANES
    int pi_kernel = NMPCMC_PI_KERNEL_AUTO;      // NMPCMC_OPT_PI_KERNEL
    int next_nmpc_lane = 0;
    Lane lane[3];
    cudaEvent_t fork = nullptr;
    // ---- multi-device (nmpcmc_gpu_ctx_create_multi): one sub-context per
    // device id; the parent itself runs on device_ids[0] (K4, unit calls)
    std::vector<nmpcmc_gpu_ctx*> subs;
    std::vector<ncclComm_t> comms;  // ncclCommInitAll over distinct device ids
    // ---- one process per GPU (nmpcmc_gpu_comm_init)
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
    nmpcmc_work_counters last_totals{};  // totals of the last run over all devices / ranks
    const nmpcmc_sim_record* last_rec = nullptr;  // gathered records of the last run (device)
    int64_t last_n = 0;
};

namespace nmpcmc_host {

/// Message of the last failed context creation on this thread (no context
/// exists to hold it); nmpcmc_gpu_last_error(NULL) returns it.
inline std::string& create_error() {
    static thread_local std::string s;
    return s;
}

inline int fail(nmpcmc_gpu_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

inline int cuda_check(nmpcmc_gpu_ctx* ctx, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return NMPCMC_OK;
    return fail(ctx, NMPCMC_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

inline int ensure(nmpcmc_gpu_ctx* ctx, void** buf, size_t* cap, size_t need) {
    if (need <= *cap) return NMPCMC_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    cudaError_t e = cudaMalloc(buf, need);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaMalloc");
    *cap = need;
    return NMPCMC_OK;
}

/// K4 on records already on ctx->device (enqueued on `stream`, synchronous):
/// aggregate_stats into agg (may be NULL) and, when counts != NULL,
/// phi_histogram with `bins` (<= 0: Freedman-Diaconis) into edges/counts.
int k4_run(nmpcmc_gpu_ctx* ctx, cudaStream_t stream, const nmpcmc_sim_record* d_rec, int64_t n,
           nmpcmc_aggregate* agg, int32_t bins, double* edges, int32_t* counts, int32_t* nbins);

/// Launch [first, first + n) on ctx->stream into ctx's device record /
/// counter buffers sized for >= cap samples (nmpcmc_gpu.cu). Enqueued only.
int run_to_device(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario& sc, uint64_t first, int64_t n, int64_t cap,
                  bool want_counters, nmpcmc_sim_record** d_rec, nmpcmc_work_counters** d_cnt);

/// Multi-device forms (nmpcmc_multi.cu) behind nmpcmc_gpu_run / _run_async.
int multi_run(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first, int64_t n, nmpcmc_sim_record* rec_out,
              nmpcmc_work_counters* cnt_out, nmpcmc_aggregate* agg_out);
int multi_run_async(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first, int64_t n,
                    nmpcmc_sim_record* rec_out, nmpcmc_work_counters* cnt_out);

/// Sum of per-sample work counters on the device into d_out (8 int64).
int counters_sum(nmpcmc_gpu_ctx* ctx, cudaStream_t stream, const nmpcmc_work_counters* d_cnt, int64_t n,
                 long long* d_out);

}  // namespace nmpcmc_host
