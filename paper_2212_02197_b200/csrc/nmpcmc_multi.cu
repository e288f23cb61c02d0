// nmpcmc_multi.cu -- device statistics (K4) and the multi-device forms of
// run_monte_carlo.
//
// The reference's run_monte_carlo(sc, n_sims, workers) (montecarlo.cpp:213-251)
// spreads samples over a thread pool on one machine. Here:
//   * one process, several GPUs: nmpcmc_gpu_ctx_create_multi(device_ids, n)
//     makes one sub-context per device; nmpcmc_gpu_run shards the global index
//     range into contiguous blocks, one host thread per device launches its
//     block and copies its records straight into the caller's buffer, then
//     the records are all-gathered over NCCL (ncclCommInitAll) onto
//     device_ids[0], where K4 computes aggregate_stats; the work counters are
//     all-reduced (int64 sum);
//   * one process per GPU (torchrun-style): nmpcmc_gpu_comm_init joins an
//     NCCL communicator, nmpcmc_gpu_run_sharded runs this rank's block,
//     all-gathers the records so every rank holds all of them in index order,
//     all-reduces the counters and runs K4 locally.
// Every RNG stream is keyed by the global sample index, so the records are
// bitwise independent of the number of devices and ranks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ctx_internal.h"
#include "stats_kernel.cuh"

namespace nmpcmc_host {

namespace {

size_t rnd256(size_t n) { return (n + 255) / 256 * 256; }

int nccl_check(nmpcmc_gpu_ctx* ctx, ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return NMPCMC_OK;
    return fail(ctx, NMPCMC_CUDA_ERROR, std::string(what) + ": " + nccl().GetErrorString(r));
}

/// The per-sample fields K4 reads, unpacked once (coalesced 8 / 1 B arrays).
__global__ void unpack_kernel(const nmpcmc_sim_record* rec, int64_t n, double* phi, unsigned char* okf,
                              unsigned char* finf) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double p = rec[i].phi;
        phi[i] = p;
        okf[i] = rec[i].failed == 0;
        finf[i] = isfinite(p) != 0;
    }
}

/// Sum of the per-sample work counters (int64, exact in any order).
__global__ void counters_sum_kernel(const nmpcmc_work_counters* c, int64_t n, long long* out) {
    long long a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const long long* v = reinterpret_cast<const long long*>(c + i);
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] += v[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        long long s = a[k];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0 && s != 0) atomicAdd(reinterpret_cast<unsigned long long*>(out + k),
                                                           (unsigned long long)s);
    }
}

int grid_for(const nmpcmc_gpu_ctx* ctx, int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    const int64_t cap = (int64_t)std::max(ctx->sm_count, 1) * 8;
    return (int)std::max<int64_t>(1, std::min(g, cap));
}

}  // namespace

int counters_sum(nmpcmc_gpu_ctx* ctx, cudaStream_t stream, const nmpcmc_work_counters* d_cnt, int64_t n,
                 long long* d_out) {
    int rc = cuda_check(ctx, cudaMemsetAsync(d_out, 0, 8 * sizeof(long long), stream), "memset");
    if (rc != NMPCMC_OK || n == 0) return rc;
    counters_sum_kernel<<<grid_for(ctx, n, 256), 256, 0, stream>>>(d_cnt, n, d_out);
    return cuda_check(ctx, cudaGetLastError(), "counters_sum launch");
}

int k4_run(nmpcmc_gpu_ctx* ctx, cudaStream_t stream, const nmpcmc_sim_record* d_rec, int64_t n,
           nmpcmc_aggregate* agg, int32_t bins, double* edges, int32_t* counts, int32_t* nbins) {
    namespace k4 = nmpcmc_dev::k4;
    if (n < 0 || n > 0x7fffffffLL) return fail(ctx, NMPCMC_INVALID_ARGUMENT, "K4: sample count out of range");
    if (counts != nullptr && bins > 200) return fail(ctx, NMPCMC_INVALID_ARGUMENT, "K4: at most 200 bins");
    const int ni = (int)n;
    // CUB temporary storage: the larger of the selection and the sort
    size_t t_sel = 0, t_sort = 0;
    cub::DeviceSelect::Flagged(nullptr, t_sel, (const double*)nullptr, (const unsigned char*)nullptr,
                               (double*)nullptr, (int*)nullptr, ni);
    cub::DeviceRadixSort::SortKeys(nullptr, t_sort, (const double*)nullptr, (double*)nullptr, ni);
    const size_t tb = std::max<size_t>(std::max(t_sel, t_sort), 256);
    const size_t nd = rnd256((size_t)n * 8), nb = rnd256((size_t)n);
    const size_t total = 5 * nd + 2 * nb + rnd256(sizeof(k4::Totals)) + rnd256(64) + rnd256(8 * 8) +
                        rnd256(sizeof(nmpcmc_aggregate)) + rnd256(200 * 4) + tb;
    int rc = ensure(ctx, &ctx->d_k4, &ctx->k4_cap, total);
    if (rc != NMPCMC_OK) return rc;
    char* p = static_cast<char*>(ctx->d_k4);
    auto take = [&](size_t bytes) {
        char* a = p;
        p += bytes;
        return a;
    };
    auto* phi = reinterpret_cast<double*>(take(nd));
    auto* ok = reinterpret_cast<double*>(take(nd));
    auto* fin = reinterpret_cast<double*>(take(nd));
    auto* sorted_ok = reinterpret_cast<double*>(take(nd));
    auto* sorted_fin = reinterpret_cast<double*>(take(nd));
    auto* okf = reinterpret_cast<unsigned char*>(take(nb));
    auto* finf = reinterpret_cast<unsigned char*>(take(nb));
    auto* tot = reinterpret_cast<k4::Totals*>(take(rnd256(sizeof(k4::Totals))));
    auto* nsel = reinterpret_cast<int*>(take(rnd256(64)));
    auto* sc = reinterpret_cast<double*>(take(rnd256(8 * 8)));  // sum, ss, mean, -, lo, hi, q25, q75
    auto* d_agg = reinterpret_cast<nmpcmc_aggregate*>(take(rnd256(sizeof(nmpcmc_aggregate))));
    auto* d_counts = reinterpret_cast<int*>(take(rnd256(200 * 4)));
    void* temp = take(tb);

    cudaError_t e = cudaMemsetAsync(tot, 0, sizeof(k4::Totals), stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(nsel, 0, 64, stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "K4 memset");
    if (n > 0) {
        k4::totals_kernel<<<grid_for(ctx, n, 256), 256, 0, stream>>>(d_rec, n, tot);
        unpack_kernel<<<grid_for(ctx, n, 256), 256, 0, stream>>>(d_rec, n, phi, okf, finf);
        size_t t1 = tb;
        e = cub::DeviceSelect::Flagged(temp, t1, phi, okf, ok, nsel, ni, stream);
        if (e == cudaSuccess) {
            t1 = tb;
            e = cub::DeviceSelect::Flagged(temp, t1, phi, finf, fin, nsel + 1, ni, stream);
        }
        if (e != cudaSuccess) return cuda_check(ctx, e, "K4 select");
    }
    // the host needs the selected counts to size the serial sums and sorts
    int hsel[2] = {0, 0};
    if (n > 0) {
        e = cudaMemcpyAsync(hsel, nsel, 2 * sizeof(int), cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) return cuda_check(ctx, e, "K4 counts");
    }
    const int n_ok = hsel[0], n_fin = hsel[1];
    if (n_ok > 0) {
        k4::serial_sum_kernel<false><<<1, 32, 0, stream>>>(ok, n_ok, nullptr, sc + 0);
        k4::mean_kernel<<<1, 1, 0, stream>>>(tot, n, sc + 0, sc + 2);
        k4::serial_sum_kernel<true><<<1, 32, 0, stream>>>(ok, n_ok, sc + 2, sc + 1);
        size_t t2 = tb;
        e = cub::DeviceRadixSort::SortKeys(temp, t2, ok, sorted_ok, n_ok, 0, 64, stream);
        if (e != cudaSuccess) return cuda_check(ctx, e, "K4 sort");
    }
    // the finite set equals the ok set unless a non-failed sample has a
    // non-finite phi; sort it separately only then
    const double* sfin = sorted_ok;
    if (n_fin > 0 && n_fin != n_ok) {
        size_t t2 = tb;
        e = cub::DeviceRadixSort::SortKeys(temp, t2, fin, sorted_fin, n_fin, 0, 64, stream);
        if (e != cudaSuccess) return cuda_check(ctx, e, "K4 sort");
        sfin = sorted_fin;
    }
    k4::finish_kernel<<<1, 1, 0, stream>>>(tot, n, sc + 0, sc + 1, sorted_ok, sfin, d_agg, sc + 4);
    if ((rc = cuda_check(ctx, cudaGetLastError(), "K4 kernels")) != NMPCMC_OK) return rc;
    nmpcmc_aggregate h_agg;
    double h_scal[4] = {0, 0, 0, 0};
    e = cudaMemcpyAsync(&h_agg, d_agg, sizeof h_agg, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess && n_fin > 0) e = cudaMemcpyAsync(h_scal, sc + 4, sizeof h_scal, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "K4 results");
    if (agg) *agg = h_agg;
    if (counts == nullptr) return NMPCMC_OK;
    if (edges == nullptr || nbins == nullptr) return fail(ctx, NMPCMC_INVALID_ARGUMENT, "K4: histogram outputs");
    // phi_histogram (montecarlo.cpp:268-304): the bin rule on the host with
    // the reference's own cbrt / ceil, the counting loop on the device
    if (n_fin == 0) {
        edges[0] = 0.0;
        edges[1] = 1.0;
        counts[0] = 0;
        *nbins = 1;
        return NMPCMC_OK;
    }
    const double lo = h_scal[0], hi = h_scal[1];
    if (bins <= 0) {
        const double iqr = h_scal[3] - h_scal[2];
        const double width = 2.0 * iqr / std::cbrt(static_cast<double>(n_fin));
        bins = width > 0.0 ? static_cast<int>(std::ceil((hi - lo) / width)) : 1;
        bins = std::clamp(bins, 1, 200);
    }
    if (hi <= lo) {
        edges[0] = lo;
        edges[1] = lo + 1.0;
        counts[0] = n_fin;
        *nbins = 1;
        return NMPCMC_OK;
    }
    const double width = (hi - lo) / bins;
    for (int b = 0; b <= bins; ++b) edges[b] = lo + b * width;
    edges[bins] = hi;
    e = cudaMemsetAsync(d_counts, 0, 200 * sizeof(int), stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "K4 memset");
    k4::hist_kernel<<<grid_for(ctx, n_fin, 256), 256, 0, stream>>>(sfin, n_fin, lo, width, bins, d_counts);
    e = cudaMemcpyAsync(counts, d_counts, (size_t)bins * sizeof(int), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_check(ctx, e, "K4 histogram");
    *nbins = bins;
    return NMPCMC_OK;
}

}  // namespace nmpcmc_host

// ------------------------------------------------------------ multi-device
namespace nmpcmc_host {
namespace {

int64_t shard_chunk(int64_t n, int G) { return G > 0 ? (n + G - 1) / G : n; }

int ensure_tot(nmpcmc_gpu_ctx* ctx) {
    return ensure(ctx, &ctx->d_tot, &ctx->tot_cap, 8 * sizeof(long long));
}

void add_totals(nmpcmc_work_counters& acc, const long long* t) {
    acc.control_steps += t[0];
    acc.shoot_full += t[1];
    acc.shoot_fonly += t[2];
    acc.ipm_stage_iters += t[3];
    acc.sqp_stage_iters += t[4];
    acc.qp_solves += t[5];
    acc.sqp_iterations += t[6];
    acc.ls_evals += t[7];
}

/// One device's block of a multi-device run: launch, copy its records (and
/// counters) into the caller's buffers at the block's offset, and sum its
/// counters on the device. Runs on its own host thread.
int run_block(nmpcmc_gpu_ctx* sub, const nmpcmc_scenario& sc, uint64_t first, int64_t cnt, int64_t cap,
              nmpcmc_sim_record* rec_out, nmpcmc_work_counters* cnt_out) {
    nmpcmc_sim_record* dr = nullptr;
    nmpcmc_work_counters* dc = nullptr;
    int rc = run_to_device(sub, sc, first, cnt, cap, true, &dr, &dc);
    if (rc == NMPCMC_OK) rc = ensure_tot(sub);
    if (rc == NMPCMC_OK && cnt > 0 && rec_out)
        rc = cuda_check(sub, cudaMemcpyAsync(rec_out, dr, (size_t)cnt * sizeof(nmpcmc_sim_record),
                                             cudaMemcpyDeviceToHost, sub->stream), "D2H records");
    if (rc == NMPCMC_OK && cnt > 0 && cnt_out)
        rc = cuda_check(sub, cudaMemcpyAsync(cnt_out, dc, (size_t)cnt * sizeof(nmpcmc_work_counters),
                                             cudaMemcpyDeviceToHost, sub->stream), "D2H counters");
    if (rc == NMPCMC_OK) rc = counters_sum(sub, sub->stream, dc, cnt, static_cast<long long*>(sub->d_tot));
    if (rc == NMPCMC_OK) rc = cuda_check(sub, cudaStreamSynchronize(sub->stream), "kernel execution");
    return rc;
}

}  // namespace

int multi_run(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first, int64_t n, nmpcmc_sim_record* rec_out,
              nmpcmc_work_counters* cnt_out, nmpcmc_aggregate* agg_out) {
    const int G = (int)ctx->subs.size();
    const int64_t c = shard_chunk(n, G);
    std::vector<int> rcs(G, NMPCMC_OK);
    std::vector<std::thread> pool;
    pool.reserve(G);
    for (int g = 0; g < G; ++g) {
        int64_t b = 0, cnt = 0;
        nmpcmc_gpu_shard_range(n, g, G, &b, &cnt);
        pool.emplace_back([&, g, b, cnt] {
            rcs[g] = run_block(ctx->subs[g], *sc, first + (uint64_t)b, cnt, c, rec_out + b, cnt_out ? cnt_out + b : nullptr);
        });
    }
    for (std::thread& t : pool) t.join();
    for (int g = 0; g < G; ++g)
        if (rcs[g] != NMPCMC_OK) return fail(ctx, rcs[g], "device " + std::to_string(ctx->subs[g]->device) + ": " +
                                                              ctx->subs[g]->err);
    // the one exchange (§8(e)): gather the 24 B records onto device_ids[0]
    // and sum the counters
    nmpcmc_gpu_ctx* root = ctx->subs[0];
    int rc;
    const size_t rec_b = (size_t)c * sizeof(nmpcmc_sim_record);
    nmpcmc_work_counters tot{};
    if (!ctx->comms.empty()) {
        for (nmpcmc_gpu_ctx* s : ctx->subs) {
            cudaSetDevice(s->device);
            if ((rc = ensure(s, &s->d_all, &s->all_cap, rec_b * G + 256)) != NMPCMC_OK) return fail(ctx, rc, s->err);
        }
        const NcclApi& N = nccl();
        if ((rc = nccl_check(ctx, N.GroupStart(), "ncclGroupStart")) != NMPCMC_OK) return rc;
        for (int g = 0; g < G; ++g) {
            nmpcmc_gpu_ctx* s = ctx->subs[g];
            N.AllGather(s->d_rec, s->d_all, rec_b, ncclUint8, ctx->comms[g], s->stream);
            N.AllReduce(s->d_tot, s->d_tot, 8, ncclInt64, ncclSum, ctx->comms[g], s->stream);
        }
        if ((rc = nccl_check(ctx, N.GroupEnd(), "ncclGroupEnd (all-gather records, all-reduce counters)")) != NMPCMC_OK)
            return rc;
        for (nmpcmc_gpu_ctx* s : ctx->subs) {
            cudaSetDevice(s->device);
            if ((rc = cuda_check(ctx, cudaStreamSynchronize(s->stream), "NCCL gather")) != NMPCMC_OK) return rc;
        }
        long long h[8];
        cudaSetDevice(root->device);
        if ((rc = cuda_check(ctx, cudaMemcpy(h, root->d_tot, sizeof h, cudaMemcpyDeviceToHost), "D2H totals")) != NMPCMC_OK)
            return rc;
        add_totals(tot, h);
    } else {
        // several blocks on one GPU (repeated device ids) or a single device:
        // peer / device copies instead of a communicator
        cudaSetDevice(root->device);
        if ((rc = ensure(root, &root->d_all, &root->all_cap, rec_b * G + 256)) != NMPCMC_OK) return fail(ctx, rc, root->err);
        for (int g = 0; g < G; ++g) {
            nmpcmc_gpu_ctx* s = ctx->subs[g];
            int64_t b = 0, cnt = 0;
            nmpcmc_gpu_shard_range(n, g, G, &b, &cnt);
            if (cnt > 0 &&
                (rc = cuda_check(ctx, cudaMemcpyPeerAsync(static_cast<nmpcmc_sim_record*>(root->d_all) + b, root->device,
                                                          s->d_rec, s->device, (size_t)cnt * sizeof(nmpcmc_sim_record),
                                                          root->stream), "gather records")) != NMPCMC_OK)
                return rc;
            long long h[8];
            cudaSetDevice(s->device);
            if ((rc = cuda_check(ctx, cudaMemcpy(h, s->d_tot, sizeof h, cudaMemcpyDeviceToHost), "D2H totals")) != NMPCMC_OK)
                return rc;
            add_totals(tot, h);
            cudaSetDevice(root->device);
        }
    }
    ctx->last_totals = tot;
    ctx->last_rec = static_cast<const nmpcmc_sim_record*>(root->d_all);
    ctx->last_n = n;
    cudaSetDevice(root->device);
    if (agg_out && (rc = k4_run(root, root->stream, static_cast<const nmpcmc_sim_record*>(root->d_all), n, agg_out, 0,
                                nullptr, nullptr, nullptr)) != NMPCMC_OK)
        return fail(ctx, rc, root->err);
    return cuda_check(ctx, cudaStreamSynchronize(root->stream), "K4");
}

int multi_run_async(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first, int64_t n,
                    nmpcmc_sim_record* rec_out, nmpcmc_work_counters* cnt_out) {
    const int G = (int)ctx->subs.size();
    for (int g = 0; g < G; ++g) {
        int64_t b = 0, cnt = 0;
        nmpcmc_gpu_shard_range(n, g, G, &b, &cnt);
        if (cnt == 0) continue;
        const int rc = nmpcmc_gpu_run_async(ctx->subs[g], sc, first + (uint64_t)b, cnt, rec_out + b,
                                            cnt_out ? cnt_out + b : nullptr);
        if (rc != NMPCMC_OK) return fail(ctx, rc, ctx->subs[g]->err);
    }
    return NMPCMC_OK;
}

}  // namespace nmpcmc_host

extern "C" {

void nmpcmc_gpu_shard_range(int64_t n, int g, int G, int64_t* begin, int64_t* count) {
    const int64_t c = nmpcmc_host::shard_chunk(n, G);
    int64_t b = (int64_t)g * c;
    if (b > n) b = n;
    int64_t e = b + c;
    if (e > n) e = n;
    if (begin) *begin = b;
    if (count) *count = e - b;
}

int nmpcmc_gpu_ctx_create_multi(const int* device_ids, int n_devices, nmpcmc_gpu_ctx** out) {
    using namespace nmpcmc_host;
    if (out == nullptr || device_ids == nullptr || n_devices < 1) return NMPCMC_INVALID_ARGUMENT;
    *out = nullptr;
    nmpcmc_gpu_ctx* ctx = nullptr;
    int rc = nmpcmc_gpu_ctx_create(device_ids[0], &ctx);
    if (rc != NMPCMC_OK) return rc;
    for (int g = 0; g < n_devices; ++g) {
        nmpcmc_gpu_ctx* s = nullptr;
        if ((rc = nmpcmc_gpu_ctx_create(device_ids[g], &s)) != NMPCMC_OK) {
            nmpcmc_gpu_ctx_destroy(ctx);
            return rc;
        }
        ctx->subs.push_back(s);
    }
    std::vector<int> ids(device_ids, device_ids + n_devices);
    std::vector<int> sorted = ids;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    if (distinct && n_devices > 1) {
        const NcclApi& N = nccl();
        if (!N.ok) {
            create_error() = "ctx_create_multi: NCCL unavailable: " + N.why;
            nmpcmc_gpu_ctx_destroy(ctx);
            return NMPCMC_CUDA_ERROR;
        }
        ctx->comms.resize(n_devices);
        const ncclResult_t r = N.CommInitAll(ctx->comms.data(), n_devices, ids.data());
        if (r != ncclSuccess) {
            create_error() = std::string("ctx_create_multi: ncclCommInitAll: ") + N.GetErrorString(r);
            ctx->comms.clear();
            nmpcmc_gpu_ctx_destroy(ctx);
            return NMPCMC_CUDA_ERROR;
        }
    }
    *out = ctx;
    return NMPCMC_OK;
}

int nmpcmc_gpu_ctx_num_devices(const nmpcmc_gpu_ctx* ctx) {
    if (ctx == nullptr) return 0;
    return ctx->subs.empty() ? 1 : (int)ctx->subs.size();
}

int nmpcmc_gpu_ctx_uses_nccl(const nmpcmc_gpu_ctx* ctx) {
    if (ctx == nullptr) return 0;
    return (!ctx->comms.empty() || ctx->comm != nullptr) ? 1 : 0;
}

int nmpcmc_gpu_aggregate_device(nmpcmc_gpu_ctx* ctx, const nmpcmc_sim_record* records_dev, int64_t n,
                                nmpcmc_aggregate* agg_out, int32_t bins, double* edges_out, int32_t* counts_out,
                                int32_t* nbins_out) {
    if (ctx == nullptr || (records_dev == nullptr && n > 0) || n < 0) return NMPCMC_INVALID_ARGUMENT;
    cudaSetDevice(ctx->device);
    return nmpcmc_host::k4_run(ctx, ctx->stream, records_dev, n, agg_out, bins, edges_out, counts_out, nbins_out);
}

int nmpcmc_gpu_last_records(nmpcmc_gpu_ctx* ctx, const nmpcmc_sim_record** records_dev, int64_t* n,
                            int* device) {
    if (ctx == nullptr || records_dev == nullptr || n == nullptr) return NMPCMC_INVALID_ARGUMENT;
    *records_dev = ctx->last_rec;
    *n = ctx->last_n;
    if (device) *device = ctx->subs.empty() ? ctx->device : ctx->subs[0]->device;
    return ctx->last_rec ? NMPCMC_OK : NMPCMC_INVALID_ARGUMENT;
}

int nmpcmc_gpu_histogram_last(nmpcmc_gpu_ctx* ctx, int32_t bins, double* edges_out, int32_t* counts_out,
                              int32_t* nbins_out) {
    if (ctx == nullptr || edges_out == nullptr || counts_out == nullptr || nbins_out == nullptr)
        return NMPCMC_INVALID_ARGUMENT;
    if (ctx->last_rec == nullptr) return nmpcmc_host::fail(ctx, NMPCMC_INVALID_ARGUMENT, "no run yet");
    nmpcmc_gpu_ctx* dev = ctx->subs.empty() ? ctx : ctx->subs[0];
    cudaSetDevice(dev->device);
    const int rc = nmpcmc_host::k4_run(dev, dev->stream, ctx->last_rec, ctx->last_n, nullptr, bins, edges_out,
                                       counts_out, nbins_out);
    return rc == NMPCMC_OK ? rc : nmpcmc_host::fail(ctx, rc, dev->err);
}

int nmpcmc_gpu_last_totals(const nmpcmc_gpu_ctx* ctx, nmpcmc_work_counters* out) {
    if (ctx == nullptr || out == nullptr) return NMPCMC_INVALID_ARGUMENT;
    *out = ctx->last_totals;
    return NMPCMC_OK;
}

int nmpcmc_gpu_nccl_unique_id(uint8_t id_out[128]) {
    using namespace nmpcmc_host;
    if (id_out == nullptr) return NMPCMC_INVALID_ARGUMENT;
    const NcclApi& N = nccl();
    if (!N.ok) return NMPCMC_CUDA_ERROR;
    ncclUniqueId id;
    if (N.GetUniqueId(&id) != ncclSuccess) return NMPCMC_CUDA_ERROR;
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id_out, &id, sizeof id);
    return NMPCMC_OK;
}

int nmpcmc_gpu_comm_init(nmpcmc_gpu_ctx* ctx, const uint8_t id[128], int rank, int nranks) {
    using namespace nmpcmc_host;
    if (ctx == nullptr || id == nullptr || nranks < 1 || rank < 0 || rank >= nranks || !ctx->subs.empty())
        return NMPCMC_INVALID_ARGUMENT;
    if (ctx->comm != nullptr) return fail(ctx, NMPCMC_INVALID_ARGUMENT, "communicator already initialised");
    ctx->rank = rank;
    ctx->nranks = nranks;
    if (nranks == 1) return NMPCMC_OK;  // nothing to exchange
    const NcclApi& N = nccl();
    if (!N.ok) return fail(ctx, NMPCMC_CUDA_ERROR, "NCCL unavailable: " + N.why);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    cudaSetDevice(ctx->device);
    return nccl_check(ctx, N.CommInitRank(&ctx->comm, nranks, uid, rank), "ncclCommInitRank");
}

int nmpcmc_gpu_run_sharded(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first_sim, int64_t n_sims,
                           nmpcmc_sim_record* records_out, nmpcmc_aggregate* agg_out) {
    using namespace nmpcmc_host;
    if (ctx == nullptr || sc == nullptr || n_sims < 1 || !ctx->subs.empty()) return NMPCMC_INVALID_ARGUMENT;
    const int R = ctx->nranks;
    const int64_t c = shard_chunk(n_sims, R);
    int64_t b = 0, cnt = 0;
    nmpcmc_gpu_shard_range(n_sims, ctx->rank, R, &b, &cnt);
    nmpcmc_sim_record* dr = nullptr;
    nmpcmc_work_counters* dc = nullptr;
    int rc = run_to_device(ctx, *sc, first_sim + (uint64_t)b, cnt, c, true, &dr, &dc);
    if (rc != NMPCMC_OK) return rc;
    if ((rc = ensure_tot(ctx)) != NMPCMC_OK) return rc;
    if ((rc = counters_sum(ctx, ctx->stream, dc, cnt, static_cast<long long*>(ctx->d_tot))) != NMPCMC_OK) return rc;
    const nmpcmc_sim_record* all = dr;
    if (ctx->comm != nullptr) {
        const size_t rec_b = (size_t)c * sizeof(nmpcmc_sim_record);
        if ((rc = ensure(ctx, &ctx->d_all, &ctx->all_cap, rec_b * R + 256)) != NMPCMC_OK) return rc;
        const NcclApi& N = nccl();
        if ((rc = nccl_check(ctx, N.GroupStart(), "ncclGroupStart")) != NMPCMC_OK) return rc;
        N.AllGather(dr, ctx->d_all, rec_b, ncclUint8, ctx->comm, ctx->stream);
        N.AllReduce(ctx->d_tot, ctx->d_tot, 8, ncclInt64, ncclSum, ctx->comm, ctx->stream);
        if ((rc = nccl_check(ctx, N.GroupEnd(), "ncclGroupEnd (all-gather records, all-reduce counters)")) != NMPCMC_OK)
            return rc;
        all = static_cast<const nmpcmc_sim_record*>(ctx->d_all);
    }
    long long h[8];
    if ((rc = cuda_check(ctx, cudaMemcpyAsync(h, ctx->d_tot, sizeof h, cudaMemcpyDeviceToHost, ctx->stream),
                         "D2H totals")) != NMPCMC_OK)
        return rc;
    if (records_out &&
        (rc = cuda_check(ctx, cudaMemcpyAsync(records_out, all, (size_t)n_sims * sizeof(nmpcmc_sim_record),
                                              cudaMemcpyDeviceToHost, ctx->stream), "D2H records")) != NMPCMC_OK)
        return rc;
    if ((rc = cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "kernel execution / NCCL")) != NMPCMC_OK) return rc;
    nmpcmc_work_counters tot{};
    add_totals(tot, h);
    ctx->last_totals = tot;
    ctx->last_rec = all;
    ctx->last_n = n_sims;
    if (agg_out) return k4_run(ctx, ctx->stream, all, n_sims, agg_out, 0, nullptr, nullptr, nullptr);
    return NMPCMC_OK;
}

}  // extern "C"

extern "C" int nmpcmc_gpu_allgather_records(nmpcmc_gpu_ctx* ctx, const nmpcmc_sim_record* local_dev, int64_t chunk,
                                            nmpcmc_sim_record* all_dev) {
    using namespace nmpcmc_host;
    if (ctx == nullptr || chunk < 0 || (chunk > 0 && (local_dev == nullptr || all_dev == nullptr)))
        return NMPCMC_INVALID_ARGUMENT;
    if (chunk == 0) return NMPCMC_OK;
    cudaSetDevice(ctx->device);
    const size_t bytes = (size_t)chunk * sizeof(nmpcmc_sim_record);
    if (ctx->comm == nullptr)  // one rank: a device copy
        return cuda_check(ctx, cudaMemcpyAsync(all_dev, local_dev, bytes, cudaMemcpyDeviceToDevice, ctx->stream),
                          "gather records");
    return nccl_check(ctx, nccl().AllGather(local_dev, all_dev, bytes, ncclUint8, ctx->comm, ctx->stream),
                      "ncclAllGather records");
}
