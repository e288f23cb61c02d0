// k_misc.cu -- K2 (PI closed loop), K5 (batched stagewise QP), the unit
// kernels behind the parity entry points (Philox blocks, normal streams, the
// device libm) and the FP64 peak probe; host launchers in launchers.h.
#include "launchers.h"
#include "pi_kernel.cuh"
#include "qp_batch_kernel.cuh"

namespace {

__global__ void philox_kernel(const uint32_t* in, int64_t n, uint32_t* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t* c = in + 6 * i;
    const uint4 r = nmpcmc_dev::philox4x32_10(make_uint4(c[0], c[1], c[2], c[3]), c[4], c[5]);
    out[4 * i + 0] = r.x;
    out[4 * i + 1] = r.y;
    out[4 * i + 2] = r.z;
    out[4 * i + 3] = r.w;
}

__global__ void normals_kernel(uint64_t seed, uint64_t stream, int64_t n, double* out) {
    // one thread replays the stream serially: exactly the host call pattern
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    nmpcmc_dev::NormalStream rng;
    rng.init(seed, stream);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.normal();
}

__global__ void libm_kernel(int fn, const double* x, int64_t n, double* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = x[i];
    double r;
    switch (fn) {
        case 0: r = xlibm_exp(v); break;
        case 1: r = xlibm_log(v); break;
        case 2: r = xlibm_sin(v); break;
        default: r = xlibm_cos(v); break;
    }
    out[i] = r;
}

// --------------------------------------------- FP64 peak (roofline denominator)
// MEASURED_PEAKS.json carries HBM and bf16 only; the closed loop runs on the
// FP64 CUDA cores, so its roofline denominator is measured here: independent
// DFMA chains, grid = 8 x SMs x 256 threads, 2 flops per DFMA.
__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, int use_fma) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
           a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    if (use_fma) {
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                a0 = __fma_rn(a0, b, c); a1 = __fma_rn(a1, b, c); a2 = __fma_rn(a2, b, c); a3 = __fma_rn(a3, b, c);
                a4 = __fma_rn(a4, b, c); a5 = __fma_rn(a5, b, c); a6 = __fma_rn(a6, b, c); a7 = __fma_rn(a7, b, c);
            }
        }
    } else {
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                a0 = __dadd_rn(a0, c); a1 = __dadd_rn(a1, c); a2 = __dadd_rn(a2, c); a3 = __dadd_rn(a3, c);
                a4 = __dadd_rn(a4, c); a5 = __dadd_rn(a5, c); a6 = __dadd_rn(a6, c); a7 = __dadd_rn(a7, c);
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

}  // namespace

namespace nmpcmc_launch {

int launch_pi(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
              nmpcmc_work_counters* d_cnt, double* d_traj, int rows, int sm_count, int pi_kernel,
              cudaStream_t stream) {
    // several lanes per sample for batches too small to fill the GPU with one
    // thread per sample (about 4 warps per SM), when one control step's
    // normals fit one window refill (the lanes keep the warp in lockstep,
    // pi_kernel.cuh); measured: config 0 (1,000) 11.0 -> 6.5 ms at 4 lanes,
    // config 1 (30,000) fastest at 1 lane (profiles/r02d_pi_variants.txt)
    constexpr int G = nmpcmc_dev::kPiLanes, block = nmpcmc_dev::kPiBlock;
    const bool three = sc.truth_variant == NMPCMC_THREE_STATE;
    const int per_step = (sc.has_noise_R != 0 ? 1 : 0) + sc.Ns * (three ? 3 : 1);
    // warp-specialised kernel (K2ws): one consumer warp of 32 samples per
    // block, P producer warps generating the normals ahead; more producers
    // when the batch leaves SMs idle
#ifndef NMPCMC_PI_WS
#define NMPCMC_PI_WS 1
#endif
    const bool sparse = three && sc.truth.sigmaA == 0.0 && sc.truth.sigmaB == 0.0;
    const int reads = nmpcmc_dev::pi_ws_reads(sc, sparse);
    if (NMPCMC_PI_WS != 0 && pi_kernel != NMPCMC_PI_KERNEL_LANES && reads <= nmpcmc_dev::kPiWsMaxPerStep &&
        nbar > 0) {
        const int64_t blocks = (n + 31) / 32;
        const int P = pi_kernel == NMPCMC_PI_KERNEL_WS3 || pi_kernel == NMPCMC_PI_KERNEL_WS7
                          ? pi_kernel
                          : (NMPCMC_PI_WS > 1 ? NMPCMC_PI_WS : (blocks >= 2 * (int64_t)sm_count ? 3 : 7));
        const size_t smem = (size_t)nmpcmc_dev::kPiWsSlots * reads * 32 * sizeof(double);
        const unsigned grid = (unsigned)blocks;
        // the whole grid is one wave only if the shared-memory carveout
        // admits the register-limited block count (the default carveout
        // capped it at 5 blocks per SM: 1.58 waves at config 1)
#define NMPCMC_PI_WS_LAUNCH(NX, PP, SP)                                                                    \
    do {                                                                                                    \
        cudaFuncSetAttribute(nmpcmc_dev::pi_ws_kernel<NX, PP, SP>, cudaFuncAttributePreferredSharedMemoryCarveout, \
                             cudaSharedmemCarveoutMaxShared);                                               \
        nmpcmc_dev::pi_ws_kernel<NX, PP, SP><<<grid, 32 * (1 + PP), smem, stream>>>(sc, first, n, nbar, d_rec, \
                                                                                    d_cnt, d_traj, rows);   \
    } while (0)
        if (P == 3) {
            if (!three)
                NMPCMC_PI_WS_LAUNCH(1, 3, false);
            else if (sparse)
                NMPCMC_PI_WS_LAUNCH(3, 3, true);
            else
                NMPCMC_PI_WS_LAUNCH(3, 3, false);
        } else {
            if (!three)
                NMPCMC_PI_WS_LAUNCH(1, 7, false);
            else if (sparse)
                NMPCMC_PI_WS_LAUNCH(3, 7, true);
            else
                NMPCMC_PI_WS_LAUNCH(3, 7, false);
        }
#undef NMPCMC_PI_WS_LAUNCH
        return NMPCMC_OK;
    }
#ifndef NMPCMC_PI_SMALL_WARPS
#define NMPCMC_PI_SMALL_WARPS 4
#endif
    const bool small = n < (int64_t)sm_count * NMPCMC_PI_SMALL_WARPS * 32;
    if (G > 1 && small && per_step < 2 * nmpcmc_dev::kPiPairs) {
        const unsigned grid = (unsigned)((n + block / G - 1) / (block / G));
        if (three)
            nmpcmc_dev::pi_kernel<3, G><<<grid, block, 0, stream>>>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows);
        else
            nmpcmc_dev::pi_kernel<1, G><<<grid, block, 0, stream>>>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows);
    } else {
        const unsigned grid = (unsigned)((n + block - 1) / block);
        if (three)
            nmpcmc_dev::pi_kernel<3, 1><<<grid, block, 0, stream>>>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows);
        else
            nmpcmc_dev::pi_kernel<1, 1><<<grid, block, 0, stream>>>(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows);
    }
    return NMPCMC_OK;
}

void launch_pi_step(nmpcmc_pi_state* states, const double* y, const double* ybar, int64_t n,
                    nmpcmc_pi_step_result* results, int sm_count, cudaStream_t stream) {
    int64_t grid = (n + 255) / 256;
    const int64_t cap = (int64_t)sm_count * 8;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    nmpcmc_dev::pi_step_kernel<<<(unsigned)grid, 256, 0, stream>>>(states, y, ybar, n, results);
}

void launch_philox(const uint32_t* in, int64_t n, uint32_t* out, cudaStream_t stream) {
    philox_kernel<<<(unsigned)((n + 127) / 128), 128, 0, stream>>>(in, n, out);
}

void launch_normals(uint64_t seed, uint64_t stream_id, int64_t n, double* out, cudaStream_t stream) {
    normals_kernel<<<1, 32, 0, stream>>>(seed, stream_id, n, out);
}

void launch_libm(int fn, const double* x, int64_t n, double* out, cudaStream_t stream) {
    libm_kernel<<<(unsigned)((n + 127) / 128), 128, 0, stream>>>(fn, x, n, out);
}

void launch_fp64_peak(int blocks, int threads, double* out, int iters, int use_fma, cudaStream_t stream) {
    fp64_peak_kernel<<<blocks, threads, 0, stream>>>(out, iters, use_fma);
}

int qp_max_nx() { return nmpcmc_dev::qpb::QX; }
int qp_max_nu() { return nmpcmc_dev::qpb::QU; }
int64_t qp_stage_doubles(int nx, int nu) { return nmpcmc_dev::qpb::stage_doubles(nx, nu); }
int64_t qp_solution_doubles(int N, int nx, int nu) { return nmpcmc_dev::qpb::solution_doubles(N, nx, nu); }
int64_t qp_slots(int sm_count, int64_t batch) { return nmpcmc_dev::qpb::qp_slots(sm_count, batch); }
int64_t qp_ws_doubles(int N, int nx, int nu) { return nmpcmc_dev::qpb::Lay(N, nx, nu).total; }

void launch_qp_batch(const nmpcmc_qp_dims& d, int64_t batch, const double* in, double* out, int32_t* status,
                     int32_t* iters, double* ws, int64_t slots, cudaStream_t stream) {
    const nmpcmc_dev::qpb::Dims kd{d.N, d.n_x, d.n_u, d.max_iter, d.mode, d.tol};
    const unsigned grid = (unsigned)((slots + nmpcmc_dev::qpb::kBlock - 1) / nmpcmc_dev::qpb::kBlock);
    nmpcmc_dev::qpb::qp_batch_kernel<<<grid, nmpcmc_dev::qpb::kBlock, 0, stream>>>(kd, batch, in, out, status, iters,
                                                                                  ws, slots);
}

}  // namespace nmpcmc_launch
