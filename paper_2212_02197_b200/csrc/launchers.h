// launchers.h -- host-side entry points of the kernel translation units.
//
// Each kernel family compiles in its own .cu (k_nmpc.cu: K3; k_gen.cu: K3w /
// K3g; k_misc.cu: K2 PI, K5 QP, unit kernels, FP64 peak), so the library
// builds in parallel; the host code (nmpcmc_gpu.cu, nmpcmc_multi.cu) sees
// only these plain functions. Not installed.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "nmpcmc_gpu.h"

namespace nmpcmc_launch {

// ---- K3: one-state NMPC closed loop, one warp per sample (k_nmpc.cu)
/// Global workspace bytes and persistent block count K3 needs.
void nmpc_gws_need(const nmpcmc_scenario& sc, int sm_count, int64_t n, size_t* bytes, int64_t* blocks);
int launch_nmpc(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
                nmpcmc_work_counters* d_cnt, double* d_traj, int rows, int sm_count, double* gws, int64_t gws_blocks,
                unsigned long long* counter, cudaStream_t stream);
int launch_ocp1(const nmpcmc_scenario& sc, int64_t batch, const double* x0, const double* t0, const double* xi0,
                double* xi, double* lam, double* pil, double* piu, int32_t* conv, int32_t* status, int sm_count,
                double* gws, int64_t gws_blocks, unsigned long long* counter, cudaStream_t stream);

// ---- K3w / K3g: any controller state dimension (k_gen.cu)
bool genw_fits(const nmpcmc_scenario& sc);
int64_t genw_blocks(const nmpcmc_scenario& sc, int sm_count, int64_t n);
int64_t gen_ws_doubles(const nmpcmc_scenario& sc);
int64_t gen_slots(const nmpcmc_scenario& sc, int sm_count, int64_t n);
/// fd = 1: the controller model's jacobians by central differences
/// (NMPCMC_OPT_CTRL_JACOBIANS).
int launch_genw(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
                nmpcmc_work_counters* d_cnt, double* d_traj, int rows, double* ws, int64_t blocks,
                unsigned long long* counter, cudaStream_t stream, int fd);
int launch_gen(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
               nmpcmc_work_counters* d_cnt, double* d_traj, int rows, double* ws, int64_t slots,
               unsigned long long* counter, cudaStream_t stream);
int launch_ocp_batch(const nmpcmc_scenario& sc, int64_t batch, const double* x0, const double* t0, const double* xi0,
                     double* xi, double* lam, double* pil, double* piu, int32_t* conv, int32_t* status, double* ws,
                     int64_t blocks, unsigned long long* counter, cudaStream_t stream, int32_t* iters = nullptr,
                     int max_trace = 0, nmpcmc_sqp_iter_log* trace = nullptr, int32_t* trace_len = nullptr);

// ---- controller-level API: batched nmpc_step on K3w's path (k_gen.cu)
int64_t nmpc_state_doubles(const nmpcmc_scenario& sc);
int launch_nmpc_step(const nmpcmc_scenario& sc, int64_t batch, double* states, const double* t, const double* y,
                     const double* sp, double* u, nmpcmc_nmpc_diag* diag, double* ws, int64_t blocks,
                     unsigned long long* counter, cudaStream_t stream);

// ---- batched sqp_solve on stagewise quadratic NLPs (k_gen.cu)
int64_t qnlp_stride(int N, int nx);
int64_t qnlp_ws_doubles(int N, int nx);
int launch_qnlp_batch(int N, int nx, const nmpcmc_sqp_options& opt, int64_t batch, const double* prob,
                      const double* xi0, double* xi, double* lam, double* pil, double* piu, int32_t* conv,
                      int32_t* iters, int32_t* status, double* ws, int64_t blocks, unsigned long long* counter,
                      cudaStream_t stream);

// ---- K2 PI, unit kernels, FP64 peak, K5 batched QP (k_misc.cu)
int launch_pi(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
              nmpcmc_work_counters* d_cnt, double* d_traj, int rows, int sm_count, int pi_kernel,
              cudaStream_t stream);
void launch_pi_step(nmpcmc_pi_state* states, const double* y, const double* ybar, int64_t n,
                    nmpcmc_pi_step_result* results, int sm_count, cudaStream_t stream);
void launch_philox(const uint32_t* in, int64_t n, uint32_t* out, cudaStream_t stream);
void launch_normals(uint64_t seed, uint64_t stream_id, int64_t n, double* out, cudaStream_t stream);
void launch_libm(int fn, const double* x, int64_t n, double* out, cudaStream_t stream);
void launch_fp64_peak(int blocks, int threads, double* out, int iters, int use_fma, cudaStream_t stream);

int qp_max_nx();
int qp_max_nu();
int64_t qp_stage_doubles(int nx, int nu);
int64_t qp_solution_doubles(int N, int nx, int nu);
int64_t qp_slots(int sm_count, int64_t batch);
int64_t qp_ws_doubles(int N, int nx, int nu);
void launch_qp_batch(const nmpcmc_qp_dims& d, int64_t batch, const double* in, double* out, int32_t* status,
                     int32_t* iters, double* ws, int64_t slots, cudaStream_t stream);

}  // namespace nmpcmc_launch
