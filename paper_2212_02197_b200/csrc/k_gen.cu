// k_gen.cu -- K3w / K3g (any controller state dimension) and their OCP batch
// form; host launchers declared in launchers.h.
#include "launchers.h"
#include "nmpc_kernel.cuh"  // shared warp helpers and certified math used by the generic kernels
#include "nmpc_gen_kernel.cuh"

namespace nmpcmc_launch {

bool genw_fits(const nmpcmc_scenario& sc) { return nmpcmc_dev::gen::genw_fits(sc); }
int64_t genw_blocks(const nmpcmc_scenario& sc, int sm_count, int64_t n) {
    return nmpcmc_dev::gen::genw_blocks(sc, sm_count, n);
}
int64_t gen_ws_doubles(const nmpcmc_scenario& sc) { return nmpcmc_dev::gen::gen_ws_doubles(sc); }
int64_t gen_slots(const nmpcmc_scenario& sc, int sm_count, int64_t n) {
    return nmpcmc_dev::gen::gen_slots(sc, sm_count, n);
}

int launch_genw(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
                nmpcmc_work_counters* d_cnt, double* d_traj, int rows, double* ws, int64_t blocks,
                unsigned long long* counter, cudaStream_t stream, int fd) {
    return nmpcmc_dev::gen::launch_genw(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, ws, blocks, counter, stream,
                                        fd);
}

int launch_gen(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
               nmpcmc_work_counters* d_cnt, double* d_traj, int rows, double* ws, int64_t slots,
               unsigned long long* counter, cudaStream_t stream) {
    return nmpcmc_dev::gen::launch_gen(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, ws, slots, counter, stream);
}

int launch_ocp_batch(const nmpcmc_scenario& sc, int64_t batch, const double* x0, const double* t0, const double* xi0,
                     double* xi, double* lam, double* pil, double* piu, int32_t* conv, int32_t* status, double* ws,
                     int64_t blocks, unsigned long long* counter, cudaStream_t stream, int32_t* iters, int max_trace,
                     nmpcmc_sqp_iter_log* trace, int32_t* trace_len) {
    return nmpcmc_dev::gen::launch_ocp_batch(sc, batch, x0, t0, xi0, xi, lam, pil, piu, conv, status, ws, blocks,
                                             counter, stream, iters, max_trace, trace, trace_len);
}

int64_t qnlp_stride(int N, int nx) { return nmpcmc_dev::gen::qnlp_stride(N, nx); }
int64_t qnlp_ws_doubles(int N, int nx) { return nmpcmc_dev::gen::qnlp_ws_doubles(N, nx); }
int launch_qnlp_batch(int N, int nx, const nmpcmc_sqp_options& opt, int64_t batch, const double* prob,
                      const double* xi0, double* xi, double* lam, double* pil, double* piu, int32_t* conv,
                      int32_t* iters, int32_t* status, double* ws, int64_t blocks, unsigned long long* counter,
                      cudaStream_t stream) {
    return nmpcmc_dev::gen::launch_qnlp_batch(N, nx, opt, batch, prob, xi0, xi, lam, pil, piu, conv, iters, status,
                                              ws, blocks, counter, stream);
}

int64_t nmpc_state_doubles(const nmpcmc_scenario& sc) { return nmpcmc_dev::gen::nmpc_state_doubles(sc); }

int launch_nmpc_step(const nmpcmc_scenario& sc, int64_t batch, double* states, const double* t, const double* y,
                     const double* sp, double* u, nmpcmc_nmpc_diag* diag, double* ws, int64_t blocks,
                     unsigned long long* counter, cudaStream_t stream) {
    return nmpcmc_dev::gen::launch_nmpc_step(sc, batch, states, t, y, sp, u, diag, ws, blocks, counter, stream);
}

}  // namespace nmpcmc_launch
