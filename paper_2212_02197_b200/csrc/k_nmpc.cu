// k_nmpc.cu -- K3 (one-state NMPC, one warp per sample) and its OCP batch
// form; host launchers declared in launchers.h.
#include "launchers.h"
#include "nmpc_kernel.cuh"

namespace nmpcmc_launch {

void nmpc_gws_need(const nmpcmc_scenario& sc, int sm_count, int64_t n, size_t* bytes, int64_t* blocks) {
    nmpcmc_dev::nmpc_gws_need(sc, sm_count, n, bytes, blocks);
}

int launch_nmpc(const nmpcmc_scenario& sc, uint64_t first, int64_t n, int nbar, nmpcmc_sim_record* d_rec,
                nmpcmc_work_counters* d_cnt, double* d_traj, int rows, int sm_count, double* gws, int64_t gws_blocks,
                unsigned long long* counter, cudaStream_t stream) {
    return nmpcmc_dev::launch_nmpc(sc, first, n, nbar, d_rec, d_cnt, d_traj, rows, sm_count, gws, gws_blocks, counter,
                                   stream);
}

int launch_ocp1(const nmpcmc_scenario& sc, int64_t batch, const double* x0, const double* t0, const double* xi0,
                double* xi, double* lam, double* pil, double* piu, int32_t* conv, int32_t* status, int sm_count,
                double* gws, int64_t gws_blocks, unsigned long long* counter, cudaStream_t stream) {
    return nmpcmc_dev::launch_ocp1(sc, batch, x0, t0, xi0, xi, lam, pil, piu, conv, status, sm_count, gws, gws_blocks,
                                   counter, stream);
}

}  // namespace nmpcmc_launch
