// nmpc_kernel.cuh -- K3: NMPC closed loop (placeholder until the kernel lands).
#pragma once
#include "device_common.cuh"
namespace nmpcmc_dev {
inline int launch_nmpc(const nmpcmc_scenario&, uint64_t, int64_t, int, nmpcmc_sim_record*,
                       nmpcmc_work_counters*, double*, int, int, cudaStream_t) {
    return NMPCMC_UNSUPPORTED;
}
}  // namespace nmpcmc_dev
