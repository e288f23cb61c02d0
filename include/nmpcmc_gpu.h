/* nmpcmc_gpu.h -- C ABI of the B200 batched closed-loop Monte Carlo engine.
 *
 * Drop-in boundary for the reference's Monte Carlo hot path
 * (/root/reference/proj/core/include/nmpcmc/montecarlo.hpp). The reference has
 * no FFI layer; its boundary is the C++ API
 *     McResult    run_monte_carlo(const Scenario&, int n_sims, int workers)   montecarlo.hpp:121
 *     SimResult   run_closed_loop(const Scenario&, uint64_t sim_index)        montecarlo.hpp:92
 *     McAggregate aggregate_stats(const std::vector<SimResult>&)              montecarlo.hpp:108
 *     Histogram   phi_histogram(const std::vector<double>&, int bins)         montecarlo.hpp:141
 *     int         validate_scenario(const Scenario&)                          montecarlo.hpp:59
 * Its Scenario holds type-erased std::function models (model.hpp:28-46) from
 * which the plant cannot be recovered, so this ABI carries the CSTR parameters
 * and variants explicitly in a POD. The C++ facade
 * include/nmpcmc_gpu.hpp keeps the reference's names and result types on top.
 *
 * Plain pointers and sizes only; no torch or CUDA types. All functions return
 * an nmpcmc_status; configuration errors map to the reference's exception
 * classes (errors.hpp:9-32), per-sample numerical failures never fail a call
 * (they are recorded in nmpcmc_sim_record.failed, montecarlo.cpp:147-155,228-236).
 */
#ifndef NMPCMC_GPU_H
#define NMPCMC_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NMPCMC_GPU_ABI_VERSION 1
#define NMPCMC_MAX_SETPOINTS 32

/* Status codes mirror the reference exception taxonomy (errors.hpp:9-32). */
typedef enum nmpcmc_status {
    NMPCMC_OK = 0,
    NMPCMC_DIMENSION_MISMATCH = 1, /* DimensionMismatch errors.hpp:9 */
    NMPCMC_NOT_POSITIVE_DEFINITE = 2, /* NotPositiveDefinite errors.hpp:15 */
    NMPCMC_NON_FINITE_STATE = 3,  /* NonFiniteState errors.hpp:20 */
    NMPCMC_DOMAIN_ERROR = 4,      /* DomainError errors.hpp:25 */
    NMPCMC_LENGTH_MISMATCH = 5,   /* LengthMismatch errors.hpp:30 */
    NMPCMC_UNSUPPORTED = 6,       /* valid for the reference, not built on device yet */
    NMPCMC_INVALID_ARGUMENT = 7,  /* null pointer / bad size at the C boundary */
    NMPCMC_CUDA_ERROR = 100,
    NMPCMC_NO_DEVICE = 101
} nmpcmc_status;

/* ControllerType (montecarlo.hpp:22): nmpc = 0, pi = 1. */
enum { NMPCMC_CTRL_NMPC = 0, NMPCMC_CTRL_PI = 1 };
/* CstrVariant (cstr.hpp:19): three_state = 0, one_state = 1. */
enum { NMPCMC_THREE_STATE = 0, NMPCMC_ONE_STATE = 1 };

/* CstrParams (cstr.hpp:21-34). Flows in mL/min. */
typedef struct nmpcmc_cstr_params {
    double V, k0, EaR, beta, cA_in, cB_in, cT_in;
    double sigmaA, sigmaB, sigmaT;
    double u_min, u_max;
} nmpcmc_cstr_params;

/* SqpOptions (sqp.hpp:50-58). */
typedef struct nmpcmc_sqp_options {
    double eps;
    double c1;
    double backtrack_factor;
    double qp_tol;
    int32_t max_iter;
    int32_t max_backtracks;
    int32_t qp_max_iter;
    int32_t _pad;
} nmpcmc_sqp_options;

/* PiState gains (controllers.hpp:16-25); Ts, u_min, u_max are taken from the
 * scenario exactly like run_closed_loop does (montecarlo.cpp:97-100). */
typedef struct nmpcmc_pi_gains {
    double kP, kI, kaw, u_bar, I_hat;
} nmpcmc_pi_gains;

/* Scenario (montecarlo.hpp:27-55) for the CSTR case study. */
typedef struct nmpcmc_scenario {
    int32_t controller;      /* NMPCMC_CTRL_* */
    int32_t truth_variant;   /* NMPCMC_THREE_STATE | NMPCMC_ONE_STATE */
    int32_t ctrl_variant;    /* NMPC controller model: THREE_STATE (K3g) or ONE_STATE */
    int32_t has_noise_R;     /* NoiseSpec::R has rows (model.cpp:41) */
    nmpcmc_cstr_params truth;
    nmpcmc_cstr_params ctrl;
    double noise_R;          /* NoiseSpec::R, 1x1 (n_y = 1) */
    double R_filter;         /* Scenario::R_filter, 1x1 */
    double Qz;               /* Scenario::Qz, 1x1 (n_z = 1) */
    double horizon_Ts;       /* Horizon::Ts */
    int32_t N;               /* Horizon::N */
    int32_t Nc;              /* Horizon::Nc */
    int32_t np;              /* Scenario::np */
    int32_t Ns;              /* Scenario::Ns */
    nmpcmc_sqp_options sqp;
    nmpcmc_pi_gains pi;
    double u_min, u_max;     /* Scenario::u_min/u_max (n_u = 1) */
    double t0, tf, Ts;
    int32_t n_setpoints;     /* SetpointProfile (montecarlo.hpp:15-20), n_z = 1 */
    int32_t record_stride;   /* Scenario::record_stride */
    double sp_times[NMPCMC_MAX_SETPOINTS];
    double sp_values[NMPCMC_MAX_SETPOINTS];
    double x0[3];            /* truth initial state (n_x of truth_variant) */
    double x0_hat[3];        /* filter prior mean (n_x of ctrl_variant) */
    double P0[9];            /* filter prior covariance, column-major */
    uint64_t base_seed;
    /* Per-sample parameter uncertainty (BASELINE configs 1, 3, 4). Not a
     * reference feature: when perturb != 0 each sample's TRUTH parameters
     * become cA_in*(1+s0*z0), cB_in*(1+s1*z1), EaR*(1+s2*z2) with z the first
     * three normals of stream (base_seed, sim_index | 2^63). The oracle
     * applies the same rule through the reference's own CounterRng. */
    int32_t perturb;
    int32_t record_trajectories; /* Scenario::record_trajectories */
    double perturb_rel_std[3];
} nmpcmc_scenario;

/* SimResult (montecarlo.hpp:72-79) without the trajectory. */
typedef struct nmpcmc_sim_record {
    double phi;              /* NaN when failed */
    int32_t failed;
    int32_t ocp_solves;
    int32_t ocp_failures;
    int32_t status;          /* nmpcmc_status that ended the run (0 if none) */
} nmpcmc_sim_record;

/* Per-sample work counters (device-measured) for the FP64 roofline
 * (SURVEY.md §8d). Shooting counts are stage intervals, not sweeps. */
typedef struct nmpcmc_work_counters {
    int64_t control_steps;
    int64_t shoot_full;      /* stage intervals shot with sensitivities */
    int64_t shoot_fonly;     /* stage intervals shot state-only */
    int64_t ipm_stage_iters; /* sum over IPM iterations of N */
    int64_t sqp_stage_iters; /* sum over SQP iterations of N */
    int64_t qp_solves;
    int64_t sqp_iterations;
    int64_t ls_evals;
} nmpcmc_work_counters;

/* McAggregate (montecarlo.hpp:95-106). */
typedef struct nmpcmc_aggregate {
    int32_t n_sims;
    int32_t n_failed;
    double mean, variance, min, max;
    double deciles[11];
    int64_t ocp_solves;
    int64_t ocp_failures;
    double ocp_success_pct;
} nmpcmc_aggregate;

typedef struct nmpcmc_gpu_ctx nmpcmc_gpu_ctx;

/* ABI self-description so bindings can check their struct layout. */
int nmpcmc_gpu_abi_version(void);
int64_t nmpcmc_gpu_struct_size(int which); /* 0 scenario, 1 record, 2 counters, 3 aggregate */

/* validate_scenario (montecarlo.cpp:34-63) plus the device support checks;
 * writes N_bar. Host only. */
int nmpcmc_gpu_validate(const nmpcmc_scenario* sc, int32_t* nbar_out);

/* Context = one device + one stream + scratch. Replaces the std::thread pool
 * of run_monte_carlo (montecarlo.cpp:218-245). */
int nmpcmc_gpu_ctx_create(int device, nmpcmc_gpu_ctx** out);
/* Number of visible CUDA devices (0 and NMPCMC_NO_DEVICE without a driver). */
int nmpcmc_gpu_device_count(int* count_out);
void nmpcmc_gpu_ctx_destroy(nmpcmc_gpu_ctx* ctx);
const char* nmpcmc_gpu_last_error(const nmpcmc_gpu_ctx* ctx);
/* Context options. NMPCMC_OPT_NMPC_KERNEL selects the NMPC kernel for a
 * one-state controller model with N <= 255:
 * WARP (default) = one warp per sample, sweep arrays in shared memory (K3);
 * GENERIC = one thread per sample, any controller state dimension (K3g);
 * THREAD = alias of GENERIC (the one-thread-per-sample K3b was retired);
 * GENERIC_WARP = one warp per sample, any controller state dimension (K3w).
 * A three-state controller model or N > 255 always runs a generic kernel:
 * K3w, or K3g when GENERIC / THREAD is selected. Results are bitwise
 * identical; only speed differs. NMPCMC_OPT_TPS_WARPS_PER_SM is accepted and
 * ignored (it tuned K3b). */
enum { NMPCMC_OPT_NMPC_KERNEL = 1, NMPCMC_OPT_TPS_WARPS_PER_SM = 2, NMPCMC_OPT_LANES = 3,
       NMPCMC_OPT_CTRL_JACOBIANS = 4, NMPCMC_OPT_PI_KERNEL = 5 };
/* NMPCMC_OPT_PI_KERNEL selects the PI closed-loop kernel. AUTO (default) =
 * the warp-specialised kernel (one consumer warp of 32 samples, producer warps
 * generating the normals ahead; 7 producers when the batch leaves SMs idle,
 * else 3) whenever a control step reads at most 40 normals, else the
 * lanes kernel; LANES = one thread (or 4 lanes, small batches) per sample
 * with the normals in a per-sample window; WS3 / WS7 = the warp-specialised
 * kernel with 3 / 7 producer warps. Results are bitwise identical. */
enum { NMPCMC_PI_KERNEL_AUTO = 0, NMPCMC_PI_KERNEL_LANES = 1, NMPCMC_PI_KERNEL_WS3 = 3, NMPCMC_PI_KERNEL_WS7 = 7 };
/* NMPCMC_OPT_CTRL_JACOBIANS: how the controller model's jacobians are formed.
 * ANALYTIC (default) = the closed forms make_cstr_model installs
 * (cstr.cpp:86-127). FD = as a Model WITHOUT analytic jacobians:
 * drift_jacobian_x / _u, measurement_jacobian_x and output_jacobian_x by the
 * reference's central differences, step max(1e-6, 1e-6 |v|)
 * (model.cpp:54-124) -- bitwise the reference run on such a Model. FD runs on
 * the generic one-warp kernel (K3w) for either controller model. */
enum { NMPCMC_JACOBIANS_ANALYTIC = 0, NMPCMC_JACOBIANS_FD = 1 };
/* NMPCMC_OPT_LANES = 2 pipelines back-to-back batches: NMPC launches alternate
 * between two internal streams with their own workspace (PI launches use a
 * third), each forked from the context stream, so one batch's drain (its last
 * wave of long samples) overlaps the next batch. Work on a lane is ordered
 * after everything enqueued on the context stream before the call; later work
 * on the context stream is ordered after the lanes only through
 * nmpcmc_gpu_join / nmpcmc_gpu_wait. 1 (default) = everything on the context
 * stream. */
enum { NMPCMC_NMPC_KERNEL_WARP = 1, NMPCMC_NMPC_KERNEL_THREAD = 2, NMPCMC_NMPC_KERNEL_GENERIC = 3,
       NMPCMC_NMPC_KERNEL_GENERIC_WARP = 4 };
int nmpcmc_gpu_set_option(nmpcmc_gpu_ctx* ctx, int32_t option, int64_t value);
/* CUDA stream the context launches on (as void*; 0 = legacy default). The
 * new stream is ordered after all work already enqueued on the old stream and
 * its lanes (join + event), because launches share the context's workspace. */
int nmpcmc_gpu_set_stream(nmpcmc_gpu_ctx* ctx, void* stream);

/* run_monte_carlo over the global sample range [first_sim, first_sim+n_sims)
 * (montecarlo.cpp:213-251; run_closed_loop per sample, montecarlo.cpp:80-157).
 * HOST buffers: records_out[n_sims] in index order; counters_out and agg_out
 * may be NULL. Synchronous. */
int nmpcmc_gpu_run(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first_sim,
                   int64_t n_sims, nmpcmc_sim_record* records_out,
                   nmpcmc_work_counters* counters_out, nmpcmc_aggregate* agg_out);

/* Asynchronous form: enqueue the batch and the copy of its records (and
 * counters, may be NULL) into HOST buffers, which must stay valid until
 * nmpcmc_gpu_wait. With pinned host memory and NMPCMC_OPT_LANES = 2,
 * consecutive calls overlap. */
int nmpcmc_gpu_run_async(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first_sim,
                         int64_t n_sims, nmpcmc_sim_record* records_out,
                         nmpcmc_work_counters* counters_out);
/* Order the context stream after all work enqueued on the lanes (no host
 * wait); no-op without lanes. */
int nmpcmc_gpu_join(nmpcmc_gpu_ctx* ctx);
/* join + wait on the host for the context stream; reports kernel errors. */
int nmpcmc_gpu_wait(nmpcmc_gpu_ctx* ctx);

/* Same, DEVICE-resident outputs (records_dev[n_sims], counters_dev may be
 * NULL), enqueued on the context stream (or a lane, NMPCMC_OPT_LANES);
 * returns after the launch. */
int nmpcmc_gpu_run_device(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first_sim,
                          int64_t n_sims, nmpcmc_sim_record* records_dev,
                          nmpcmc_work_counters* counters_dev);

/* Trajectory recording (montecarlo.cpp:126-146, Trajectory montecarlo.hpp:64-67).
 * traj_out: HOST, n_sims * rows * 5 doubles, rows = nmpcmc_gpu_traj_rows(sc);
 * per row (t, z, z_bar, u, y); unused rows of failed runs are NaN. */
int32_t nmpcmc_gpu_traj_rows(const nmpcmc_scenario* sc);
int nmpcmc_gpu_run_traj(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first_sim,
                        int64_t n_sims, nmpcmc_sim_record* records_out, double* traj_out);

/* aggregate_stats (montecarlo.cpp:172-211), index order, host. */
int nmpcmc_gpu_aggregate(const nmpcmc_sim_record* records, int64_t n, nmpcmc_aggregate* out);

/* phi_histogram (montecarlo.cpp:268-304), host. edges_out[201], counts_out[200]. */
int nmpcmc_gpu_histogram(const double* phi, int64_t n, int32_t bins, double* edges_out,
                         int32_t* counts_out, int32_t* nbins_out);

/* ---- Statistics on the device (K4; north_star "final block reduction") --
 * aggregate_stats (montecarlo.cpp:172-211) and, when counts_out != NULL,
 * phi_histogram (montecarlo.cpp:268-304; bins <= 0: Freedman-Diaconis,
 * edges_out[201], counts_out[200]) of DEVICE-resident records, bitwise the
 * reference's host results: exact integer totals, the serial index-order sums
 * of the mean and the two-pass variance, a device sort for min / max /
 * deciles. agg_out may be NULL. nmpcmc_gpu_run computes its agg_out this way. */
int nmpcmc_gpu_aggregate_device(nmpcmc_gpu_ctx* ctx, const nmpcmc_sim_record* records_dev, int64_t n,
                                nmpcmc_aggregate* agg_out, int32_t bins, double* edges_out,
                                int32_t* counts_out, int32_t* nbins_out);
/* The records of the last nmpcmc_gpu_run / nmpcmc_gpu_run_sharded stay on the
 * device (all of them, gathered, on device_ids[0] for a multi-device context)
 * until the next call: their device pointer, count and device id. */
int nmpcmc_gpu_last_records(nmpcmc_gpu_ctx* ctx, const nmpcmc_sim_record** records_dev, int64_t* n,
                            int* device);
/* phi_histogram of the last run's records, on the device (see above). */
int nmpcmc_gpu_histogram_last(nmpcmc_gpu_ctx* ctx, int32_t bins, double* edges_out, int32_t* counts_out,
                              int32_t* nbins_out);
/* Work counters of the last run summed over all samples, devices and ranks
 * (an NCCL int64 all-reduce when several GPUs took part). */
int nmpcmc_gpu_last_totals(const nmpcmc_gpu_ctx* ctx, nmpcmc_work_counters* out);

/* ---- Multi-GPU --------------------------------
 * run_monte_carlo's worker pool (montecarlo.cpp:213-251) across the GPUs of
 * one process: a context over n_devices devices, one sub-context (stream,
 * workspace) per id. On it nmpcmc_gpu_run shards [first, first + n) into
 * contiguous blocks (nmpcmc_gpu_shard_range), one host thread per device
 * launches its block and copies its records into records_out at the block's
 * offset; the records are then all-gathered over NCCL onto device_ids[0]
 * (ncclCommInitAll; the only exchange) where K4 computes agg_out, and the
 * work counters are all-reduced. Records are bitwise independent of the
 * device count (every stream is keyed by the global sample index).
 * nmpcmc_gpu_run_async / _join / _wait / _run_traj / _set_option work per
 * device the same way; _run_device and _set_stream are single-device only.
 * Repeated ids are allowed (several blocks share a GPU; peer copies replace
 * NCCL); with distinct ids NCCL is required (loaded with dlopen). On failure
 * nmpcmc_gpu_last_error(NULL) says why. */
int nmpcmc_gpu_ctx_create_multi(const int* device_ids, int n_devices, nmpcmc_gpu_ctx** out);
int nmpcmc_gpu_ctx_num_devices(const nmpcmc_gpu_ctx* ctx);
/* 1 when records are exchanged over NCCL (distinct devices or ranks). */
int nmpcmc_gpu_ctx_uses_nccl(const nmpcmc_gpu_ctx* ctx);
/* Block g of G of [0, n): [g*ceil(n/G), min(n, (g+1)*ceil(n/G))). Host only. */
void nmpcmc_gpu_shard_range(int64_t n, int g, int G, int64_t* begin, int64_t* count);

/* One process per GPU (torchrun-style launch): rank 0 creates an NCCL id and
 * ships it to the others out of band; every rank joins with its own
 * single-device context. nmpcmc_gpu_run_sharded then runs this rank's block
 * of [first, first + n), all-gathers the records (NCCL) so that
 * records_out[n] (HOST, may be NULL) holds all of them in index order on every
 * rank, all-reduces the work counters (nmpcmc_gpu_last_totals) and computes
 * agg_out (may be NULL) with K4. Without nmpcmc_gpu_comm_init it is
 * nmpcmc_gpu_run on one GPU. */
int nmpcmc_gpu_nccl_unique_id(uint8_t id_out[128]);
int nmpcmc_gpu_comm_init(nmpcmc_gpu_ctx* ctx, const uint8_t id[128], int rank, int nranks);
int nmpcmc_gpu_run_sharded(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, uint64_t first_sim, int64_t n_sims,
                           nmpcmc_sim_record* records_out, nmpcmc_aggregate* agg_out);
/* The exchange alone, for callers that run their blocks themselves (e.g.
 * with nmpcmc_gpu_run_device): all-gather `chunk` DEVICE records from every
 * rank into all_dev[nranks * chunk] (rank r's at r * chunk), enqueued on the
 * context stream (NCCL; a device copy with one rank). */
int nmpcmc_gpu_allgather_records(nmpcmc_gpu_ctx* ctx, const nmpcmc_sim_record* local_dev, int64_t chunk,
                                 nmpcmc_sim_record* all_dev);

/* Unit-level device entry points (parity tests of rng.cpp and the libm). */
/* CounterRng::philox_block (rng.cpp:31-43): in[6*n] = counter[4], key[2]; out[4*n]. */
int nmpcmc_gpu_philox_blocks(nmpcmc_gpu_ctx* ctx, const uint32_t* in, int64_t n, uint32_t* out);
/* CounterRng(seed, stream).normal() x n (rng.cpp:78-91). */
int nmpcmc_gpu_normals(nmpcmc_gpu_ctx* ctx, uint64_t seed, uint64_t stream, int64_t n,
                       double* out);
/* fn: 0 exp, 1 log, 2 sin, 3 cos of x[n] with the device libm. */
int nmpcmc_gpu_libm(nmpcmc_gpu_ctx* ctx, int32_t fn, const double* x, int64_t n, double* out);

/* Measured FP64 throughput of the device (TFLOP/s): the roofline denominator
 * for the FP64 closed-loop kernels (use_fma=1: DFMA, 2 flops each; 0: DADD). */
int nmpcmc_gpu_fp64_peak(nmpcmc_gpu_ctx* ctx, int use_fma, double* tflops_out);

/* ---- Batched OCP service ---------------------
 * sqp_solve (sqp.hpp:148-151, sqp.cpp:182-411) on the regulator OcpProblem
 * (sqp.hpp:27-50) of the scenario's controller model (ctrl, ctrl_variant),
 * horizon {N, horizon_Ts, Nc}, Qz, u_min/u_max, setpoint profile and
 * SqpOptions, for `batch` instances: instance b starts at state x0[b*nx ..]
 * (nx = 1 or 3 by ctrl_variant) at time t0[b] (setpoints at t0 + k Ts,
 * k = 1..N). xi0 == NULL: cold start exactly as nmpc_step
 * (controllers.cpp:166-185); else xi0[b*L ..] with zero duals. HOST buffers;
 * L = N (1 + nx). Outputs per instance: xi[L], lambda[N nx], pi_l[N], pi_u[N]
 * (SqpReport, sqp.hpp:79-90), converged, status (0, or NMPCMC_DOMAIN_ERROR if
 * a DomainError escaped the solve). Bitwise the reference's results. */
int nmpcmc_gpu_solve_ocp_batch(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, int64_t batch,
                               const double* x0, const double* t0, const double* xi0, double* xi,
                               double* lambda, double* pi_l, double* pi_u, int32_t* converged,
                               int32_t* status);

/* SqpIterationLog (sqp.hpp:64-77): one record per SQP iteration, pushed
 * where sqp_solve pushes it (sqp.cpp:274, :327, :350, :406). qp_status is
 * NMPCMC_QP_OPTIMAL / _MAXITER / _FAILED. */
typedef struct nmpcmc_sqp_iter_log {
    double alpha;
    double merit_before;
    double merit_after;
    double directional_derivative;
    double grad_l_inf;   /* at iteration start */
    double g_inf;        /* at iteration start */
    double step_inf;     /* |alpha * delta_xi|_inf */
    int32_t ls_evals;
    int32_t qp_iterations;
    int32_t qp_status;
    int32_t armijo_exhausted;
    int32_t bfgs_reset;
    int32_t _pad;
} nmpcmc_sqp_iter_log;
/* The OCP service with SqpReport's per-iteration trace (SqpReport::trace,
 * sqp.hpp:90) and iteration count: trace[b * max_trace ..] holds up to
 * max_trace records of instance b, trace_len[b] the number sqp_solve pushed
 * (may exceed max_trace; the excess is dropped), iterations[b] =
 * SqpReport::iterations. HOST buffers; runs on K3w's code path for either
 * controller model. Bitwise the reference's trace. */
int nmpcmc_gpu_solve_ocp_batch_traced(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, int64_t batch,
                                      const double* x0, const double* t0, const double* xi0, double* xi,
                                      double* lambda, double* pi_l, double* pi_u, int32_t* converged,
                                      int32_t* status, int32_t* iterations, int32_t max_trace,
                                      nmpcmc_sqp_iter_log* trace, int32_t* trace_len);

/* ---- Batched standalone stagewise QP ----------
 * solve_qp (qp.hpp:47-56, qp.cpp:173-423; mode 0) or riccati_factor_solve
 * (qp.hpp:42-45, qp.cpp:157-171; mode 1) for `batch` independent QPs of the
 * same dimensions, bitwise the reference's results. n_x <= 8, n_u <= 4.
 * stages: HOST, batch * (N+1) * nmpcmc_qp_stage_doubles(n_x, n_u) doubles;
 * per stage Q[nx*nx] M[nx*nu] R[nu*nu] q[nx] r[nu] Jx[nx*nx] Ju[nx*nu] b[nx]
 * lb[nu] ub[nu] (QpStageData, qp.hpp:24-30; matrices column-major; members a
 * stage does not use are ignored: stage 0 has no Q M q Jx, stage N only Q q).
 * solutions: HOST, batch * nmpcmc_qp_solution_doubles(N, n_x, n_u):
 * delta_xi[N(nu+nx)] mu[N nx] nu_l[N nu] nu_u[N nu] (QpSolution, qp.hpp:34-41).
 * status[batch]: NMPCMC_QP_*; iterations[batch]: IPM iterations. Per-QP
 * DomainError (lb > ub) and NotPositiveDefinite (mode 1) are statuses, not
 * call failures; the call fails only on bad dimensions (DIMENSION_MISMATCH). */
typedef struct nmpcmc_qp_dims {
    int32_t N;        /* stages 0..N: N inputs, terminal state N */
    int32_t n_x;
    int32_t n_u;
    int32_t max_iter; /* solve_qp max_iter (default 50) */
    double tol;       /* solve_qp tol (default 1e-10) */
    int32_t mode;     /* 0 solve_qp, 1 riccati_factor_solve */
    int32_t _pad;
} nmpcmc_qp_dims;
enum { NMPCMC_QP_OPTIMAL = 0, NMPCMC_QP_MAXITER = 1, NMPCMC_QP_FAILED = 2, NMPCMC_QP_DOMAIN_ERROR = 3,
       NMPCMC_QP_NOT_POSITIVE_DEFINITE = 4 };
int64_t nmpcmc_qp_stage_doubles(int32_t n_x, int32_t n_u);
int64_t nmpcmc_qp_solution_doubles(int32_t N, int32_t n_x, int32_t n_u);
int nmpcmc_gpu_solve_qp_batch(nmpcmc_gpu_ctx* ctx, const nmpcmc_qp_dims* dims, int64_t batch,
                              const double* stages, double* solutions, int32_t* status,
                              int32_t* iterations);

/* ---- Controller-level API (controllers.hpp:16-93) ----------------------
 * PiState (controllers.hpp:16-25) and PiStepResult (:29-37); next_I_hat is
 * result.next.I_hat (the rest of result.next equals the input state). */
typedef struct nmpcmc_pi_state {
    double kP, kI, kaw, Ts, u_bar, u_min, u_max, I_hat;
} nmpcmc_pi_state;
typedef struct nmpcmc_pi_step_result {
    double e, P, I, u_hat, u, I_aw, next_I_hat;
} nmpcmc_pi_step_result;
/* pi_step (controllers.hpp:49, controllers.cpp:12-23) for n independent
 * controllers: states[i] advances to result.next in place; results may be
 * NULL. _batch takes HOST buffers (synchronous); _device takes DEVICE
 * buffers and is enqueued on the context stream. */
int nmpcmc_gpu_pi_step_batch(nmpcmc_gpu_ctx* ctx, nmpcmc_pi_state* states, const double* y, const double* y_bar,
                             int64_t n, nmpcmc_pi_step_result* results);
int nmpcmc_gpu_pi_step_device(nmpcmc_gpu_ctx* ctx, nmpcmc_pi_state* states_dev, const double* y_dev,
                              const double* y_bar_dev, int64_t n, nmpcmc_pi_step_result* results_dev);

/* A batch of B device-resident NmpcStates (controllers.hpp:54-65) for the
 * scenario's controller model (ctrl, ctrl_variant; n_x = 1 or 3), horizon,
 * Qz, R_filter, np, u_min / u_max and SqpOptions -- make_nmpc_state
 * (controllers.cpp:25-48) per instance with prior x0_hat[b*n_x ..] and
 * P0[b*n_x*n_x ..] (column-major; NULL = the scenario's x0_hat / P0 for
 * every instance). HOST inputs; the states stay on the context's device. */
typedef struct nmpcmc_nmpc_batch nmpcmc_nmpc_batch;
int nmpcmc_gpu_nmpc_batch_create(nmpcmc_gpu_ctx* ctx, const nmpcmc_scenario* sc, int64_t batch,
                                 const double* x0_hat, const double* P0, nmpcmc_nmpc_batch** out);
void nmpcmc_gpu_nmpc_batch_destroy(nmpcmc_nmpc_batch* st);
/* NmpcDiagnostics (controllers.hpp:68-73) of one step: the posterior
 * estimate (FilterState) and innovation, SqpReport.converged / .iterations,
 * warm_started, and status = the nmpcmc_status of the exception nmpc_step
 * threw (0 if none). Entries beyond n_x are 0; NaN where the step threw
 * before producing them. */
typedef struct nmpcmc_nmpc_diag {
    double x_filtered[3];
    double P_filtered[9];
    double innovation;
    int32_t converged;
    int32_t sqp_iterations;
    int32_t warm_started;
    int32_t status;
} nmpcmc_nmpc_diag;
/* nmpc_step (controllers.hpp:92-93, controllers.cpp:114-212) on every
 * instance: measurement y[b] at time t[b]; setpoints[b*N + k] = zbar at
 * stage k+1 (NULL: the scenario's SetpointProfile at t[b] + (k+1) Ts, as
 * run_closed_loop passes them); no disturbance. u_out[b] = the applied
 * input, NaN when the step threw (diag status). The states advance exactly
 * as the reference's NmpcState does, including under exceptions. HOST
 * buffers, synchronous; diag may be NULL. One warp per instance on K3w's
 * code path; bitwise the reference's results. */
int nmpcmc_gpu_nmpc_step_batch(nmpcmc_gpu_ctx* ctx, nmpcmc_nmpc_batch* st, const double* t, const double* y,
                               const double* setpoints, double* u_out, nmpcmc_nmpc_diag* diag);
/* Read the states back: x_hat[B*n_x], P[B*n_x*n_x] (the filter prediction
 * valid at the next sample), last_xi[B*N*(1+n_x)], last_lambda[B*N*n_x],
 * last_pi_l[B*N], last_pi_u[B*N] (meaningful where warm[b] = 1), warm[B].
 * Any pointer may be NULL. */
int nmpcmc_gpu_nmpc_batch_get(nmpcmc_nmpc_batch* st, double* x_hat, double* P, double* last_xi,
                              double* last_lambda, double* last_pi_l, double* last_pi_u, int32_t* warm);
int64_t nmpcmc_gpu_nmpc_batch_size(const nmpcmc_nmpc_batch* st);

/* ---- Batched SQP on stagewise quadratic NLPs ---
 * sqp_solve (sqp.hpp:148-151, sqp.cpp:182-411) through the SqpProblem
 * interface (sqp.hpp:15-25) on `batch` problems of the quadratic kind --
 * the problems the reference's SQP tests pose: xi = (u_0, x_1, ...,
 * u_{N-1}, x_N), n_u = 1, n_x = 1 or 3, x_0 given,
 *   f = sum_k [1/2 R_k u_k^2 + r_k u_k + 1/2 x_{k+1}' Q_k x_{k+1} + q_k' x_{k+1}]
 *   x_{k+1} = A_k x_k + B_k u_k + c_k,   u_min <= u_k <= u_max.
 * problems: HOST, batch * nmpcmc_qnlp_doubles(N, n_x) doubles; per problem
 * x0[n_x] u_min u_max, then per stage k = 0..N-1: R r Q[n_x*n_x] q[n_x]
 * A[n_x*n_x] B[n_x] c[n_x] (column-major). The objective and dynamics are
 * evaluated in the order documented in csrc/nmpc_gen_kernel.cuh (Qnlp).
 * xi0: HOST batch * N*(1+n_x) start iterates, or NULL for zeros; duals start
 * at zero, Hessian blocks at identity. Outputs as nmpcmc_gpu_solve_ocp_batch
 * plus iterations (SqpReport::iterations). One warp per problem. */
typedef struct nmpcmc_qnlp_dims {
    int32_t N;
    int32_t n_x;  /* 1 or 3 */
    int32_t n_u;  /* must be 1 */
    int32_t _pad;
    nmpcmc_sqp_options sqp;
} nmpcmc_qnlp_dims;
int64_t nmpcmc_qnlp_doubles(int32_t N, int32_t n_x);
int nmpcmc_gpu_sqp_solve_qnlp_batch(nmpcmc_gpu_ctx* ctx, const nmpcmc_qnlp_dims* dims, int64_t batch,
                                    const double* problems, const double* xi0, double* xi, double* lambda,
                                    double* pi_l, double* pi_u, int32_t* converged, int32_t* iterations,
                                    int32_t* status);

#ifdef __cplusplus
}
#endif

#endif /* NMPCMC_GPU_H */
