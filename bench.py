#!/usr/bin/env python
"""Benchmark of the batched stochastic CSTR closed loop (BASELINE.json).

Workload (BASELINE config 3, the config the "NMPC and PI" metric is quoted
on): NMPC closed loops (one-state controller model, N=60, SQP max_iter=20,
eps=1e-6, 720 control steps of Ts=10 s, 10 Euler-Maruyama substeps) with
per-sample Gaussian parameter uncertainty, run side by side with the PI batch
on identical noise streams and parameters. One step = one batch of S NMPC
samples + the same S PI samples, consecutive global sample indices of the
30,000-sample config (each rank its own range: weak scaling, no data-path
collective). value = NMPC samples per second of the whole job (the PI batch is
inside the timed step). The per-sample records of the last step are gathered
with NCCL at the end for the statistics (the only collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified reference core, glibc libm, its run_closed_loop worker pool)
on this host's cores for the same workload, rank 0 only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TOTAL_SIMS = 30000  # BASELINE config 3 size
METRIC = "CSTR closed-loop NMPC sims/sec (config 3: NMPC N=60 + PI side by side, per-sim parameter uncertainty)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sims-per-step", type=int, default=9472,
                    help="NMPC (and PI) samples per rank per step (9,472 = 4 waves of 148 SMs x 16 resident samples)")
    ap.add_argument("--horizon", type=int, default=60)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-lanes", action="store_true",
                    help="serial batches on one stream (default: NMPCMC_OPT_LANES=2 pipelining)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="NMPC samples for the CPU baseline (0 = host cores)")
    return ap.parse_args()


def scenarios(N):
    from paper_2212_02197_b200 import configs
    sc_n = configs.make_scenario("nmpc", N=N, perturb=True)
    sc_p = configs.make_scenario("pi", perturb=True)
    return sc_n, sc_p


def workload_config(args, world):
    return {"workload": "BASELINE config 3: NMPC closed-loop CSTR (N=60) + PI side by side",
            "n_sims_total": TOTAL_SIMS, "sims_per_step_per_rank": args.sims_per_step,
            "horizon_N": args.horizon, "control_steps": 720, "Ts": 10.0, "em_substeps": 10,
            "sqp_max_iter": 20, "controller_model": "one_state", "truth_model": "three_state",
            "param_uncertainty_rel_std": [0.05, 0.05, 0.05], "parallelism": f"samples sharded x{world}",
            "l2": "working set on chip (smem per sample); inputs are one 1 KB scenario, no L2 flush needed"}


# ------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------- reference arm
def cpu_reference(sc_n, sc_p, n_sims, first=0):
    """The unmodified reference (oracle/_ref, glibc) on all host cores: NMPC
    and PI batches of n_sims samples. Returns (nmpc_wall_s, pi_wall_s, cores)."""
    from oracle import lib as O
    L = O.ref("glibc")
    cores = os.cpu_count() or 1
    _, wall_n = O.run_batch(L, sc_n, first, n_sims, cores)
    _, wall_p = O.run_batch(L, sc_p, first, n_sims, cores)
    return wall_n, wall_p, cores


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    sc_n, sc_p = scenarios(args.horizon)
    cores = os.cpu_count() or 1
    n = args.cpu_sample or cores
    for w in range(args.warmup):
        cpu_reference(sc_n, sc_p, n, first=w * n)
    walls = []
    for k in range(args.steps):
        wn, wp, cores = cpu_reference(sc_n, sc_p, n, first=(args.warmup + k) * n)
        walls.append(wn + wp)
    total = sum(walls)
    value = n * args.steps / total
    sample = (f"{n} NMPC + {n} PI samples per step (full 720-step closed loops, distinct index ranges), "
              f"{cores} worker threads, reference run_closed_loop pool")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "sims/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded per-sample noise and parameters)",
            "config": workload_config(args, 1),
            "cpu_baseline": {"value": value, "unit": "sims/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "sims/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- our arm
def run_ours(args):
    import ctypes as C

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2212_02197_b200 import abi, engine, workmodel

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    sc_n, sc_p = scenarios(args.horizon)
    S, K, W = args.sims_per_step, args.steps, args.warmup
    ctx = engine.Context(local)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    rec_sz, cnt_sz = C.sizeof(abi.SimRecord), C.sizeof(abi.WorkCounters)
    nsteps = W + K
    rec_n = torch.empty((nsteps, S * rec_sz), dtype=torch.uint8, device="cuda")
    rec_p = torch.empty((nsteps, S * rec_sz), dtype=torch.uint8, device="cuda")
    cnt_n = torch.empty((nsteps, S * cnt_sz), dtype=torch.uint8, device="cuda")
    cnt_p = torch.empty((nsteps, S * cnt_sz), dtype=torch.uint8, device="cuda")

    def first_of(j):
        return ((j * world + rank) * S) % TOTAL_SIMS

    lanes = not args.no_lanes
    ev = []

    def step(j, timed):
        """One step: the NMPC batch and the PI batch of the same indices. With
        lanes, consecutive NMPC batches run on alternating library streams, so
        a batch's drain (its last wave of long samples) overlaps the next."""
        first = first_of(j)
        if timed and not lanes:
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(stream)
        ctx.run_device(sc_n, first, S, rec_n[j].data_ptr(), cnt_n[j].data_ptr())
        if timed and not lanes:
            e[1].record(stream)
        ctx.run_device(sc_p, first, S, rec_p[j].data_ptr(), cnt_p[j].data_ptr())
        if timed and not lanes:
            e[2].record(stream)
            ev.append(e)

    ctx.set_lanes(2 if lanes else 1)
    for j in range(W):
        step(j, False)
    ctx.join()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for j in range(W, W + K):
        step(j, True)
    ctx.join()  # the stream now waits for every lane
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    elapsed = t0.elapsed_time(t1) / 1e3
    elapsed_max = max_over_ranks(elapsed)
    value = world * S * K / elapsed_max

    # kernel times: serial mode brackets each launch with events on the launch
    # stream; with lanes the launches overlap, so the NMPC kernel's time per
    # launch is the pipeline period (elapsed / K, PI on its own lane inside it)
    # and the PI kernel is timed alone once after the timed region
    if lanes:
        nmpc_kernel_s = elapsed
        ctx.set_lanes(1)
        pe = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        pe[0].record(stream)
        ctx.run_device(sc_p, first_of(W), S, rec_p[W].data_ptr(), cnt_p[W].data_ptr())
        pe[1].record(stream)
        torch.cuda.synchronize()
        pi_kernel_s = K * pe[0].elapsed_time(pe[1]) / 1e3
    else:
        nmpc_kernel_s = sum(e[0].elapsed_time(e[1]) for e in ev) / 1e3
        pi_kernel_s = sum(e[1].elapsed_time(e[2]) for e in ev) / 1e3

    # roofline of the dominant kernel (NMPC) from the device work counters
    cn = np.frombuffer(cnt_n[W:].cpu().numpy().tobytes(), dtype=abi.COUNTERS_DTYPE)
    cp = np.frombuffer(cnt_p[W:].cpu().numpy().tobytes(), dtype=abi.COUNTERS_DTYPE)
    nmpc_flops = workmodel.nmpc_flops(cn)
    pi_flops = workmodel.pi_flops(int(cp["control_steps"].sum()))
    peak_fma = ctx.fp64_peak(True)
    peak_add = ctx.fp64_peak(False)
    achieved = nmpc_flops / nmpc_kernel_s / 1e12

    # end to end through the public C ABI with HOST buffers: every step enqueues
    # its batches (H2D = the scenario PODs, passed as kernel arguments) and the
    # copy of its records into pinned host memory (D2H); one wait at the end
    Ke = K
    ctx.set_lanes(2 if lanes else 1)
    host_n = [torch.empty(S * rec_sz, dtype=torch.uint8).pin_memory() for _ in range(Ke)]
    host_p = [torch.empty(S * rec_sz, dtype=torch.uint8).pin_memory() for _ in range(Ke)]
    torch.cuda.synchronize()
    barrier()
    te = time.perf_counter()
    for j in range(Ke):
        ctx.run_async(sc_n, first_of(W + K + j), S, host_n[j].data_ptr())
        ctx.run_async(sc_p, first_of(W + K + j), S, host_p[j].data_ptr())
    ctx.wait()
    e2e_s = max_over_ranks(time.perf_counter() - te)
    e2e_value = world * S * Ke / e2e_s
    ctx.set_lanes(1)

    # PI at BASELINE config 1's own size (30,000 perturbed samples, one launch):
    # the step's PI batch above is launch-bound at S samples
    n_pi = TOTAL_SIMS
    rec_pi = torch.empty(n_pi * rec_sz, dtype=torch.uint8, device="cuda")
    ctx.run_device(sc_p, 0, n_pi, rec_pi.data_ptr())
    pe = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    pe[0].record(stream)
    ctx.run_device(sc_p, 0, n_pi, rec_pi.data_ptr())
    pe[1].record(stream)
    torch.cuda.synchronize()
    pi_cfg1_s = pe[0].elapsed_time(pe[1]) / 1e3

    # final statistics: gather the last timed step's records from every rank (NCCL)
    last_n, last_p = rec_n[W + K - 1], rec_p[W + K - 1]
    if world > 1:
        gn = torch.empty((world, last_n.numel()), dtype=torch.uint8, device="cuda")
        gp = torch.empty((world, last_p.numel()), dtype=torch.uint8, device="cuda")
        dist.all_gather_into_tensor(gn, last_n.contiguous())
        dist.all_gather_into_tensor(gp, last_p.contiguous())
    else:
        gn, gp = last_n[None], last_p[None]
    stats = None
    if rank == 0:
        all_n = np.frombuffer(gn.cpu().numpy().tobytes(), dtype=abi.RECORD_DTYPE)
        all_p = np.frombuffer(gp.cpu().numpy().tobytes(), dtype=abi.RECORD_DTYPE)
        an, ap_ = engine.aggregate_stats(all_n), engine.aggregate_stats(all_p)
        hn = engine.phi_histogram(all_n["phi"])
        stats = {"samples": int(len(all_n)),
                 "nmpc": {k: an[k] for k in ("n_failed", "mean", "variance", "ocp_solves", "ocp_failures",
                                             "ocp_success_pct")} | {"hist_bins": int(len(hn.counts))},
                 "pi": {k: ap_[k] for k in ("n_failed", "mean", "variance")}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = os.cpu_count() or 1
            n = args.cpu_sample or cores
            wn, wp, cores = cpu_reference(sc_n, sc_p, n, first=0)
            cpu = {"value": n / (wn + wp), "unit": "sims/s", "cores": cores, "kind": "reference",
                   "sample": f"first {n} samples of config 3 (NMPC + PI side by side, full 720-step loops), "
                             f"unmodified reference core (oracle/_ref, glibc), {cores} worker threads",
                   "nmpc_only_sims_per_s": n / wn, "pi_only_sims_per_s": n / wp}
        except Exception as exc:  # the reference build is missing on this host
            cpu = {"value": None, "unit": "sims/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "sims/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": 1e3 * elapsed_max / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded per-sample noise and parameters)",
            "config": workload_config(args, world),
            "e2e": {"value": e2e_value, "unit": "sims/s", "h2d_bytes_per_step": 2 * C.sizeof(abi.Scenario),
                    "d2h_bytes_per_step": 2 * S * rec_sz, "steps": Ke,
                    "api": "nmpcmc_gpu_run_async (host records, pinned) x 2 per step + nmpcmc_gpu_wait"},
            "pipelining": "lanes=2 (NMPCMC_OPT_LANES): consecutive batches overlap at their drain" if lanes
                          else "serial batches on one stream",
            "gpu_launches": 2 * K,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak_fma, "unit": "TFLOP/s",
                         "frac": achieved / peak_fma, "traffic": None,
                         "traffic_note": "ncu --set full of the same kernel (2,368 samples x 6 steps): 325.5 MB DRAM "
                                         "per launch, 2.4 GB/s -- workspace spill from L2, HBM idle "
                                         "(profiles/r01d_nmpc_ncu_summary.md)",
                         "kernel": "nmpc_kernel<3,64>", "kernel_ms_per_step": 1e3 * nmpc_kernel_s / K,
                         "kernel_time": "pipeline period elapsed/K (launches overlap on two lanes)" if lanes
                                        else "CUDA events around each launch on its stream",
                         "flops_per_step": nmpc_flops / K,
                         "peak_source": "measured on this GPU: DFMA throughput kernel (nmpcmc_gpu_fp64_peak), "
                                        "2 flops/DFMA; MEASURED_PEAKS.json has no FP64 entry",
                         "peak_nonfma_issue": peak_add,
                         "frac_of_nonfma_issue": achieved / peak_add,
                         "note": "--fmad=false for bit parity: no FMA contraction, so the attainable rate "
                                 "is the FP64 issue rate (peak_nonfma_issue)"},
            "pi": {"kernel_ms_per_step": 1e3 * pi_kernel_s / K, "sims_per_s_kernel": S * K / pi_kernel_s,
                   "achieved_tflops": pi_flops / pi_kernel_s / 1e12},
            "pi_config1": {"n_sims": n_pi, "ms": 1e3 * pi_cfg1_s, "sims_per_s": n_pi / pi_cfg1_s,
                           "achieved_tflops": workmodel.pi_flops(n_pi * 720) / pi_cfg1_s / 1e12,
                           "note": "BASELINE config 1 (PI, 30k samples, per-sim parameters) as one launch, "
                                   "device-timed; reference PI rate: cpu_baseline.pi_only_sims_per_s"},
            "work_per_nmpc_sample": {k: float(cn[k].sum()) / (S * K) for k in cn.dtype.names},
            "clocks": clocks,
            "stats_last_step": stats,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
