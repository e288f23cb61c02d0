#!/usr/bin/env python
"""Benchmark of the batched stochastic CSTR closed loop (BASELINE.json).

Workload (BASELINE config 3, the config the "NMPC and PI" metric is quoted
on): NMPC closed loops (one-state controller model, N=60, SQP max_iter=20,
eps=1e-6, 720 control steps of Ts=10 s, 10 Euler-Maruyama substeps) with
per-sample Gaussian parameter uncertainty, run side by side with the PI batch
on identical noise streams and parameters. One step = one batch of S NMPC
samples + the same S PI samples, consecutive global sample indices of the
30,000-sample config (S = 10,000 divides 30,000, so every batch lies inside
the config's index set and the default 3 steps cover it exactly; 4.2 waves of
2,368 resident samples per batch, profiles/r02/r02g_bench_S*.json; each rank takes its own
batches: weak scaling, no data-path collective). value = NMPC samples per
second of the whole job (the PI batch is inside the timed step). At the end
the last step's records are all-gathered by the library over NCCL and the
statistics (K4) computed on the device -- the only collective.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run (one rank per GPU, 127.0.0.1 rendezvous).
--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified reference core, glibc libm) on this host's cores for the same
workload: one load-balanced worker pool over all K steps' samples (the
reference's atomic-counter pattern, montecarlo.cpp:220-245), rank 0 only.
"""
import argparse
import json
import os
import socket
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
    ap.add_argument("--sims-per-step", type=int, default=10000,
                    help="NMPC (and PI) samples per rank per step (10,000 = 30,000 / 3: batches tile config 3)")
    ap.add_argument("--horizon", type=int, default=60)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-legs", action="store_true", help="skip the config 0/1/2 and three-state side legs")
    ap.add_argument("--no-lanes", action="store_true",
                    help="serial batches on one stream (default: NMPCMC_OPT_LANES=2 pipelining)")
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="NMPC samples per step of the CPU reference (0 = host cores)")
    ap.add_argument("--e2e-steps", type=int, default=0, help="steps of the end-to-end leg (0 = max(3, K // 4))")
    return ap.parse_args()


def scenarios(N):
    from paper_2212_02197_b200 import configs
    sc_n = configs.make_scenario("nmpc", N=N, perturb=True)
    sc_p = configs.make_scenario("pi", perturb=True)
    return sc_n, sc_p


def workload_config(args, world):
    return {"workload": "BASELINE config 3: NMPC closed-loop CSTR (N=60) + PI side by side",
            "n_sims_total": TOTAL_SIMS, "sims_per_step_per_rank": args.sims_per_step,
            "index_order": "step j of rank r runs global indices ((j*world + r) * S) mod 30000 + [0, S); "
                           "S divides 30000, so batches tile the config's index set",
            "horizon_N": args.horizon, "control_steps": 720, "Ts": 10.0, "em_substeps": 10,
            "sqp_max_iter": 20, "controller_model": "one_state", "truth_model": "three_state",
            "param_uncertainty_rel_std": [0.05, 0.05, 0.05], "parallelism": f"samples sharded x{world}",
            "l2": "no flush needed: inputs are one 1 KB scenario per launch; the working set is per-sample "
                  "on-chip state (shared memory + an L2-resident slab), regenerated every sample"}


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
def cpu_pool(sc, first, n, cores=None):
    """The unmodified reference (oracle/_ref, glibc): run_closed_loop over
    samples [first, first + n) on a pool of `cores` threads pulling indices
    from an atomic counter (load-balanced: the wall time is not set by one
    straggler per thread). Returns (records, wall_s, cores)."""
    from oracle import lib as O
    L = O.ref("glibc")
    cores = cores or os.cpu_count() or 1
    rec, wall = O.run_batch(L, sc, first, n, cores)
    return rec, wall, cores


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    sc_n, sc_p = scenarios(args.horizon)
    cores = os.cpu_count() or 1
    n = args.cpu_sample or cores
    K = args.steps
    # warm-up: W steps of the (cheap) PI batch and one NMPC step's worth, on
    # indices past the timed range (a CPU pool has no other state to warm)
    for w in range(args.warmup):
        cpu_pool(sc_p, TOTAL_SIMS - (w + 1) * n, n, cores)
    cpu_pool(sc_n, TOTAL_SIMS - n, n, cores)
    # the K steps' samples as ONE pool each (NMPC, PI): per-step time = total / K
    rec_n, wall_n, _ = cpu_pool(sc_n, 0, K * n, cores)
    _, wall_p, _ = cpu_pool(sc_p, 0, K * n, cores)
    total = wall_n + wall_p
    value = n * K / total
    sample = (f"{K} steps x {n} NMPC + {n} PI samples of config 3 (global indices [0, {K * n}), full 720-step "
              f"closed loops), run as one load-balanced pool of {cores} threads per controller "
              f"(reference run_closed_loop, atomic index counter); value = {K * n} / (NMPC + PI wall)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "sims/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": 1e3 * total / K,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded per-sample noise and parameters)",
            "config": workload_config(args, 1),
            "cpu_baseline": {"value": value, "unit": "sims/s", "cores": cores, "kind": "reference",
                             "sample": sample, "nmpc_failed": int(rec_n["failed"].sum()),
                             "nmpc_wall_s": wall_n, "pi_wall_s": wall_p},
            "e2e": {"value": value, "unit": "sims/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- our arm
def _traffic(kernel_control_steps_per_launch):
    """DRAM bytes per bench launch of the NMPC kernel, scaled from the
    committed ncu --set full capture (profiles/ncu_traffic.json: dram read +
    write of one captured launch and that launch's control steps)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None, "no ncu capture committed"
    with open(path) as fh:
        t = json.load(fh)
    per_step = t["dram_bytes"] / t["control_steps"]
    return per_step * kernel_control_steps_per_launch, (
        f"{t['capture']}: {t['dram_bytes'] / 1e6:.1f} MB DRAM read+write over {t['control_steps']} control steps, "
        f"scaled to this launch's control steps ({t['source']})")


def _k3_name(sc):
    """The NMPC kernel the library dispatches for sc (nmpcmc_gpu.cu launch():
    K3 for a one-state controller with N <= 255, stride ws_stride_for(N))."""
    from paper_2212_02197_b200 import abi
    if sc.ctrl_variant != abi.ONE_STATE or sc.N > 255:
        return f"nmpc_genw_kernel<{3 if sc.truth_variant == abi.THREE_STATE else 1},3> (K3w, one warp per sample)"
    st = 32 if sc.N < 32 else 64 if sc.N < 64 else 128 if sc.N < 128 else 256
    return f"nmpc_kernel<{3 if sc.truth_variant == abi.THREE_STATE else 1},{st}> (K3, one warp per sample)"


def run_ours(args):
    import ctypes as C

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2212_02197_b200 import abi, configs, engine, workmodel

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    ctx = engine.Context(local)
    if world > 1:
        # torch.distributed: barrier + max-over-ranks timing, and shipping the
        # library's NCCL id; the record exchange itself is the library's NCCL
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        box = [engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        ctx.comm_init(box[0], rank, world)

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
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    rec_sz, cnt_sz = C.sizeof(abi.SimRecord), C.sizeof(abi.WorkCounters)
    nsteps = W + K
    rec_n = torch.empty((nsteps, S * rec_sz), dtype=torch.uint8, device="cuda")
    rec_p = torch.empty((nsteps, S * rec_sz), dtype=torch.uint8, device="cuda")
    cnt_n = torch.empty((nsteps, S * cnt_sz), dtype=torch.uint8, device="cuda")
    cnt_p = torch.empty((nsteps, S * cnt_sz), dtype=torch.uint8, device="cuda")

    def first_of(j):
        f = ((j * world + rank) * S) % TOTAL_SIMS
        return f if f + S <= TOTAL_SIMS else 0  # S not dividing 30000: restart the set

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
    ocps = int(cn["control_steps"].sum())
    traffic, traffic_note = _traffic(ocps / K)

    # end to end through the public C ABI with HOST buffers: every step enqueues
    # its batches (H2D = the scenario PODs, passed as kernel arguments) and the
    # copy of its records into pinned host memory (D2H); one wait at the end
    Ke = args.e2e_steps or max(3, K // 4)
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

    def timed_leg(sc, n, first=0, counters=True):
        """One device-timed launch of n samples (after a small warm launch)."""
        rec = torch.empty(n * rec_sz, dtype=torch.uint8, device="cuda")
        cnt = torch.empty(n * cnt_sz, dtype=torch.uint8, device="cuda") if counters else None
        if sc.controller == abi.CTRL_PI:
            ctx.run_device(sc, first, n, rec.data_ptr())  # warm (the NMPC kernels ran above)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        e[0].record(stream)
        ctx.run_device(sc, first, n, rec.data_ptr(), cnt.data_ptr() if counters else 0)
        e[1].record(stream)
        torch.cuda.synchronize()
        s = e[0].elapsed_time(e[1]) / 1e3
        c = np.frombuffer(cnt.cpu().numpy().tobytes(), dtype=abi.COUNTERS_DTYPE) if counters else None
        r = np.frombuffer(rec.cpu().numpy().tobytes(), dtype=abi.RECORD_DTYPE)
        return s, c, r

    # final statistics: the library all-gathers the last timed step's records
    # over NCCL (one rank: a device copy) and K4 reduces them on the device
    last = W + K - 1
    all_n = torch.empty(world * S * rec_sz, dtype=torch.uint8, device="cuda")
    all_p = torch.empty(world * S * rec_sz, dtype=torch.uint8, device="cuda")
    ctx.allgather_records(rec_n[last].data_ptr(), S, all_n.data_ptr())
    ctx.allgather_records(rec_p[last].data_ptr(), S, all_p.data_ptr())
    an, hn = ctx.aggregate_device(all_n.data_ptr(), world * S, bins=0)
    ap_, _ = ctx.aggregate_device(all_p.data_ptr(), world * S)

    legs = {}
    if not args.no_legs and rank == 0 and world == 1:  # single-GPU side measurements
        # PI at BASELINE configs 0 and 1 (one launch each); flops from the
        # counters (failed samples count the steps they ran)
        for name, kw, n in (("pi_config0", dict(controller="pi"), 1000),
                            ("pi_config1", dict(controller="pi", perturb=True), TOTAL_SIMS)):
            s, c, r = timed_leg(configs.make_scenario(**kw), n)
            legs[name] = {"n_sims": n, "ms": 1e3 * s, "sims_per_s": n / s,
                          "achieved_tflops": workmodel.pi_flops(int(c["control_steps"].sum())) / s / 1e12,
                          "failed": int(r["failed"].sum())}
        # NMPC config 2 (1,000 unperturbed samples, one launch) with the paper's
        # one-state controller model, and read literally (three-state CD-EKF +
        # OCP, kernel K3w); and config 3 with the three-state model
        for name, kw, n, nx in (("nmpc_config2", dict(controller="nmpc", N=args.horizon), 1000, 1),
                                ("nmpc_config2_three_state", dict(controller="nmpc", N=args.horizon,
                                                                  ctrl_variant=abi.THREE_STATE), 1000, 3),
                                ("nmpc_config3_three_state", dict(controller="nmpc", N=args.horizon, perturb=True,
                                                                  ctrl_variant=abi.THREE_STATE), 2368, 3)):
            s, c, r = timed_leg(configs.make_scenario(**kw), n)
            legs[name] = {"n_sims": n, "s": s, "sims_per_s": n / s, "ocps_per_s": float(c["control_steps"].sum()) / s,
                          "achieved_tflops": workmodel.nmpc_flops(c, nx=nx) / s / 1e12,
                          "failed": int(r["failed"].sum()),
                          "note": "one launch of n samples (includes the final wave's drain)"}
    stats = {"samples": world * S, "computed_by": "K4 on the device after the library's NCCL all-gather",
             "nmpc": {k: an[k] for k in ("n_failed", "mean", "variance", "ocp_solves", "ocp_failures",
                                         "ocp_success_pct")} | {"hist_bins": int(len(hn.counts))},
             "pi": {k: ap_[k] for k in ("n_failed", "mean", "variance")}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = os.cpu_count() or 1
            n = args.cpu_sample or 4 * cores
            _, wn, cores = cpu_pool(sc_n, 0, n)
            _, wp, _ = cpu_pool(sc_p, 0, n)
            cpu = {"value": n / (wn + wp), "unit": "sims/s", "cores": cores, "kind": "reference",
                   "sample": f"first {n} samples of config 3 (NMPC + PI side by side, full 720-step loops), "
                             f"unmodified reference core (oracle/_ref, glibc), one load-balanced pool of "
                             f"{cores} threads per controller",
                   "nmpc_only_sims_per_s": n / wn, "pi_only_sims_per_s": n / wp}
            if legs:
                ref_legs = {}
                for name, kw in (("nmpc_config2", dict(controller="nmpc", N=args.horizon)),
                                 ("nmpc_config2_three_state", dict(controller="nmpc", N=args.horizon,
                                                                   ctrl_variant=abi.THREE_STATE))):
                    r, w, _ = cpu_pool(configs.make_scenario(**kw), 0, cores)
                    ref_legs[name] = {"sims_per_s": cores / w, "sample": f"first {cores} samples, {cores} threads"}
                _, w, _ = cpu_pool(configs.make_scenario("pi", perturb=True), 0, 2000)
                ref_legs["pi_config1"] = {"sims_per_s": 2000 / w, "sample": f"first 2000 samples, {cores} threads"}
                cpu["legs"] = ref_legs
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
            "ocps_per_s": world * ocps / elapsed_max,
            "pipelining": "lanes=2 (NMPCMC_OPT_LANES): consecutive batches overlap at their drain" if lanes
                          else "serial batches on one stream",
            "gpu_launches": 2 * K,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak_fma, "unit": "TFLOP/s",
                         "frac": achieved / peak_fma, "traffic": traffic, "traffic_note": traffic_note,
                         "kernel": _k3_name(sc_n),
                         "kernel_ms_per_step": 1e3 * nmpc_kernel_s / K,
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
            "legs": legs,
            "work_per_nmpc_sample": {k: float(cn[k].sum()) / (S * K) for k in cn.dtype.names},
            "clocks": clocks,
            "stats_last_step": stats,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args):
    """--gpus N outside torchrun: re-launch this script with one rank per GPU
    (torch.distributed.run, 127.0.0.1 rendezvous); rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
    cmd += [a for a in sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
