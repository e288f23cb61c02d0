"""BASELINE config 4 scaling sweep on one GPU: NMPC closed loop, horizons
N in {30, 60, 120}, batch sizes from the command line. Prints one JSON line
per point (sims/s, FP64 TFLOP/s from the device work counters, failures).

  python tools/sweep_config4.py [--sims 10000 100000] [--horizons 30 60 120] [--out DIR]

With --out, each point also writes its result files (aggregate JSON with the
scenario echo, Φ histogram CSV; paper_2212_02197_b200/results.py).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2212_02197_b200 import abi, configs, engine, results, workmodel


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sims", type=int, nargs="+", default=[10000])
    ap.add_argument("--horizons", type=int, nargs="+", default=[30, 60, 120])
    ap.add_argument("--kernel", default="warp")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    ctx = engine.Context(0)
    ctx.set_nmpc_kernel(args.kernel)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    for N in args.horizons:
        sc = configs.make_scenario("nmpc", N=N, perturb=True)
        for n in args.sims:
            rec = torch.empty(n * 24, dtype=torch.uint8, device="cuda")
            cnt = torch.empty(n * 64, dtype=torch.uint8, device="cuda")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            ctx.run_device(sc, 0, n, rec.data_ptr(), cnt.data_ptr())
            e1.record(stream)
            torch.cuda.synchronize()
            s = e0.elapsed_time(e1) / 1e3
            r = np.frombuffer(rec.cpu().numpy().tobytes(), dtype=abi.RECORD_DTYPE)
            c = np.frombuffer(cnt.cpu().numpy().tobytes(), dtype=abi.COUNTERS_DTYPE)
            fl = workmodel.nmpc_flops(c)
            agg = engine.aggregate_stats(r)
            if args.out:
                os.makedirs(args.out, exist_ok=True)
                mc = engine.McResult(r, agg, s, c, 0)
                tag = f"cfg4_N{N}_n{n}"
                results.write_aggregate_json(os.path.join(args.out, tag + "_aggregate.json"), sc, mc,
                                             extra={"device_seconds": s, "kernel": args.kernel})
                results.write_histogram_csv(os.path.join(args.out, tag + "_hist.csv"),
                                            engine.phi_histogram(r["phi"]), sc)
            print(json.dumps({"N": N, "n_sims": n, "seconds": s, "sims_per_s": n / s,
                              "fp64_tflops": fl / s / 1e12, "n_failed": agg["n_failed"],
                              "phi_mean": agg["mean"], "ocp_success_pct": agg["ocp_success_pct"],
                              "ipm_stage_iters_per_s": float(c["ipm_stage_iters"].sum()) / s}), flush=True)


if __name__ == "__main__":
    main()
