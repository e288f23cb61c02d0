"""BASELINE config 2 read literally: 1,000 NMPC closed loops with the CD-EKF
and the OCP on the three-state CSTR model (K3w). Times the GPU batch, writes
the result files, and checks the first samples bitwise against the exact-libm
reference (oracle/_ref, when present) with its host-core time beside it.

  python tools/config2_literal.py [n_sims] [out_dir]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_02197_b200 import configs, engine, results  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/config2_literal"
os.makedirs(out, exist_ok=True)
sc = configs.make_scenario("nmpc", N=60, ctrl_variant=configs.THREE_STATE)
ctx = engine.Context(0)
ctx.run(sc, 0, 32)  # warm-up
t = time.perf_counter()
rec, cnt = ctx.run(sc, 0, n, counters=True)
gpu_s = time.perf_counter() - t
mc = engine.McResult(rec, engine.aggregate_stats(rec), gpu_s, cnt, 0)
results.write_aggregate_json(os.path.join(out, "config2_literal_aggregate.json"), sc, mc,
                             extra={"kernel": "K3w (nmpc_genw_kernel<3,3>)"})
results.write_histogram_csv(os.path.join(out, "config2_literal_hist.csv"), engine.phi_histogram(rec["phi"]), sc)
line = {"config": "BASELINE config 2, three-state controller model (CD-EKF + OCP on 3 states), N=60, 720 steps",
        "n_sims": n, "gpu_seconds": gpu_s, "gpu_sims_per_s": n / gpu_s,
        "n_failed": int(rec["failed"].sum()), "phi_mean": mc.aggregate["mean"]}
try:
    from oracle import lib as O
    m = os.cpu_count() or 8  # one sample per host thread
    ref, wall = O.run_batch(O.ref("xlibm"), sc, 0, m, os.cpu_count())
    same = all(np.array_equal(rec[f][:m], ref[f], equal_nan=(f == "phi")) for f in ("phi", "failed", "ocp_solves",
                                                                                  "ocp_failures"))
    _, wall_g = O.run_batch(O.ref("glibc"), sc, 0, m, os.cpu_count())
    line.update(ref_sample=m, ref_bitwise_first_samples=bool(same), ref_sims_per_s=m / wall_g,
                ref_threads=os.cpu_count())
except Exception as exc:  # reference build absent
    line["ref"] = f"unavailable: {exc}"
print(json.dumps(line), flush=True)
