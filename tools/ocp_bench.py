"""Throughput of the batched OCP service (sqp_solve on the regulator
OcpProblem, one warp per instance) vs the reference's sqp_solve on the host
cores: ocp_bench.py [batch] [N] [three]. Random initial states around the
operating range, random times over the setpoint profile; cold starts."""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_02197_b200 import configs, engine, qp as Q  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
N = int(sys.argv[2]) if len(sys.argv) > 2 else 60
three = len(sys.argv) > 3 and sys.argv[3] == "three"
kw = dict(controller="nmpc", N=N, ctrl_variant=configs.THREE_STATE if three else configs.ONE_STATE)
sc = configs.make_scenario(**kw)
nx = 3 if three else 1
rng = np.random.default_rng(7)
p = configs.study_params()
T = rng.uniform(322.0, 348.0, B)
x0 = np.array([configs.manifold_state(p, t)[3 - nx:] for t in T]) * (1.0 + 0.01 * rng.standard_normal((B, nx)))
t0 = rng.uniform(0.0, 7000.0, B)
ctx = engine.Context(0)
Q.solve_ocp_batch(sc, x0[:64], t0[:64], ctx=ctx)
t = time.perf_counter()
out = Q.solve_ocp_batch(sc, x0, t0, ctx=ctx)
dt = time.perf_counter() - t
line = {"batch": B, "N": N, "model": "three-state" if three else "one-state", "gpu_s": dt, "gpu_ocps_per_s": B / dt,
        "converged_frac": float(out["converged"].mean())}
try:
    from oracle import lib as O
    L = O.ref("xlibm")
    n = min(B, 4 * (os.cpu_count() or 1))
    chunks = np.array_split(np.arange(n), os.cpu_count() or 1)
    t = time.perf_counter()
    with ThreadPoolExecutor(len(chunks)) as ex:
        parts = list(ex.map(lambda c: O.solve_ocp_batch(L, sc, x0[c], t0[c]), chunks))
    wall = time.perf_counter() - t
    ref_xi = np.concatenate([q["xi"] for q in parts])
    line.update(ref_ocps_per_s=n / wall, ref_threads=len(chunks), ref_sample=n,
                bitwise_sample=bool(np.array_equal(ref_xi, out["xi"][:n])))
except Exception as exc:
    line["ref"] = f"unavailable: {exc}"
print(json.dumps(line), flush=True)
