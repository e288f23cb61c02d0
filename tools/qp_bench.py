"""Throughput of the batched QP service (K5) vs the reference's solve_qp on
one host core: qp_bench.py [batch] [N] [nx] [nu]. Random box-constrained
instances (paper_2212_02197_b200.qp.random_instance), seeded."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_02197_b200 import engine, qp as Q  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
N, nx, nu = (int(v) for v in (sys.argv[2:5] if len(sys.argv) > 4 else (60, 3, 1)))
rng = np.random.default_rng(11)
base = Q.pack([Q.random_instance(rng, N, nx, nu) for _ in range(256)], nx, nu)
packed = np.ascontiguousarray(np.concatenate([base] * (batch // 256 + 1))[:batch])
ctx = engine.Context(0)
Q.solve_qp_batch(packed[:512], nx, nu, ctx=ctx, raw=True)
t = time.perf_counter()
sol, st, it = Q.solve_qp_batch(packed, nx, nu, ctx=ctx, raw=True)
dt = time.perf_counter() - t
line = {"batch": batch, "N": N, "nx": nx, "nu": nu, "gpu_s": dt, "gpu_qps_per_s": batch / dt,
        "optimal_frac": float(np.mean(st == Q.OPTIMAL)), "mean_iters": float(it.mean())}
try:
    from oracle import lib as O
    L = O.ref("glibc")
    n = 256
    t = time.perf_counter()
    rsol, rst, rit = O.solve_qp_batch(L, packed[:n], nx, nu)
    line["ref_1core_qps_per_s"] = n / (time.perf_counter() - t)
    line["bitwise_first_256"] = bool(np.array_equal(rsol, sol[:n]) and np.array_equal(rst, st[:n]))
except Exception as exc:  # reference build absent (GPU box)
    line["ref"] = f"unavailable: {exc}"
print(line, flush=True)
