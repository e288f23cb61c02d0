"""A/B timing of several builds of libnmpcmc_gpu.so on the same box.

usage: python tools/ab_time.py <n_sims> <n_steps> <N> lib1.so [lib2.so ...]
Each library runs in its own process (NMPCMC_GPU_LIB); records are hashed so
the builds can be checked for bitwise-identical results.
"""
import hashlib
import os
import subprocess
import sys

CHILD = r"""
import sys, time, hashlib
sys.path.insert(0, %r)
from paper_2212_02197_b200 import configs, engine
n, steps, N = %d, %d, %d
sc = configs.make_scenario("nmpc", n_steps=steps, N=N, perturb=True)
ctx = engine.Context(0)
ctx.set_nmpc_kernel("warp")
ctx.run(sc, 0, min(n, 2368))  # warm-up
best = 1e30
for _ in range(2):
    t = time.perf_counter()
    rec, cnt = ctx.run(sc, 0, n, counters=True)
    best = min(best, time.perf_counter() - t)
ipm = int(cnt["ipm_stage_iters"].sum())
h = hashlib.sha1(rec.tobytes()).hexdigest()[:12]
print(f"{best*1e3:9.1f} ms  {ipm/best/1e6:7.1f} M ipm-stage-iters/s  {n/best*steps/720:7.1f} sims/s(720-step equiv)  rec {h}")
"""


def main():
    n, steps, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for lib in sys.argv[4:]:
        env = dict(os.environ, NMPCMC_GPU_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", CHILD % (root, n, steps, N)], env=env,
                             capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr.strip()[-300:]
        print(f"{os.path.basename(lib):24s} {line}", flush=True)


if __name__ == "__main__":
    main()
