"""One closed-loop launch for profiling/timing:
prof_launch.py <pi|nmpc> <n_sims> <n_steps> <N> [kernel] [warps_per_sm] [repeats]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_02197_b200 import configs, engine
ctl, n, steps, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
kind = sys.argv[5] if len(sys.argv) > 5 else "thread"
wps = int(sys.argv[6]) if len(sys.argv) > 6 else 8
rep = int(sys.argv[7]) if len(sys.argv) > 7 else 1
sc = configs.make_scenario(ctl, n_steps=steps, N=N, perturb=True)
ctx = engine.Context(0)
ctx.set_nmpc_kernel(kind)
ctx.set_tps_warps_per_sm(wps)
for _ in range(rep):
    t = time.perf_counter()
    rec, cnt = ctx.run(sc, 0, n, counters=True)
    dt = time.perf_counter() - t
    ipm = int(cnt["ipm_stage_iters"].sum())
    print(f"{kind} wps={wps} n={n} steps={steps}: {dt*1e3:.1f} ms, {ipm/dt/1e6:.1f} M ipm-stage-iters/s, "
          f"failed {int(rec['failed'].sum())}, ipm {ipm}, shoot {int(cnt['shoot_full'].sum())}", flush=True)
