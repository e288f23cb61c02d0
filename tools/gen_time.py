"""Time the generic NMPC kernels: gen_time.py <n> <steps> <N> [ctrl_variant: 0=three, 1=one] [generic|generic_warp]"""
import sys, os, time, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_02197_b200 import configs, engine, workmodel
n, steps, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cv = int(sys.argv[4]) if len(sys.argv) > 4 else 0
kind = sys.argv[5] if len(sys.argv) > 5 else "generic"
sc = configs.make_scenario("nmpc", n_steps=steps, N=N, perturb=True, ctrl_variant=cv)
ctx = engine.Context(0)
ctx.set_nmpc_kernel(kind)
ctx.run(sc, 0, min(n, 256))
reps = int(os.environ.get("GEN_TIME_REPS", "3"))
times = []
for _ in range(reps):
    t = time.perf_counter()
    rec, cnt = ctx.run(sc, 0, n, counters=True)
    times.append(time.perf_counter() - t)
dt = min(times)
ipm = int(cnt["ipm_stage_iters"].sum())
print(f"{kind} ctrl_variant={cv} n={n} steps={steps} N={N}: {dt*1e3:.1f} ms, {n*steps/720/dt:.2f} sims/s (720-step equiv), "
      f"{ipm/dt/1e6:.1f} M ipm-stage-iters/s, {workmodel.nmpc_flops(cnt, 3 if cv == 0 else 1)/dt/1e12:.3f} TF/s, "
      f"failed {int(rec['failed'].sum())}, rec {hashlib.sha1(rec.tobytes()).hexdigest()[:12]}, "
      f"runs ms {[round(x * 1e3, 1) for x in times]}", flush=True)
