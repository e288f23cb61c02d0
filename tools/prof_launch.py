"""One closed-loop launch for profiling: prof_launch.py <pi|nmpc> <n_sims> <n_steps> <N> [repeats]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_02197_b200 import configs, engine
ctl, n, steps, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rep = int(sys.argv[5]) if len(sys.argv) > 5 else 1
sc = configs.make_scenario(ctl, n_steps=steps, N=N, perturb=True)
ctx = engine.Context(0)
for _ in range(rep):
    rec, cnt = ctx.run(sc, 0, n, counters=True)
print("failed", int(rec["failed"].sum()), "ipm", int(cnt["ipm_stage_iters"].sum()), "shoot", int(cnt["shoot_full"].sum()))
