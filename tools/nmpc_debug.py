"""Compare GPU NMPC trajectories with the golden reference; print first divergence."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import load_golden
from paper_2212_02197_b200 import configs, engine

ctx = engine.Context(0)
for name in sys.argv[1:]:
    d, kw, sc = load_golden(name)
    want = d["rec_xlibm"]
    got, cnt = ctx.run(sc, int(d["first"]), len(want), counters=True)
    eq = (got["phi"] == want["phi"]) | (np.isnan(got["phi"]) & np.isnan(want["phi"]))
    print(name, "phi equal:", eq.sum(), "/", len(want), "failed got/want", got["failed"].sum(), want["failed"].sum(),
          "solves eq", np.mean(got["ocp_solves"] == want["ocp_solves"]), "failures eq", np.mean(got["ocp_failures"] == want["ocp_failures"]))
    print(" got ", got[:6]); print(" want", want[:6]); print(" status", got["status"][:16])
    sct = configs.make_scenario(**kw, record=True)
    wt = d["traj_xlibm"]
    _, tr = ctx.run_traj(sct, int(d["first"]), wt.shape[0])
    for s in range(wt.shape[0]):
        diff = ~((tr[s] == wt[s]) | (np.isnan(tr[s]) & np.isnan(wt[s])))
        rows = np.where(diff.any(axis=1))[0]
        if len(rows):
            r = rows[0]
            print(f"  sample {s}: first diverging row {r} of {wt.shape[1]}: got {tr[s][r]} want {wt[s][r]}")
            if r > 0: print(f"     prev row got {tr[s][r-1]} want {wt[s][r-1]}")
        else:
            print(f"  sample {s}: trajectory identical")
