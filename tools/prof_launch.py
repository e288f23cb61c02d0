"""One NMPC (or PI) launch for ncu captures.

usage: python tools/prof_launch.py {nmpc|nmpc3|pi} <n_sims> <n_steps> [N] [kernel]
kernel: warp (K3, default) | generic_warp (K3w) | generic (K3g).
A warm-up launch of the same configuration runs first, so capture the second
launch (ncu -k regex:<name> -s 1 -c 1). Prints the launch's work counters
(control steps, for scaling the DRAM traffic to the bench's launches).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2212_02197_b200 import abi, configs, engine
    kind, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    N = int(sys.argv[4]) if len(sys.argv) > 4 else 60
    kernel = sys.argv[5] if len(sys.argv) > 5 else "warp"
    ctrl = "pi" if kind == "pi" else "nmpc"
    sc = configs.make_scenario(ctrl, n_steps=steps, N=N, perturb=True,
                               ctrl_variant=abi.THREE_STATE if kind == "nmpc3" else abi.ONE_STATE)
    ctx = engine.Context(0)
    if ctrl == "nmpc":
        ctx.set_nmpc_kernel(kernel)
    elif os.environ.get("NMPCMC_PI_KERNEL"):
        ctx.set_pi_kernel(os.environ["NMPCMC_PI_KERNEL"])
    ctx.run(sc, 0, n)
    t = time.perf_counter()
    rec, cnt = ctx.run(sc, 0, n, counters=True)
    s = time.perf_counter() - t
    print(json.dumps({"kind": kind, "n_sims": n, "n_steps": steps, "N": N, "kernel": kernel, "seconds": s,
                      "control_steps": int(cnt["control_steps"].sum()), "failed": int(rec["failed"].sum())}))


if __name__ == "__main__":
    main()
