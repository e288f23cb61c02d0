"""Randomised scenario fixtures (tests/golden/fuzz.npz) from the UNMODIFIED
reference: closed-loop records of many small random scenarios covering the
option space (horizons, RK / EM step counts, SQP limits and tolerances, noise
on/off, filter settings, unstable-branch setpoints, both controller and truth
models, parameter perturbation, bounds). Scenarios the reference's own
validation rejects are skipped. Raw scenario bytes are stored (these are not
configs.make_scenario outputs).

  python tests/golden/make_fuzz.py [n_scenarios] [seed] [--long]

--long: NMPC only, 20-60 control steps, horizons 10-80 -> fuzz_long.npz.
"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import lib as O  # noqa: E402
from paper_2212_02197_b200 import abi, configs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def random_scenario(rng, long=False):
    nmpc = long or rng.uniform() < 0.8
    steps = int(rng.integers(20, 61)) if long else int(rng.integers(4, 21))
    Ts = float(rng.choice([2.0, 5.0, 10.0, 20.0]))
    kw = dict(controller="nmpc" if nmpc else "pi", n_steps=steps, Ts=Ts, Ns=int(rng.integers(1, 13)),
              N=int(rng.integers(10, 81)) if long else int(rng.integers(3, 41)), Nc=int(rng.integers(1, 7)), np_=int(rng.integers(1, 7)),
              max_iter=int(rng.integers(1, 21)), eps=float(rng.choice([1e-4, 1e-6, 1e-8])),
              perturb=bool(rng.uniform() < 0.5), rel_std=tuple(float(x) for x in rng.uniform(0.0, 0.2, 3)),
              base_seed=int(rng.integers(0, 2**62)),
              ctrl_variant=abi.THREE_STATE if rng.uniform() < 0.3 else abi.ONE_STATE,
              truth_variant=abi.ONE_STATE if rng.uniform() < 0.25 else abi.THREE_STATE,
              noise_R=float(rng.choice([0.0, 0.01, 0.3])), R_filter=float(rng.choice([1e-4, 0.01, 1.0])),
              Qz=float(rng.choice([0.1, 1.0, 10.0])), sigma_t=float(rng.choice([0.0, 2.5, 8.0])),
              T0=float(rng.choice([330.0, 335.0, 345.0])),
              pi_gains=(float(rng.uniform(-20, -1)), float(rng.uniform(-0.5, 0.0)), float(rng.uniform(-0.5, 0.0)),
                        float(rng.uniform(300, 800))))
    nsp = int(rng.integers(1, 6))
    tf = steps * Ts
    times = tuple(sorted([0.0] + [float(x) for x in rng.uniform(0.0, tf, nsp - 1)]))
    kw["setpoints"] = (times, tuple(float(v) for v in rng.uniform(320.0, 360.0, nsp)))
    sc = configs.make_scenario(**kw)
    sc.has_noise_R = 0 if rng.uniform() < 0.15 else 1
    if rng.uniform() < 0.3:
        sc.truth.sigmaA = sc.truth.sigmaB = 0.06
    if rng.uniform() < 0.2:
        sc.u_min, sc.u_max = 200.0, 900.0
    sc.sqp.qp_max_iter = int(rng.integers(5, 51))
    sc.sqp.max_backtracks = int(rng.integers(1, 31))
    sc.sqp.backtrack_factor = float(rng.choice([0.3, 0.5, 0.7]))
    sc.sqp.c1 = float(rng.choice([1e-4, 1e-2]))
    return sc


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    long = "--long" in sys.argv
    n = int(args[0]) if len(args) > 0 else 60
    seed = int(args[1]) if len(args) > 1 else 20261020
    rng = np.random.default_rng(seed)
    Lx, Lg = O.ref("xlibm"), O.ref("glibc")
    scen, rec_x, rec_g, firsts = [], [], [], []
    t0 = time.time()
    while len(scen) < n:
        sc = random_scenario(rng, long)
        nbar = C.c_int(0)
        if Lx.nmpcmc_ref_validate(C.byref(sc), C.byref(nbar)) != 0:
            continue
        first = int(rng.integers(0, 10**6))
        rx, _ = O.run_batch(Lx, sc, first, 6, 6)
        rg, _ = O.run_batch(Lg, sc, first, 6, 6)
        scen.append(np.frombuffer(bytes(sc), dtype=np.uint8))
        rec_x.append(rx)
        rec_g.append(rg)
        firsts.append(first)
    np.savez_compressed(os.path.join(OUT, "fuzz_long.npz" if long else "fuzz.npz"), scenarios=np.array(scen), rec_xlibm=np.array(rec_x),
                        rec_glibc=np.array(rec_g), first=np.array(firsts), seed=np.array(seed))
    fails = int(sum(int(r["failed"].sum()) for r in rec_x))
    print(f"fuzz: {n} scenarios x 6 samples in {time.time() - t0:.1f}s, {fails} failed samples")


if __name__ == "__main__":
    main()
