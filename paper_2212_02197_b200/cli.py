"""Command-line driver (SPEC.md cli module: simulate | montecarlo | benchmark |
histogram, --config PATH, --set section.key=value, --out DIR, --workers N,
--sims N, --seed N). The reference ships only a stub
(/root/reference/proj/tools/src/main.cpp:3-6); this is the GPU form of the
workflows it specifies, over the same engine the C ABI exposes.

  python -m paper_2212_02197_b200.cli montecarlo --config exp.ini --set controller.N=30 --sims 10000
  python -m paper_2212_02197_b200.cli simulate --set controller.type=pi --out runs/pi
  python -m paper_2212_02197_b200.cli benchmark --workers 1,2,4,8 --sims 2000
  python -m paper_2212_02197_b200.cli histogram --in runs/mc/records.csv --bins 50

Config file: INI sections (human-editable key/value with sections), every
key optional; defaults are BASELINE config 0 / 2 (configs.make_scenario).
  [controller] type (pi|nmpc), variant (one_state|three_state), N, Nc, np,
               Qz, R_filter, u_min, u_max, kP, kI, kaw, u_bar, I_hat, eps,
               max_iter, max_backtracks, c1, backtrack_factor, qp_tol, qp_max_iter
  [model]      truth_variant, V, k0, EaR, beta, cA_in, cB_in, cT_in, sigmaA,
               sigmaB, sigmaT (truth and controller model alike)
  [noise]      R (measurement variance; 0 = exact measurements)
  [scenario]   t0, tf, Ts, Ns, T0, seed, setpoint_times, setpoint_values
               (comma lists), perturb, perturb_rel_std (comma list of 3)
  [run]        sims, first, workers (GPU count), stride, trajectories, bins
`--workers` counts GPUs (the reference's worker threads); records are bitwise
independent of it. Every output file embeds the effective scenario and seed
(results.py). On failure the exit status is non-zero and a machine-readable
error record is printed to stderr (and written to OUT/error.json).
"""
import argparse
import configparser
import csv
import json
import math
import os
import sys
import time

import numpy as np

from . import abi, configs, engine, results

SECTIONS = {
    "controller": {"type", "variant", "N", "Nc", "np", "Qz", "R_filter", "u_min", "u_max", "kP", "kI", "kaw",
                   "u_bar", "I_hat", "eps", "max_iter", "max_backtracks", "c1", "backtrack_factor", "qp_tol",
                   "qp_max_iter"},
    "model": {"truth_variant", "V", "k0", "EaR", "beta", "cA_in", "cB_in", "cT_in", "sigmaA", "sigmaB", "sigmaT"},
    "noise": {"R"},
    "scenario": {"t0", "tf", "Ts", "Ns", "T0", "seed", "setpoint_times", "setpoint_values", "perturb",
                 "perturb_rel_std"},
    "run": {"sims", "first", "workers", "stride", "trajectories", "bins"},
}
VARIANTS = {"one_state": abi.ONE_STATE, "three_state": abi.THREE_STATE}


class ConfigError(ValueError):
    """ParseError / ValidationError of load_config (location or invariant named)."""

    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


def _floats(v):
    return [float(x) for x in str(v).replace(";", ",").split(",") if x.strip()]


def _bool(v):
    s = str(v).strip().lower()
    if s in ("1", "true", "yes", "on"):
        return True
    if s in ("0", "false", "no", "off"):
        return False
    raise ValueError(f"not a boolean: {v!r}")


def load_config(path=None, overrides=()):
    """load_config (SPEC.md cli): the config file (optional) plus --set
    overrides -> {section: {key: str}}; unknown sections/keys and parse errors
    raise ConfigError naming the location."""
    cp = configparser.ConfigParser(interpolation=None, inline_comment_prefixes=("#", ";"))
    cp.optionxform = str
    if path is not None:
        if not os.path.exists(path):
            raise ConfigError("ParseError", f"{path}: no such file")
        try:
            with open(path) as fh:
                cp.read_file(fh, source=path)
        except configparser.Error as e:
            raise ConfigError("ParseError", f"{path}: {e}") from e
    cfg = {s: dict(cp.items(s)) for s in cp.sections()}
    for ov in overrides:
        if "=" not in ov or "." not in ov.split("=", 1)[0]:
            raise ConfigError("ParseError", f"--set {ov!r}: expected section.key=value")
        k, v = ov.split("=", 1)
        s, key = k.split(".", 1)
        cfg.setdefault(s.strip(), {})[key.strip()] = v.strip()
    for s, kv in cfg.items():
        if s not in SECTIONS:
            raise ConfigError("ParseError", f"unknown section [{s}]")
        for k in kv:
            if k not in SECTIONS[s]:
                raise ConfigError("ParseError", f"unknown key {s}.{k}")
    return cfg


def build_scenario(cfg):
    """The effective nmpcmc_scenario of a config: configs.make_scenario
    defaults, then every given key; validated (validate_scenario,
    montecarlo.cpp:34-63) with the violated invariant in the error."""
    c, m, n, s = (cfg.get(k, {}) for k in ("controller", "model", "noise", "scenario"))
    try:
        kw = {"controller": c.get("type", "pi")}
        if kw["controller"] not in ("pi", "nmpc"):
            raise ValueError(f"controller.type must be pi or nmpc, got {kw['controller']!r}")
        if "variant" in c:
            kw["ctrl_variant"] = VARIANTS[c["variant"]]
        if "truth_variant" in m:
            kw["truth_variant"] = VARIANTS[m["truth_variant"]]
        for key, name, conv in (("N", "N", int), ("Nc", "Nc", int), ("np", "np_", int), ("Qz", "Qz", float),
                                ("R_filter", "R_filter", float), ("eps", "eps", float),
                                ("max_iter", "max_iter", int)):
            if key in c:
                kw[name] = conv(c[key])
        if "R" in n:
            kw["noise_R"] = float(n["R"])
        for key, name, conv in (("Ts", "Ts", float), ("Ns", "Ns", int), ("T0", "T0", float),
                                ("seed", "base_seed", int)):
            if key in s:
                kw[name] = conv(s[key])
        if "sigmaT" in m:
            kw["sigma_t"] = float(m["sigmaT"])
        if "perturb" in s:
            kw["perturb"] = _bool(s["perturb"])
        if "perturb_rel_std" in s:
            kw["rel_std"] = tuple(_floats(s["perturb_rel_std"]))
        if "setpoint_times" in s or "setpoint_values" in s:
            kw["setpoints"] = (tuple(_floats(s.get("setpoint_times", "0"))),
                               tuple(_floats(s.get("setpoint_values", "335"))))
        Ts = kw.get("Ts", 10.0)
        t0 = float(s.get("t0", 0.0))
        tf = float(s["tf"]) if "tf" in s else t0 + 720 * Ts
        steps = (tf - t0) / Ts
        kw["n_steps"] = max(int(round(steps)), 1)
        sc = configs.make_scenario(**kw)
        sc.t0, sc.tf = t0, tf
        for key in ("u_min", "u_max"):
            if key in c:
                setattr(sc, key, float(c[key]))
                setattr(sc.truth, key, float(c[key]))
                setattr(sc.ctrl, key, float(c[key]))
        for key in ("kP", "kI", "kaw", "u_bar", "I_hat"):
            if key in c:
                setattr(sc.pi, key, float(c[key]))
        for key, conv in (("max_backtracks", int), ("c1", float), ("backtrack_factor", float), ("qp_tol", float),
                          ("qp_max_iter", int)):
            if key in c:
                setattr(sc.sqp, key, conv(c[key]))
        for key in ("V", "k0", "EaR", "beta", "cA_in", "cB_in", "cT_in", "sigmaA", "sigmaB"):
            if key in m:
                setattr(sc.truth, key, float(m[key]))
                setattr(sc.ctrl, key, float(m[key]))
    except (KeyError, ValueError) as e:
        raise ConfigError("ValidationError", f"bad value: {e}") from e
    try:
        engine.validate_scenario(sc)
    except engine.NmpcmcError as e:
        raise ConfigError("ValidationError", f"{e} ({_violated(sc)})") from e
    return sc


def _violated(sc):
    """Name the validate_scenario invariant (montecarlo.cpp:34-63) a
    scenario breaks, for the error record."""
    steps = (sc.tf - sc.t0) / sc.Ts if sc.Ts > 0 else float("nan")
    if not sc.Ts > 0 or not sc.tf > sc.t0:
        return "scenario: Ts > 0 and tf > t0 required"
    if abs(steps - round(steps)) > 1e-9 * max(1.0, abs(steps)):
        return f"N_bar integrality rule: (tf - t0) / Ts = {steps!r} is not an integer"
    if sc.Ns < 1:
        return "scenario.Ns must be at least 1"
    if not sc.u_min <= sc.u_max:
        return "controller.u_min <= controller.u_max required"
    if sc.n_setpoints < 1 or sc.sp_times[0] > sc.t0:
        return "setpoint profile must cover t0"
    if sc.controller == abi.CTRL_NMPC and (sc.N < 1 or sc.Nc < 1 or sc.np < 1):
        return "controller.N, Nc, np must be positive"
    return "see validate_scenario"


def _run_cfg(cfg, args):
    r = cfg.get("run", {})
    sims = args.sims if args.sims is not None else int(r.get("sims", 1000))
    workers = args.workers if args.workers is not None else r.get("workers", "1")
    return sims, int(r.get("first", 0)), str(workers), int(r.get("trajectories", 0)), int(r.get("bins", 0))


def _context(n_gpus):
    n_gpus = int(n_gpus)
    if n_gpus <= 1:
        return engine.Context(0)
    return engine.Context(devices=list(range(n_gpus)))


def _write_records(path, rec, first, sc):
    with open(path, "w", newline="") as fh:
        results._header(fh, sc, kind="records", first_sim=int(first), n_sims=int(len(rec)))
        w = csv.writer(fh)
        w.writerow(["sim_index", "phi", "failed", "ocp_solves", "ocp_failures"])
        for i, r in enumerate(rec):
            phi = float(r["phi"])
            w.writerow([first + i, "nan" if math.isnan(phi) else repr(phi), int(r["failed"]), int(r["ocp_solves"]),
                        int(r["ocp_failures"])])


def _read_records(path):
    with open(path, newline="") as fh:
        meta = results._read_header(fh)
        rows = list(csv.reader(fh))[1:]
    phi = np.array([float(r[1]) for r in rows])
    return phi, meta


def cmd_simulate(cfg, args, sc):
    """One closed loop (sim index run.first): trajectory CSV + summary JSON."""
    _, first, _, _, _ = _run_cfg(cfg, args)
    sc.record_trajectories = 1
    sc.record_stride = int(cfg.get("run", {}).get("stride", 1))
    ctx = engine.Context(0)
    t = time.perf_counter()
    rec, traj = ctx.run_traj(sc, first, 1)
    wall = time.perf_counter() - t
    results.write_trajectory_csv(os.path.join(args.out, "trajectory.csv"), traj[0], first, sc)
    r = rec[0]
    doc = {"format": "nmpcmc-simulation", "version": results.FORMAT_VERSION, "sim_index": first,
           "phi": results._plain(float(r["phi"])), "failed": bool(r["failed"]), "ocp_solves": int(r["ocp_solves"]),
           "ocp_failures": int(r["ocp_failures"]), "status": int(r["status"]), "wall_seconds": wall,
           "seeds": {"base_seed": int(sc.base_seed)}, "scenario": results.scenario_to_dict(sc)}
    with open(os.path.join(args.out, "summary.json"), "w") as fh:
        json.dump(doc, fh, indent=1, allow_nan=False)
    return doc


def cmd_montecarlo(cfg, args, sc):
    """run_monte_carlo over run.sims samples on `workers` GPUs: aggregate
    JSON + histogram CSV + records CSV (+ trajectories of the first k)."""
    sims, first, workers, n_traj, bins = _run_cfg(cfg, args)
    ctx = _context(workers)
    t = time.perf_counter()
    rec, _, agg = ctx.run(sc, first, sims, aggregate=True)
    wall = time.perf_counter() - t
    res = engine.McResult(rec, agg, wall, None, first)
    doc = results.write_aggregate_json(os.path.join(args.out, "aggregate.json"), sc, res,
                                       extra={"gpus": ctx.num_devices})
    results.write_histogram_csv(os.path.join(args.out, "histogram.csv"), engine.phi_histogram(rec["phi"], bins), sc)
    _write_records(os.path.join(args.out, "records.csv"), rec, first, sc)
    if n_traj > 0:
        sct = abi.Scenario.from_buffer_copy(bytes(sc))
        sct.record_trajectories = 1
        _, traj = engine.Context(0).run_traj(sct, first, n_traj)
        for i in range(n_traj):
            results.write_trajectory_csv(os.path.join(args.out, f"trajectory_{first + i}.csv"), traj[i], first + i,
                                         sct)
    return doc


def cmd_benchmark(cfg, args, sc):
    """scaling_benchmark (montecarlo.cpp:253-266) over GPU counts: speedup CSV
    (workers, seconds, speedup = T(1) / T(w)); T(1) from the first entry equal
    to one, else from an extra one-GPU run, as the reference does. Counts
    above the visible GPUs are skipped and noted; records must be identical
    at every count."""
    sims, first, workers, _, _ = _run_cfg(cfg, args)
    counts = [int(w) for w in workers.split(",")]
    ngpu = engine.device_count()

    def timed(w):
        ctx = _context(w)
        ctx.run(sc, first, min(sims, 64))  # warm-up (module load, workspaces)
        t = time.perf_counter()
        rec, _ = ctx.run(sc, first, sims)
        return time.perf_counter() - t, rec

    t1, ref = timed(1) if 1 not in counts else (None, None)
    rows = []
    for w in counts:
        if w > ngpu:
            rows.append((w, float("nan"), float("nan"), f"skipped: {ngpu} GPU(s) visible"))
            continue
        s, rec = timed(w)
        if ref is None:
            ref = rec
        elif rec.tobytes() != ref.tobytes():
            raise RuntimeError(f"records differ at {w} GPUs")
        if t1 is None and w == 1:
            t1 = s
        rows.append((w, s, t1 / s, "records identical"))
    with open(os.path.join(args.out, "speedup.csv"), "w", newline="") as fh:
        results._header(fh, sc, kind="scaling_benchmark", n_sims=sims)
        wr = csv.writer(fh)
        wr.writerow(["workers", "seconds", "speedup", "note"])
        for w, s, sp, note in rows:
            wr.writerow([w, repr(s), repr(sp), note])
    return {"rows": rows}


def cmd_histogram(cfg, args, sc):
    """Re-bin an existing records file (bins <= 0: Freedman-Diaconis)."""
    src = args.inp or os.path.join(args.out, "records.csv")
    phi, meta = _read_records(src)
    bins = args.bins if args.bins is not None else _run_cfg(cfg, args)[4]
    h = engine.phi_histogram(phi, bins)
    sc2 = results.scenario_from_dict(meta["scenario"]) if "scenario" in meta else sc
    results.write_histogram_csv(os.path.join(args.out, "histogram.csv"), h, sc2)
    return {"bins": int(len(h.counts)), "source": src}


COMMANDS = {"simulate": cmd_simulate, "montecarlo": cmd_montecarlo, "benchmark": cmd_benchmark,
            "histogram": cmd_histogram}


def main(argv=None):
    ap = argparse.ArgumentParser(prog="nmpcmc", description=__doc__.split("\n\n")[0])
    ap.add_argument("command", choices=sorted(COMMANDS))
    ap.add_argument("--config")
    ap.add_argument("--set", action="append", default=[], metavar="SECTION.KEY=VALUE")
    ap.add_argument("--out", default=".")
    ap.add_argument("--workers", help="GPU count (benchmark: comma list)")
    ap.add_argument("--sims", type=int)
    ap.add_argument("--seed", type=int)
    ap.add_argument("--bins", type=int)
    ap.add_argument("--in", dest="inp", help="histogram: records.csv to re-bin")
    args = ap.parse_args(argv)
    os.makedirs(args.out, exist_ok=True)
    try:
        overrides = list(args.set) + ([f"scenario.seed={args.seed}"] if args.seed is not None else [])
        cfg = load_config(args.config, overrides)
        sc = build_scenario(cfg)
        out = COMMANDS[args.command](cfg, args, sc)
        print(json.dumps({"command": args.command, "out": args.out, "ok": True,
                          **({"phi": out.get("phi")} if isinstance(out, dict) and "phi" in out else {})}))
        return 0
    except Exception as e:  # noqa: BLE001 -- the CLI reports every failure as a record
        err = {"command": args.command, "ok": False, "error": type(e).__name__,
               "kind": getattr(e, "kind", type(e).__name__), "message": str(e)}
        with open(os.path.join(args.out, "error.json"), "w") as fh:
            json.dump(err, fh)
        print(json.dumps(err), file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
