"""Result files of a Monte Carlo run (SPEC.md, montecarlo "External
Interfaces": aggregate JSON with statistics + config echo + seeds, CSV
histogram with bin edges and counts, optional per-run CSV trajectories with
columns t, z, zbar, u, y).

The reference specifies these formats but ships no writer (its CLI is a stub,
tools/src/main.cpp:3-6). The keys and columns here are stable, and every file
embeds the effective scenario and base seed, so any result can be re-derived
from its own header (SPEC.md cli "Invariants & Properties"). Floats are written
with Python's shortest round-trip repr, so files reload bit for bit. NaN and
infinities become the strings "nan", "inf", "-inf".
"""
import csv
import ctypes as C
import json
import math
from typing import Optional

import numpy as np

from . import abi
from .engine import Histogram, McResult

FORMAT_VERSION = 1


def _plain(x):
    """Non-finite floats become the strings "inf", "-inf", "nan" (JSON has
    no literal for them), so unbounded inputs round-trip bit for bit."""
    if isinstance(x, float) and not math.isfinite(x):
        return "nan" if math.isnan(x) else ("inf" if x > 0 else "-inf")
    return x


def _num(v):
    """Inverse of _plain (None from version-1 files reads as NaN)."""
    if v is None:
        return float("nan")
    if isinstance(v, str):
        return float(v)
    return v


def _struct_to_dict(s) -> dict:
    out = {}
    for name, typ in s._fields_:
        if name.startswith("_"):
            continue
        v = getattr(s, name)
        if isinstance(v, C.Structure):
            out[name] = _struct_to_dict(v)
        elif isinstance(v, C.Array):
            out[name] = [_plain(float(e)) for e in v]
        else:
            out[name] = _plain(v)
    return out


def scenario_to_dict(sc: abi.Scenario) -> dict:
    """The effective scenario, every field; arrays trimmed to their used
    length (setpoints to n_setpoints, states to the model dimensions)."""
    d = _struct_to_dict(sc)
    ns = sc.n_setpoints
    d["sp_times"], d["sp_values"] = d["sp_times"][:ns], d["sp_values"][:ns]
    nxt = 3 if sc.truth_variant == abi.THREE_STATE else 1
    nxc = 3 if sc.ctrl_variant == abi.THREE_STATE else 1
    d["x0"] = d["x0"][:nxt]
    d["x0_hat"] = d["x0_hat"][:nxc]
    d["P0"] = d["P0"][: nxc * nxc]
    return d


def _fill(s, d: dict):
    for name, typ in s._fields_:
        if name not in d:
            continue
        v = d[name]
        cur = getattr(s, name)
        if isinstance(cur, C.Structure):
            _fill(cur, v)
        elif isinstance(cur, C.Array):
            for i, e in enumerate(v):
                cur[i] = _num(e)
        else:
            setattr(s, name, _num(v))


def scenario_from_dict(d: dict) -> abi.Scenario:
    sc = abi.Scenario()
    _fill(sc, d)
    return sc


def write_aggregate_json(path: str, sc: abi.Scenario, result: McResult, extra: Optional[dict] = None) -> dict:
    """Aggregate JSON: McAggregate (montecarlo.hpp:95-106) + the sample range,
    the wall clock of the batch, the effective scenario and its seeds."""
    agg = {k: (_plain(float(v)) if isinstance(v, float) else v) for k, v in result.aggregate.items()}
    if "deciles" in agg:
        agg["deciles"] = [_plain(float(x)) for x in result.aggregate["deciles"]]
    doc = {
        "format": "nmpcmc-aggregate",
        "version": FORMAT_VERSION,
        "aggregate": agg,
        "first_sim": int(result.first_sim),
        "n_sims": int(len(result.records)),
        "wall_seconds": float(result.wall_seconds),
        "seeds": {"base_seed": int(sc.base_seed), "noise_stream": "sim_index",
                  "parameter_stream": "sim_index | 2^63" if sc.perturb else None},
        "scenario": scenario_to_dict(sc),
    }
    if extra:
        doc["extra"] = extra
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1, allow_nan=False)
    return doc


def read_aggregate_json(path: str) -> dict:
    with open(path) as fh:
        doc = json.load(fh)
    if doc.get("format") != "nmpcmc-aggregate":
        raise ValueError(f"{path}: not an aggregate file")
    return doc


def _header(fh, sc: Optional[abi.Scenario], **kw):
    meta = {"version": FORMAT_VERSION, **kw}
    if sc is not None:
        meta["base_seed"] = int(sc.base_seed)
        meta["scenario"] = scenario_to_dict(sc)
    fh.write("# " + json.dumps(meta, allow_nan=False) + "\n")


def _read_header(fh) -> dict:
    line = fh.readline()
    if not line.startswith("# "):
        raise ValueError("missing metadata header")
    return json.loads(line[2:])


def write_histogram_csv(path: str, hist: Histogram, sc: Optional[abi.Scenario] = None):
    """Histogram CSV: one row per bin (bin_lo, bin_hi, count), after a '#'
    metadata line with the scenario echo (phi_histogram, montecarlo.cpp:268-304)."""
    with open(path, "w", newline="") as fh:
        _header(fh, sc, kind="phi_histogram", bins=int(len(hist.counts)))
        w = csv.writer(fh)
        w.writerow(["bin_lo", "bin_hi", "count"])
        for i, c in enumerate(hist.counts):
            w.writerow([repr(float(hist.edges[i])), repr(float(hist.edges[i + 1])), int(c)])


def read_histogram_csv(path: str):
    with open(path, newline="") as fh:
        meta = _read_header(fh)
        rows = list(csv.reader(fh))
    body = rows[1:]
    edges = np.array([float(r[0]) for r in body] + ([float(body[-1][1])] if body else []))
    counts = np.array([int(r[2]) for r in body], dtype=np.int32)
    return Histogram(edges, counts), meta


def write_trajectory_csv(path: str, traj: np.ndarray, sim_index: int, sc: Optional[abi.Scenario] = None):
    """Per-run trajectory CSV (columns t, z, zbar, u, y; Trajectory,
    montecarlo.hpp:64-67). Unused trailing rows (NaN time) are dropped; the
    final row has no u, y (written empty)."""
    tr = np.asarray(traj, dtype=np.float64)
    tr = tr[~np.isnan(tr[:, 0])]
    with open(path, "w", newline="") as fh:
        _header(fh, sc, kind="trajectory", sim_index=int(sim_index), rows=int(len(tr)))
        w = csv.writer(fh)
        w.writerow(["t", "z", "zbar", "u", "y"])
        for r in tr:
            w.writerow(["" if math.isnan(v) else repr(float(v)) for v in r])


def read_trajectory_csv(path: str):
    with open(path, newline="") as fh:
        meta = _read_header(fh)
        rows = list(csv.reader(fh))
    body = np.array([[float("nan") if v == "" else float(v) for v in r] for r in rows[1:]], dtype=np.float64)
    return body.reshape(-1, 5), meta
