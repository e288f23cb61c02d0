"""CLI (SPEC.md cli module): load_config + --set overrides, validation errors
naming the invariant, and the four workflows on the GPU with their result
files (simulate: trajectory CSV + summary JSON; montecarlo: aggregate JSON +
histogram CSV + records CSV; benchmark: speedup CSV; histogram: re-bin)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_2212_02197_b200 import cli, configs, results

CFG = """
[controller]
type = nmpc      # BASELINE config 2 shape, shortened
N = 30
[scenario]
tf = 600
seed = 12345
[run]
sims = 64
"""


def test_load_config_defaults_and_overrides(tmp_path):
    p = tmp_path / "exp.ini"
    p.write_text(CFG)
    cfg = cli.load_config(str(p), ["controller.N=20", "run.sims=8"])
    sc = cli.build_scenario(cfg)
    assert sc.N == 20 and sc.tf == 600.0 and sc.controller == 0
    assert cfg["run"]["sims"] == "8"
    # minimal config: every default applied (configs.make_scenario = BASELINE config 0)
    d = cli.build_scenario(cli.load_config(None, []))
    ref = configs.make_scenario("pi")
    assert bytes(d) == bytes(ref)


def test_config_round_trips_through_the_result_echo(tmp_path):
    sc = cli.build_scenario(cli.load_config(None, ["controller.type=nmpc", "controller.N=60", "scenario.Ts=1",
                                                   "scenario.tf=600", "scenario.Ns=20", "controller.u_max=1000"]))
    back = results.scenario_from_dict(json.loads(json.dumps(results.scenario_to_dict(sc))))
    assert bytes(back) == bytes(sc)


@pytest.mark.parametrize("override,kind,needle", [
    ("scenario.tf=605", "ValidationError", "N_bar integrality"),
    ("bogus.key=1", "ParseError", "unknown section"),
    ("controller.nope=1", "ParseError", "unknown key controller.nope"),
    ("controller.type=lqr", "ValidationError", "pi or nmpc"),
])
def test_config_errors_name_the_problem(override, kind, needle):
    with pytest.raises(cli.ConfigError) as e:
        cli.build_scenario(cli.load_config(None, [override]))
    assert e.value.kind == kind and needle in str(e.value)


def test_parse_error_has_location(tmp_path):
    p = tmp_path / "bad.ini"
    p.write_text("[controller]\ntype = pi\nthis line is not key value\n")
    with pytest.raises(cli.ConfigError) as e:
        cli.load_config(str(p))
    assert e.value.kind == "ParseError" and "line  3" in str(e.value)


def test_cli_error_record_without_gpu_work(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_2212_02197_b200.cli", "montecarlo", "--set", "scenario.tf=605",
                        "--out", str(tmp_path)], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode != 0
    err = json.loads(r.stderr.strip().splitlines()[-1])
    assert err["ok"] is False and err["kind"] == "ValidationError"
    assert json.loads((tmp_path / "error.json").read_text())["kind"] == "ValidationError"


def _cli(tmp_path, *args):
    r = subprocess.run([sys.executable, "-m", "paper_2212_02197_b200.cli", *args, "--out", str(tmp_path)], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_cli_simulate_trajectory_reproduces_phi(tmp_path):
    # noise-free PI loop: the summary's phi is phi_metric (montecarlo.cpp:65-78)
    # of the written trajectory, and a second run writes identical files
    args = ["simulate", "--set", "model.sigmaT=0", "--set", "noise.R=0", "--set", "scenario.tf=1200"]
    _cli(tmp_path / "a", *args)
    _cli(tmp_path / "b", *args)
    doc = json.loads((tmp_path / "a" / "summary.json").read_text())
    traj, meta = results.read_trajectory_csv(str(tmp_path / "a" / "trajectory.csv"))
    assert meta["kind"] == "trajectory" and traj.shape == (121, 5)
    assert not doc["failed"]
    acc = 0.0
    for z, zbar in traj[:, 1:3]:
        acc += (z - zbar) * (z - zbar)
    assert acc / len(traj) == doc["phi"]
    assert (tmp_path / "a" / "trajectory.csv").read_bytes() == (tmp_path / "b" / "trajectory.csv").read_bytes()


@pytest.mark.gpu
def test_cli_montecarlo_and_histogram(tmp_path):
    p = tmp_path / "exp.ini"
    p.write_text(CFG)
    _cli(tmp_path, "montecarlo", "--config", str(p))
    agg = results.read_aggregate_json(str(tmp_path / "aggregate.json"))
    assert agg["n_sims"] == 64 and agg["seeds"]["base_seed"] == 12345
    hist, _ = results.read_histogram_csv(str(tmp_path / "histogram.csv"))
    assert hist.counts.sum() == 64 - agg["aggregate"]["n_failed"]
    # the records reproduce the aggregate through the engine's own aggregate_stats
    phi, meta = cli._read_records(str(tmp_path / "records.csv"))
    assert meta["n_sims"] == 64
    assert np.nanmean(phi) == pytest.approx(agg["aggregate"]["mean"], rel=1e-12)
    # re-bin into 10 bins
    out2 = tmp_path / "rebin"
    _cli(out2, "histogram", "--in", str(tmp_path / "records.csv"), "--bins", "10")
    h2, _ = results.read_histogram_csv(str(out2 / "histogram.csv"))
    assert len(h2.counts) == 10 and h2.counts.sum() == hist.counts.sum()


@pytest.mark.gpu
def test_cli_benchmark_speedup_csv(tmp_path):
    _cli(tmp_path, "benchmark", "--set", "controller.type=pi", "--workers", "1,2", "--sims", "2000")
    import csv
    with open(tmp_path / "speedup.csv") as fh:
        fh.readline()
        rows = list(csv.DictReader(fh))
    assert rows[0]["workers"] == "1" and float(rows[0]["speedup"]) == 1.0
    assert len(rows) == 2
