"""Result files (paper_2212_02197_b200/results.py; SPEC.md montecarlo
"External Interfaces"): stable keys/columns, config echo, bit-exact reload.
CPU only: records come from the committed golden fixtures."""
import numpy as np

from conftest import load_golden
from paper_2212_02197_b200 import abi, configs, engine, results


def _mc(name):
    d, kw, sc = load_golden(name)
    rec = d["rec_xlibm"]
    return sc, kw, d, engine.McResult(rec, engine.aggregate_stats(rec), 1.25, None, int(d["first"]))


def test_scenario_echo_round_trips_bytes():
    for kw in (dict(controller="pi", perturb=True), dict(controller="nmpc", N=30, ctrl_variant=abi.THREE_STATE)):
        sc = configs.make_scenario(**kw)
        back = results.scenario_from_dict(results.scenario_to_dict(sc))
        assert bytes(back) == bytes(sc)


def test_aggregate_json(tmp_path):
    sc, _, d, mc = _mc("pi_cfg1")
    p = tmp_path / "agg.json"
    results.write_aggregate_json(str(p), sc, mc, extra={"note": "test"})
    doc = results.read_aggregate_json(str(p))
    assert doc["format"] == "nmpcmc-aggregate" and doc["version"] == 1
    assert set(doc) == {"format", "version", "aggregate", "first_sim", "n_sims", "wall_seconds", "seeds",
                        "scenario", "extra"}
    assert set(doc["aggregate"]) == set(mc.aggregate)
    assert doc["aggregate"]["mean"] == mc.aggregate["mean"]  # shortest repr round-trips exactly
    assert doc["aggregate"]["deciles"] == [float(x) for x in mc.aggregate["deciles"]]
    assert doc["seeds"]["base_seed"] == sc.base_seed
    assert doc["n_sims"] == len(d["rec_xlibm"])
    assert bytes(results.scenario_from_dict(doc["scenario"])) == bytes(sc)


def test_histogram_csv(tmp_path):
    sc, _, d, _ = _mc("pi_cfg0")
    h = engine.phi_histogram(d["rec_xlibm"]["phi"])
    p = tmp_path / "hist.csv"
    results.write_histogram_csv(str(p), h, sc)
    back, meta = results.read_histogram_csv(str(p))
    np.testing.assert_array_equal(back.edges, h.edges)
    np.testing.assert_array_equal(back.counts, h.counts)
    assert meta["kind"] == "phi_histogram" and meta["base_seed"] == sc.base_seed
    assert open(p).read().splitlines()[1] == "bin_lo,bin_hi,count"


def test_trajectory_csv(tmp_path):
    _, kw, d, _ = _mc("nmpc_n30_short")
    sct = configs.make_scenario(**kw, record=True)
    tr = d["traj_xlibm"][0]
    p = tmp_path / "traj.csv"
    results.write_trajectory_csv(str(p), tr, 0, sct)
    back, meta = results.read_trajectory_csv(str(p))
    want = tr[~np.isnan(tr[:, 0])]
    np.testing.assert_array_equal(back, want)
    assert meta["rows"] == len(want) and meta["sim_index"] == 0
    assert open(p).read().splitlines()[1] == "t,z,zbar,u,y"


def test_unbounded_inputs_round_trip():
    """Non-finite scenario fields (unbounded inputs) survive the JSON echo
    bit for bit (they used to come back as NaN)."""
    sc = configs.make_scenario("nmpc", N=30)
    sc.u_min, sc.u_max = float("-inf"), float("inf")
    sc.ctrl.u_max = float("inf")
    import json
    d = json.loads(json.dumps(results.scenario_to_dict(sc), allow_nan=False))
    back = results.scenario_from_dict(d)
    assert bytes(back) == bytes(sc)
    assert back.u_min == float("-inf") and back.u_max == float("inf")
