"""The oracle's C++ restatement (oracle/port/nmpcmc_port.cpp) against the
compiled reference: bitwise on the golden fixtures in both libm modes,
three-state controller model included (the device runs it on K3g)."""
import os

import numpy as np
import pytest

from conftest import assert_records_equal, load_golden
from oracle import lib as O
from paper_2212_02197_b200 import abi, configs

CASES = [("pi_cfg0", 256), ("pi_cfg1", 256), ("pi_onestate", 64), ("pi_quiet", 16),
         ("nmpc_n30_short", 8), ("nmpc_n120_short", 2), ("nmpc3_n30_short", 8), ("nmpc3_n60_pert_short", 4)]


@pytest.mark.parametrize("libm", ["xlibm", "glibc"])
@pytest.mark.parametrize("name,n", CASES)
def test_port_reproduces_reference_golden(name, n, libm):
    d, _, sc = load_golden(name)
    want = d[f"rec_{libm}"][:n]
    got, _ = O.run_batch(O.port(libm), sc, int(d["first"]), n, os.cpu_count(), prefix=O.port_prefix(libm))
    assert_records_equal(got, want)


def test_port_trajectories_match_reference():
    d, kw, _ = load_golden("nmpc_n30_short")
    sct = configs.make_scenario(**kw, record=True)
    want = d["traj_xlibm"][0]
    rec, traj = O.run_traj(O.port("xlibm"), sct, 0, want.shape[0], prefix=O.port_prefix("xlibm"))
    np.testing.assert_array_equal(traj, want)


@pytest.mark.skipif(not O.ref_available() and not os.path.isdir("/root/reference"), reason="no reference build")
def test_port_three_state_controller_matches_reference():
    sc = configs.make_scenario("nmpc", N=10, n_steps=6, ctrl_variant=abi.THREE_STATE)
    ref, _ = O.run_batch(O.ref("xlibm"), sc, 0, 4, 4)
    got, _ = O.run_batch(O.port("xlibm"), sc, 0, 4, 4, prefix=O.port_prefix("xlibm"))
    assert_records_equal(got, ref)
