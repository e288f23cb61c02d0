"""The finite-difference fixtures (make_golden.py fd) are the reference run
on a controller Model without analytic jacobians (model.cpp:54-124). CPU."""
import numpy as np
import pytest

from conftest import assert_records_equal, load_golden
from oracle import lib as O


@pytest.mark.skipif(not O.ref_available(), reason="reference build not present")
@pytest.mark.parametrize("name", ["nmpc_fd_n30", "nmpc3_fd_n20"])
def test_fd_fixture_is_the_reference(name):
    d, _, sc = load_golden(name)
    L = O.ref("xlibm")
    L.nmpcmc_ref_set_ctrl_fd(1)
    try:
        rec, _ = O.run_batch(L, sc, int(d["first"]), len(d["rec_xlibm"]))
    finally:
        L.nmpcmc_ref_set_ctrl_fd(0)
    assert_records_equal(rec, d["rec_xlibm"])
    ana, _ = O.run_batch(L, sc, int(d["first"]), len(d["rec_xlibm"]))
    assert not np.array_equal(ana["phi"], d["rec_xlibm"]["phi"])
