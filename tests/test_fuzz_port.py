"""The oracle's C++ restatement (oracle/port) against the reference on
randomised scenarios (tests/golden/fuzz.npz: 200 short ones; fuzz_long.npz:
60 longer NMPC runs; make_fuzz.py): bitwise records in both libm modes. CPU
only."""
import os

import numpy as np
import pytest

from conftest import assert_records_equal
from oracle import lib as O
from paper_2212_02197_b200 import abi

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FUZZ_FILES = ["fuzz.npz", "fuzz_long.npz"]


def fuzz_cases(name="fuzz.npz"):
    d = np.load(os.path.join(GOLDEN, name))
    return [(abi.Scenario.from_buffer_copy(d["scenarios"][i].tobytes()), int(d["first"][i]),
             d["rec_xlibm"][i], d["rec_glibc"][i]) for i in range(len(d["first"]))]


@pytest.mark.parametrize("fname", FUZZ_FILES)
@pytest.mark.parametrize("libm", ["xlibm", "glibc"])
def test_port_matches_reference_on_random_scenarios(libm, fname):
    L = O.port(libm)
    for i, (sc, first, rx, rg) in enumerate(fuzz_cases(fname)):
        got, _ = O.run_batch(L, sc, first, len(rx), os.cpu_count(), prefix=O.port_prefix(libm))
        assert_records_equal(got, rx if libm == "xlibm" else rg)
