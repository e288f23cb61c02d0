import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2212_02197_b200 import engine
    return engine.Context(0)


def load_golden(name):
    import json

    import numpy as np

    from paper_2212_02197_b200 import configs
    d = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    kwargs = json.loads(str(d["kwargs"]))
    sc = configs.make_scenario(**kwargs)
    assert bytes(sc) == d["scenario"].tobytes(), f"{name}: scenario factory drifted from the fixture"
    return d, kwargs, sc


def assert_records_equal(got, want, fields=("phi", "failed", "ocp_solves", "ocp_failures")):
    """Bitwise equality of per-sample records (NaN phi of failed runs equal)."""
    import numpy as np
    for f in fields:
        np.testing.assert_array_equal(got[f], want[f], err_msg=f"field {f}")
