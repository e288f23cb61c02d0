"""The roofline's per-unit flop constants (paper_2212_02197_b200/workmodel.py)
are measured: re-run the op-counting build of the port (oracle/port/
flopcount.cpp) on a short config-3 run and require agreement."""
import json
import os
import subprocess

import pytest

from paper_2212_02197_b200 import workmodel

ORACLE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle")


def test_workmodel_constants_match_op_count():
    exe = os.path.join(ORACLE, "_build", "flopcount")
    r = subprocess.run(["make", "-C", ORACLE, "flops"], capture_output=True, text=True)
    if r.returncode != 0 or not os.path.exists(exe):
        pytest.skip("flopcount build unavailable: " + r.stderr[-300:])
    out = subprocess.run([exe, "1", "12"], capture_output=True, text=True, timeout=600, check=True).stdout
    d = json.loads(out)
    E = workmodel.EXP
    for nx in (1, 3):
        got = d[f"nx{nx}_N60"]
        m = workmodel._MEASURED[nx]
        # per-interval/per-step constants are exact functions of the formulas
        assert got["shoot_full"] - 20 * E == m["shoot_full"]
        assert got["shoot_fonly"] == m["shoot_fonly"]
        assert got["ekf_step"] - 20 * E == m["ekf_step"]
        assert got["plant_step"] == m["plant_step"]
        # per-stage IPM / SQP figures depend mildly on the iterates
        assert abs(got["ipm_stage"] / m["ipm_stage"] - 1) < 0.03
        assert abs(got["sqp_stage"] / m["sqp_stage"] - 1) < 0.08
