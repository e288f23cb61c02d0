"""C-ABI library: loads without a GPU, exports every symbol include/*.h
declares, struct layouts match the ctypes mirror, and the host-side entry
points (validate, aggregate, histogram) equal the reference's."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden
from oracle import lib as O
from paper_2212_02197_b200 import abi, configs, engine


def _declared_symbols():
    txt = open(os.path.join(ROOT, "include", "nmpcmc_gpu.h")).read()
    return sorted(set(re.findall(r"\b(nmpcmc_gpu_[a-z_0-9]+)\s*\(", txt)))


def test_library_loads_and_exports_all_symbols():
    lib = engine.library()
    syms = _declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.nmpcmc_gpu_abi_version() == 1


def test_no_device_is_an_error_not_a_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(engine.CudaError):
        engine.Context(0)


def test_validate_matches_reference_rules():
    sc = configs.make_scenario("pi")
    assert engine.validate_scenario(sc) == 720
    bad = configs.make_scenario("pi")
    bad.tf = 7205.0  # not a multiple of Ts
    with pytest.raises(engine.DomainError):
        engine.validate_scenario(bad)
    bad = configs.make_scenario("pi")
    bad.sp_times[0] = 10.0  # profile starts after t0
    with pytest.raises(engine.DomainError):
        engine.validate_scenario(bad)
    bad = configs.make_scenario("nmpc")
    bad.horizon_Ts = 5.0
    with pytest.raises(engine.DomainError):
        engine.validate_scenario(bad)
    three = configs.make_scenario("nmpc", ctrl_variant=abi.THREE_STATE)
    assert engine.validate_scenario(three) == 720  # runs on K3g
    bad = configs.make_scenario("nmpc", ctrl_variant=abi.THREE_STATE)
    bad.ctrl_variant = 7
    with pytest.raises(engine.DomainError):
        engine.validate_scenario(bad)
    big = configs.make_scenario("nmpc", N=5000)
    with pytest.raises(engine.Unsupported):
        engine.validate_scenario(big)
    neg = configs.make_scenario("pi", noise_R=-1.0)
    with pytest.raises(engine.NotPositiveDefinite):
        engine.validate_scenario(neg)


@pytest.mark.parametrize("name", ["pi_cfg0", "pi_cfg1"])
def test_aggregate_and_histogram_equal_reference(name):
    d, _, _ = load_golden(name)
    rec = d["rec_xlibm"]
    got = engine.aggregate_stats(rec)
    L = O.ref("xlibm")
    want = abi.Aggregate()
    r = np.ascontiguousarray(rec)
    L.nmpcmc_ref_aggregate(r.ctypes.data_as(C.POINTER(abi.SimRecord)), len(r), C.byref(want))
    assert got == abi.aggregate_to_dict(want)
    h = engine.phi_histogram(rec["phi"])
    edges = np.zeros(201)
    counts = np.zeros(200, dtype=np.int32)
    nb = C.c_int(0)
    phi = np.ascontiguousarray(rec["phi"])
    L.nmpcmc_ref_histogram(phi.ctypes.data_as(C.POINTER(C.c_double)), len(phi), 0,
                           edges.ctypes.data_as(C.POINTER(C.c_double)),
                           counts.ctypes.data_as(C.POINTER(C.c_int)), C.byref(nb))
    np.testing.assert_array_equal(h.edges, edges[: nb.value + 1])
    np.testing.assert_array_equal(h.counts, counts[: nb.value])


def test_aggregate_edge_cases():
    empty_ok = np.zeros(3, dtype=abi.RECORD_DTYPE)
    empty_ok["failed"] = 1
    empty_ok["phi"] = np.nan
    a = engine.aggregate_stats(empty_ok)
    assert a["n_failed"] == 3 and np.isnan(a["mean"]) and a["ocp_success_pct"] == 100.0
    one = np.zeros(1, dtype=abi.RECORD_DTYPE)
    one["phi"] = 2.5
    a = engine.aggregate_stats(one)
    assert a["mean"] == 2.5 and a["variance"] == 0.0 and a["deciles"] == [2.5] * 11
    h = engine.phi_histogram([np.nan, np.inf])
    assert h.edges.tolist() == [0.0, 1.0] and h.counts.tolist() == [0]
    h = engine.phi_histogram([3.0, 3.0])
    assert h.edges.tolist() == [3.0, 4.0] and h.counts.tolist() == [2]
