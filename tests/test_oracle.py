"""The oracle itself, pinned before it is trusted (task §③):
 - the reference build reproduces the reference's own known-answer tests
   (Philox KATs test_rng.cpp:13-38, frozen rate test_cstr.cpp:26-32,
   PI seven-equation law test_controllers.cpp:94-145, RNG golden values of
   SURVEY.md §8c);
 - the committed golden fixtures were produced by this build;
 - the two libm link variants agree where the survey says they must
   (PI closed loop within 1e-9)."""
import ctypes as C
import math

import numpy as np
import pytest

from conftest import assert_records_equal, load_golden
from oracle import lib as O
from paper_2212_02197_b200 import abi, configs

needs_ref = pytest.mark.skipif(not O.ref_available() and not __import__("os").path.isdir("/root/reference"),
                               reason="oracle/_ref not built and /root/reference absent")

KATS = [
    ((0, 0, 0, 0, 0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 6, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@needs_ref
@pytest.mark.parametrize("libm", ["glibc", "xlibm"])
def test_ref_philox_kats(libm):
    L = O.ref(libm)
    for inp, want in KATS:
        a = (C.c_uint32 * 6)(*inp)
        out = (C.c_uint32 * 4)()
        L.nmpcmc_ref_philox_block(a, out)
        assert tuple(out) == want


@needs_ref
def test_ref_normals_survey_values():
    # CounterRng(12345, 7).normal() x 4 (glibc build)
    L = O.ref("glibc")
    v = np.zeros(4)
    L.nmpcmc_ref_normals(12345, 7, 4, v.ctypes.data_as(C.POINTER(C.c_double)))
    assert v.tolist() == [-1.7944990614004552, 1.1959385384939205, 1.3008388521805516, -0.55292810623727406]


@needs_ref
def test_ref_frozen_rate_and_k0():
    configs.check_k0()
    L = O.ref("glibc")
    p = abi.CstrParams(**configs.study_params())
    c = (C.c_double * 3)(0.5, 0.5, 300.0)
    assert L.nmpcmc_ref_reaction_rate(C.byref(p), c) == pytest.approx(0.005978248215701345, rel=1e-13)
    c = (C.c_double * 3)(0.5, 0.5, 0.0)
    assert math.isnan(L.nmpcmc_ref_reaction_rate(C.byref(p), c))  # DomainError


@needs_ref
def test_ref_pi_step_law():
    L = O.ref("glibc")
    st = (C.c_double * 8)(-1e-3, -1e-4, -1e-1, 1.0, 400.0, 0.0, 1000.0, 0.0)
    out = (C.c_double * 7)()
    L.nmpcmc_ref_pi_step(st, C.c_double(300.0), C.c_double(310.0), out)
    e = 310.0 - 300.0
    P = -1e-3 * e
    I = 0.0 + 1.0 * -1e-4 * e
    u_hat = 400.0 + P + I
    assert list(out) == [e, P, I, u_hat, u_hat, 0.0, I]


@needs_ref
@pytest.mark.parametrize("name", ["pi_cfg0", "pi_cfg1", "pi_onestate", "pi_quiet"])
def test_golden_pi_reproduced_by_ref(name):
    d, kw, sc = load_golden(name)
    for libm in ("xlibm", "glibc"):
        rec, _ = O.run_batch(O.ref(libm), sc, int(d["first"]), len(d[f"rec_{libm}"]))
        assert_records_equal(rec, d[f"rec_{libm}"])


@pytest.mark.parametrize("name,frac", [("pi_cfg0", 1.0), ("pi_cfg1", 0.95), ("pi_onestate", 1.0),
                                        ("pi_quiet", 1.0)])
def test_golden_pi_libm_variants_agree(name, frac):
    """Exact-libm vs glibc reference: PI cost within 1e-9.
    With per-sample parameters (config 1) a few samples sit in an oscillatory
    regime (phi ~ 1e2..1e4) where 1-ulp libm differences grow; those are why
    parity is pinned in exact-libm mode."""
    d, _, _ = load_golden(name)
    x, g = d["rec_xlibm"], d["rec_glibc"]
    np.testing.assert_array_equal(x["failed"], g["failed"])
    ok = x["failed"] == 0
    rel = np.abs(x["phi"][ok] - g["phi"][ok]) / np.abs(g["phi"][ok])
    assert np.mean(rel <= 1e-9) >= frac


def test_golden_rng_fixture_kats():
    d = np.load(__import__("conftest").GOLDEN + "/rng.npz")
    # first normals of (12345, 7) in the glibc build are the survey's values
    assert d["normals_glibc_0"][:4].tolist() == [-1.7944990614004552, 1.1959385384939205,
                                                 1.3008388521805516, -0.55292810623727406]
    # the libm variants differ in at most a few ulp, and rarely
    for i in range(4):
        a, b = d[f"normals_xlibm_{i}"], d[f"normals_glibc_{i}"]
        assert np.mean(a != b) < 0.05
        np.testing.assert_allclose(a, b, rtol=1e-14, atol=1e-300)
