"""Device building blocks vs the oracle, bitwise: Philox4x32-10 (rng.cpp:31-43)
incl. the reference KATs, the Box-Muller normal stream (rng.cpp:78-91), and the
device libm vs its host build."""
import numpy as np
import pytest

from conftest import GOLDEN
from oracle import lib as O

pytestmark = pytest.mark.gpu

KATS = [
    ((0, 0, 0, 0, 0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 6, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_philox_kats(gpu_ctx):
    out = gpu_ctx.philox_blocks(np.array([k[0] for k in KATS], dtype=np.uint32))
    assert [tuple(int(v) for v in r) for r in out] == [k[1] for k in KATS]


def test_philox_random_blocks(gpu_ctx):
    d = np.load(f"{GOLDEN}/rng.npz")
    np.testing.assert_array_equal(gpu_ctx.philox_blocks(d["philox_in"]), d["philox_out"])


def test_normal_stream_bitwise_exact_libm(gpu_ctx):
    d = np.load(f"{GOLDEN}/rng.npz")
    for i, (seed, stream) in enumerate(d["streams"]):
        got = gpu_ctx.normals(int(seed), int(stream), 257)
        np.testing.assert_array_equal(got, d[f"normals_xlibm_{i}"])
        # against the glibc reference: same stream within libm rounding
        np.testing.assert_allclose(got, d[f"normals_glibc_{i}"], rtol=1e-14, atol=1e-300)


@pytest.mark.parametrize("fn,lo,hi", [("exp", -40.0, 0.0), ("exp", -700.0, 700.0), ("log", 1e-300, 1.0),
                                      ("log", 1e-3, 1e3), ("sin", 0.0, 6.3), ("cos", 0.0, 6.3),
                                      ("sin", -2e4, 2e4)])
def test_device_libm_equals_host_build(gpu_ctx, fn, lo, hi):
    x = np.random.default_rng(5).uniform(lo, hi, 20000)
    L = O.xlibm()
    f = getattr(L, f"nmx_{fn}")
    want = np.array([f(float(v)) for v in x])
    np.testing.assert_array_equal(gpu_ctx.libm(fn, x), want)


def test_device_libm_special_values(gpu_ctx):
    x = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1e-310, 709.78, -745.0, -746.0])
    L = O.xlibm()
    for fn in ("exp", "log", "sin", "cos"):
        f = getattr(L, f"nmx_{fn}")
        got = gpu_ctx.libm(fn, x)
        want = np.array([f(float(v)) for v in x])
        np.testing.assert_array_equal(got, want)
