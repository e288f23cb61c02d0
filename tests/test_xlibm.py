"""Portable libm (paper_2212_02197_b200/csrc/xlibm.h), host build: accuracy vs
mpmath and agreement with glibc. The device build is checked bitwise against
this host build in test_gpu_units.py."""
import math

import numpy as np
import pytest

from oracle import lib as O

mp = pytest.importorskip("mpmath")
mp.mp.prec = 120


def _ulp_err(got, exact):
    e = float(exact)
    return float(abs(mp.mpf(got) - exact) / math.ulp(e)) if e != 0 else 0.0


CASES = [
    ("exp", mp.exp, lambda r: r.uniform(-32.0, -20.0, 1500)),   # Arrhenius range exp(-EaR/T)
    ("exp", mp.exp, lambda r: r.uniform(-700.0, 700.0, 1500)),
    ("log", mp.log, lambda r: r.uniform(0.0, 1.0, 1500)),        # Box-Muller u1
    ("log", mp.log, lambda r: 1.0 - r.uniform(0.0, 1e-3, 800)),
    ("log", mp.log, lambda r: np.exp(r.uniform(-700.0, 700.0, 800))),
    ("sin", mp.sin, lambda r: r.uniform(0.0, 2 * np.pi, 1500)),  # Box-Muller angle
    ("cos", mp.cos, lambda r: r.uniform(0.0, 2 * np.pi, 1500)),
]


@pytest.mark.parametrize("name,ref,gen", CASES)
def test_xlibm_accuracy(name, ref, gen):
    L = O.xlibm()
    f = getattr(L, f"nmx_{name}")
    xs = gen(np.random.default_rng(11))
    errs = np.array([_ulp_err(f(float(x)), ref(mp.mpf(float(x)))) for x in xs])
    assert errs.max() < 0.6, errs.max()
    assert np.mean(errs > 0.5) < 0.005
    glibc = getattr(math, name)
    agree = np.mean([f(float(x)) == glibc(float(x)) for x in xs])
    assert agree > 0.99


def test_xlibm_special_values():
    L = O.xlibm()
    assert L.nmx_exp(0.0) == 1.0 and L.nmx_log(1.0) == 0.0
    assert L.nmx_exp(-1000.0) == 0.0 and math.isinf(L.nmx_exp(1000.0))
    assert math.isinf(L.nmx_log(0.0)) and L.nmx_log(0.0) < 0
    assert math.isnan(L.nmx_log(-1.0)) and math.isnan(L.nmx_exp(float("nan")))
    assert L.nmx_sin(0.0) == 0.0 and L.nmx_cos(0.0) == 1.0
    assert math.isnan(L.nmx_sin(float("inf")))
    # subnormal in and out
    assert L.nmx_exp(-745.0) == 5e-324
    assert abs(L.nmx_log(5e-324) - math.log(5e-324)) <= math.ulp(744.0)
