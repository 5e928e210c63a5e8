"""Pins the oracle restatement (and, where built, the reference shim) to
known answers:

* the reference's own unit-test oracles, restated for D3Q19
  (proj/tests/test_physics.cpp:41-72,147-190; proj/tests/test_lattice.cpp:25-126),
* golden end states produced by running the reference itself
  (tests/golden/golden_states.json, generator tests/golden/make_golden.py).
"""
import ctypes as C
import math
import os
import random

import numpy as np
import pytest

from paper_1510_03560_b200 import capi, scenario as S
from tests import scenarios
from tests.golden_check import assert_matches_golden, load_golden


def _lib(kind):
    if kind == "oracle":
        return C.CDLL(capi.ORACLE_LIB), "plbm_oracle_kat_"
    if not os.path.exists(capi.REF_LIB):
        pytest.skip("reference shim not built")
    return C.CDLL(capi.REF_LIB), "plbm_ref_kat_"


def _bind(kind):
    lib, p = _lib(kind)
    f = {}
    dp = C.POINTER(C.c_double)
    f["pr"] = getattr(lib, p + "pr_pressure")
    f["pr"].restype = C.c_double
    f["pr"].argtypes = [C.c_double, C.POINTER(S.ComponentDesc), C.POINTER(C.c_int)]
    f["psi"] = getattr(lib, p + "psi")
    f["psi"].restype = C.c_double
    f["psi"].argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_int)]
    f["feq"] = getattr(lib, p + "equilibrium")
    f["feq"].argtypes = [C.c_double, dp, dp]
    f["mom"] = getattr(lib, p + "moments")
    f["mom"].argtypes = [dp, dp, dp]
    f["intra"] = getattr(lib, p + "intra_force")
    f["intra"].argtypes = [dp, C.c_long, C.POINTER(C.c_long), C.POINTER(S.ComponentDesc), dp]
    f["inter"] = getattr(lib, p + "inter_force")
    f["inter"].argtypes = [C.c_double, dp, C.c_long, C.POINTER(C.c_long), C.c_double, dp]
    f["stencil"] = getattr(lib, p + "stencil")
    f["stencil"].argtypes = [C.POINTER(C.c_int), dp, C.POINTER(C.c_int)]
    return f


def _comp(c: S.Component) -> S.ComponentDesc:
    return S.CScenario(S.Scenario(components=[c])).desc.components[0]


def _pr_component():
    # proj/tests/test_physics.cpp:25-35
    Tc = 0.072922004074134239
    return S.Component(a=2.0 / 49.0, b=2.0 / 21.0, R=1.0, omega=0.344, Tc=Tc, T=0.85 * Tc)


KINDS = ["oracle", "ref"]


@pytest.mark.parametrize("kind", KINDS)
def test_stencil_moment_constraints(built, kind):
    f = _bind(kind)
    e = (C.c_int * 57)()
    w = (C.c_double * 19)()
    opp = (C.c_int * 19)()
    f["stencil"](e, w, opp)
    e = np.array(e).reshape(19, 3)
    w = np.array(w)
    assert tuple(e[0]) == (0, 0, 0) and w[0] == w.max()
    assert abs(w.sum() - 1.0) < 1e-15
    assert np.all(np.abs(w @ e) < 1e-15)
    m2 = np.einsum("i,ia,ib->ab", w, e, e)
    assert np.all(np.abs(m2 - np.eye(3) / 3.0) < 1e-15)
    for i in range(19):
        assert tuple(e[opp[i]]) == tuple(-e[i])
    assert sum(1 for i in range(19) if e[i][0] == 1) == 5  # crossing_count (topology.cpp:85-89)


@pytest.mark.parametrize("kind", KINDS)
def test_pr_pressure_oracles(built, kind):
    f = _bind(kind)
    pole = C.c_int()
    p = _comp(_pr_component())
    # frozen scalar oracle (test_physics.cpp:46-47)
    assert math.isclose(f["pr"](2.0, C.byref(p), C.byref(pole)), 0.014606129043274824,
                        rel_tol=1e-14)
    assert f["pr"](0.0, C.byref(p), C.byref(pole)) == 0.0
    f["pr"](1.0 / p.b, C.byref(p), C.byref(pole))
    assert pole.value == 1  # EOS pole
    # a = 0 -> rho R T / (1 - b rho)
    q = _comp(S.Component(**{**_pr_component().__dict__, "a": 0.0}))
    assert math.isclose(f["pr"](1.5, C.byref(q), C.byref(pole)),
                        1.5 * q.R * q.T / (1.0 - q.b * 1.5), rel_tol=1e-14)


@pytest.mark.parametrize("kind", KINDS)
def test_psi_clamp(built, kind):
    f = _bind(kind)
    cl = C.c_int()
    assert f["psi"](1.0, 0.0, -1.0, C.byref(cl)) > 0 and cl.value == 0
    assert f["psi"](1.0, 1.0, -1.0, C.byref(cl)) == 0.0 and cl.value == 1
    # ideal gas R T = cs2: psi is a signed zero (sqrt(-0) = -0 for g < 0)
    v = f["psi"](1.0, 1.0 / 3.0, -1.0, C.byref(cl))
    assert v == 0.0 and math.copysign(1.0, v) == -1.0 and cl.value == 0


@pytest.mark.parametrize("kind", KINDS)
def test_equilibrium_and_moments(built, kind):
    f = _bind(kind)
    out = (C.c_double * 19)()
    f["feq"](1.0, (C.c_double * 3)(0.1, 0.0, 0.0), out)
    # (1/18)(1 + 0.3 + 0.045 - 0.015) = 133/1800 (D3Q19 analogue of test_lattice.cpp:87-95)
    assert math.isclose(out[1], 133.0 / 1800.0, rel_tol=1e-14)
    f["feq"](0.0, (C.c_double * 3)(0.3, -0.2, 0.1), out)
    assert all(v == 0.0 for v in out)
    rng = random.Random(20240817)  # test_lattice.cpp:98-126 round trip
    rho, u = C.c_double(), (C.c_double * 3)()
    for _ in range(1000):
        r0 = rng.uniform(1e-3, 2.0)
        v0 = [rng.uniform(-0.1, 0.1) for _ in range(3)]
        f["feq"](r0, (C.c_double * 3)(*v0), out)
        f["mom"](out, C.byref(rho), u)
        assert abs(rho.value - r0) < 1e-12
        assert max(abs(u[a] - v0[a]) for a in range(3)) < 1e-12
    z = (C.c_double * 19)()
    f["mom"](z, C.byref(rho), u)
    assert rho.value == 0.0 and list(u) == [0.0, 0.0, 0.0]


@pytest.mark.parametrize("kind", KINDS)
def test_force_step_profile_oracles(built, kind):
    # psi = 1 for x < 3, 2 for x >= 3 on a 7x7x3 grid, cell (3,3,1):
    # sum w psi e_x = 1/6, sum w psi^2 e_x = 1/2 (also for D3Q19), so with
    # beta = 1.16, g = -1: F_x = 26/75 (test_physics.cpp:147-166); the inter
    # force with g = 0.2 and psi_self = 3 is -0.1 (test_physics.cpp:168-190).
    f = _bind(kind)
    nx, ny, nz = 7, 7, 3
    psi = np.fromfunction(lambda z, y, x: np.where(x < 3, 1.0, 2.0), (nz, ny, nx)).ravel()
    stride = (C.c_long * 3)(1, nx, nx * ny)
    cell = 3 + nx * (3 + ny * 1)
    F = (C.c_double * 3)()
    p = _comp(S.Component(**{**_pr_component().__dict__, "beta": 1.16, "g_self": -1.0}))
    f["intra"](psi.ctypes.data_as(C.POINTER(C.c_double)), cell, stride, C.byref(p), F)
    assert math.isclose(F[0], 26.0 / 75.0, rel_tol=1e-12)
    assert abs(F[1]) < 1e-15 and abs(F[2]) < 1e-15
    f["inter"](3.0, psi.ctypes.data_as(C.POINTER(C.c_double)), cell, stride, 0.2, F)
    assert math.isclose(F[0], -0.1, rel_tol=1e-13)


@pytest.mark.parametrize("name", sorted(load_golden()))
def test_oracle_reproduces_reference_golden_states(built, name):
    make, steps = scenarios.ALL[name]
    eng = capi.oracle_engine(make())
    eng.step(steps)
    assert_matches_golden(eng, name)


def test_oracle_matches_reference_c1_at_baseline_scale():
    """BASELINE configs[0] exactly (64^3, 16^3 tiles, S = 1e-12, 500 steps):
    the C restatement against the reference's own state digests
    (tests/golden/make_golden_large.py)."""
    import json
    from paper_1510_03560_b200 import capi
    from tests.golden.make_golden_large import LARGE, OUT, summary
    g = json.load(open(OUT))["c1_exact"]
    sc, steps, _ = LARGE["c1_exact"]()
    orc = capi.oracle_engine(sc)
    orc.step(steps)
    d = summary(orc)
    assert d["counters"] == g["counters"]
    assert d["creation_log"] == g["creation_log"]
    assert d["tiles"] == g["tiles"]
    assert d["digests"] == g["digests"]
