"""The oracle is pinned before it is trusted (CPU only).

1. Fingerprints the survey recorded for the reference itself.
2. Known answers restated from the reference's own unit tests (proj/tests/*.cpp).
3. The plain-C restatement (oracle/swdg_port.c) is bitwise equal to the compiled
   reference (oracle/_ref) on every stage-path function, over meshes, degrees, wet/dry
   states and viscosity settings.
"""
import math

import numpy as np
import pytest

from oracle import port, ref
from tests.helpers import MESHES, beq, build, random_state, scenario_params, smooth_state

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


# ---------------------------------------------------------------- fingerprints
@pytest.mark.parametrize("sid,kx,T,steps,fp", [
    ("wetdry_dambreak", 12, 0.2, 12, "b7a50b5a3ff22ec4"),
    ("parabolic_dam_dry", 8, 0.1, 13, "a57e2e67759014a6"),
])
def test_reference_fingerprints(sid, kx, T, steps, fp):
    s, n, t = ref.run_simulation(sid, kx, kx, 0, T)
    assert n == steps and abs(t - T) < 1e-12
    assert ref.fnv1a_state(s) == fp


# ---------------------------------------------------------------- known answers
def test_es_flux_known_answers():
    # zero jump reduces to the EC flux (test_fluxes.cpp:113-121)
    w = [1.5, 0.6, -0.9]
    f = port.es_flux(w, w, 0.2, 0.2, 1.0, 0.0, 9.81)
    u = w[1] / w[0]
    ec = [w[0] * u, w[0] * u * u + 0.5 * 9.81 * w[0] ** 2, w[0] * u * (w[2] / w[0])]
    assert np.allclose(f, ec, atol=1e-14, rtol=0)
    # dry-right pair at rest: mass flux sqrt(10)/4 (test_fluxes.cpp:148-153)
    f = port.es_flux([1.0, 0, 0], [0.0, 0, 0], 0.0, 0.0, 1.0, 0.0, 10.0)
    assert abs(f[0] - math.sqrt(10.0) / 4.0) < 1e-14
    # non-unit normal rejected (test_fluxes.cpp:199-203)
    with pytest.raises(RuntimeError):
        port.es_flux([1, 0, 0], [1, 0, 0], 0, 0, 0.9, 0.0, 9.81)


def test_hand_assembled_single_element():
    """test_dg_rhs.cpp:133-171: one periodic N=1 element, h = 1|2 along xi, at rest."""
    m = ref.build_mesh("cartesian", 1, 1, 1, 0.0, 2.0, 0.0, 2.0, True, True)
    p = ref.params(g=10.0)
    h = np.zeros(4)
    h[[0, 1]] = 1.0
    h[[2, 3]] = 2.0
    s = [h, np.zeros(4), np.zeros(4)]
    g = 10.0

    def fsharp2(a, b):
        return g * (0.5 * (a + b)) ** 2 - 0.5 * g * 0.5 * (a * a + b * b)

    fstar = 0.5 * g * 0.5 * (1.0 + 4.0)
    lhs0 = fsharp2(1.0, 2.0) - fstar
    lhs1 = -fsharp2(2.0, 1.0) + fstar
    for out in (port.assemble_rhs(m, p, s), ref.assemble_rhs(m, p, s)):
        for j in range(2):
            assert abs(out[1][j] - (-lhs0)) < 1e-13
            assert abs(out[1][2 + j] - (-lhs1)) < 1e-13
            assert abs(out[2][j]) < 1e-13


def test_lake_at_rest_well_balanced():
    """test_dg_rhs.cpp:62-93 and SURVEY §8d config C1 (discontinuous b off mesh lines)."""
    m = ref.build_mesh("curved_dam", 4, 16, 16).bathymetry("step", 0.0, 0.3, 0.1)
    p = ref.params(g=9.81)
    b = m.arrays["b"]
    s = [1.0 - b, np.zeros_like(b), np.zeros_like(b)]
    r = port.assemble_rhs(m, p, s)
    assert max(np.abs(x).max() for x in r) < 1e-11


def test_limiter_hand_case():
    """test_limiter.cpp:65-80: mean 0.9, minimum -0.1 -> theta 0.9."""
    m = ref.build_mesh("cartesian", 1, 1, 1)
    p = ref.params()
    rest = (0.9 * 4.0 + 0.1) / 3.0
    h = np.array([rest, rest, rest, -0.1])
    hu = np.full(4, 0.4)
    hv = np.zeros(4)
    theta = np.zeros(1)
    import ctypes as C
    ref.check(ref.lib().ref_limit_all(m.handle, C.byref(p), ref.ptr(h), ref.ptr(hu),
                                      ref.ptr(hv), 0, ref.ptr(theta)))
    assert abs(theta[0] - 0.9) < 1e-14
    assert h.min() >= 0.0 and abs(h.min()) < 1e-15


def test_dt_exact_value():
    """test_timeloop.cpp:55-63: uniform Cartesian rest state, dt = 0.5*0.1/(7 sqrt(g*2))."""
    m = ref.build_mesh("cartesian", 3, 10, 10)
    p = ref.params(g=9.81)
    n = m.n_nodes
    s = [np.full(n, 2.0), np.zeros(n), np.zeros(n)]
    dt = port.compute_dt(m, p, s, 0.5)
    assert abs(dt - 0.5 * 0.1 / (7.0 * math.sqrt(9.81 * 2.0))) < 1e-15
    # all-dry fallback (test_timeloop.cpp:82-89)
    s0 = [np.zeros(n)] * 3
    assert port.compute_dt(m, p, s0, 0.5) == ref.compute_dt(m, p, s0, 0.5)


# ---------------------------------------------------------------- port == reference
@pytest.mark.parametrize("name", sorted(MESHES))
def test_port_assemble_rhs_bitwise(name):
    m = build(name)
    rng = np.random.default_rng(7)
    p = ref.params(g=9.81)
    for dry in (0.0, 0.15):
        s = random_state(m.n_nodes, rng, dry_prob=dry)
        assert beq(port.assemble_rhs(m, p, s), ref.assemble_rhs(m, p, s))


@pytest.mark.parametrize("name", ["wavy_N4", "dam_N4", "wavy_N7", "cart_1x1_periodic_N2"])
def test_port_viscous_rhs_bitwise(name):
    m = build(name)
    rng = np.random.default_rng(11)
    N = m.degree
    smin = -(4.0 + 4.25 * math.log10(N)) - 1.0
    for state in (random_state(m.n_nodes, rng), smooth_state(m, 0.3)):
        # a band placed so smooth fields land inside the sine ramp
        for band in ((smin, smin + 2.0), (-6.5, -5.0)):
            p = ref.params(g=9.81, visc=True, epsilon0=0.1, sigma_min=band[0], sigma_max=band[1])
            integ = ref.Integrator(m, p)
            r_ref = integ.evaluate_rhs(state)
            r_port, eps = port.evaluate_rhs(m, p, state)
            assert beq(r_port, r_ref)
            assert beq([eps], [integ.last_eps()])


def test_port_viscosity_ramp_exercised():
    m = build("wavy_N4")
    p = ref.params(g=9.81, visc=True, epsilon0=0.1, sigma_min=-6.5, sigma_max=-5.0)
    eps = port.compute_viscosity(m, p, smooth_state(m, 0.3)[0])
    inside = (eps > 0) & (eps < 0.1)
    assert inside.any(), "no element inside the sine ramp: the log10/sin path is untested"


@pytest.mark.parametrize("sid,kx,deg", [("wetdry_dambreak", 10, 3), ("parabolic_dam_dry", 8, 3),
                                        ("oscillating_lake", 12, 4), ("three_mound", 10, 2)])
def test_port_try_step_sequence_bitwise(sid, kx, deg):
    m, st = ref.scenario_mesh(sid, kx, kx, deg)
    p, cfg = scenario_params(sid, deg)
    integ = ref.Integrator(m, p)
    s1 = [a.copy() for a in st]
    s2 = [a.copy() for a in st]
    t = 0.0
    for _ in range(8):
        dt = ref.compute_dt(m, p, s1, cfg["cfl"])
        assert dt == port.compute_dt(m, p, s2, cfg["cfl"])
        a = integ.try_step(s1, t, dt)
        b = port.try_step(m, p, s2, t, dt)
        assert (a.accepted, a.n_limited) == (b.accepted, b.n_limited)
        assert a.min_stage_h == b.min_stage_h and a.max_eps == b.max_eps
        assert beq(s1, s2)
        t += dt
    d1, d2 = ref.diagnostics(m, p, s1), port.diagnostics(m, p, s2)
    for k in ("mass", "entropy", "min_h", "positivity_dt"):
        assert getattr(d1, k) == getattr(d2, k)


def test_port_reject_and_abort():
    m, st = ref.scenario_mesh("wetdry_dambreak", 8, 8, 3)
    p, cfg = scenario_params("wetdry_dambreak")
    dt = 20 * ref.compute_dt(m, p, st, cfg["cfl"])  # far above CFL: negative means
    s1 = [a.copy() for a in st]
    s2 = [a.copy() for a in st]
    a = ref.Integrator(m, p).try_step(s1, 0.0, dt)
    b = port.try_step(m, p, s2, 0.0, dt)
    assert a.accepted == b.accepted == 0
    assert beq(s1, st) and beq(s2, st)
    p0 = scenario_params("wetdry_dambreak", limiter_enabled=0.0)[0]
    with pytest.raises(ArithmeticError):
        port.try_step(m, p0, [a.copy() for a in st], 0.0, dt)
    with pytest.raises(RuntimeError, match="reference error 3"):
        ref.Integrator(m, p0).try_step([a.copy() for a in st], 0.0, dt)


def test_port_forcing_bitwise():
    """Manufactured traveling-wave forcing (validate.hpp:543-556)."""
    m = ref.build_mesh("cartesian", 3, 6, 6, periodic_x=True, periodic_y=True)
    p = ref.params(g=9.81)
    fp = (2.0, 0.2, 0.7, 0.3, 2 * math.pi, 9.81)
    x, y = m.arrays["x"], m.arrays["y"]
    h = 2.0 + 0.2 * np.sin(2 * math.pi * (x + y))
    s1 = [h.copy(), h * 0.7, h * 0.3]
    s2 = [a.copy() for a in s1]
    integ = ref.Integrator(m, p, forcing=fp)
    for k in range(3):
        dt = ref.compute_dt(m, p, s1, 0.4)
        integ.try_step(s1, k * dt, dt)
        port.try_step(m, p, s2, k * dt, dt, forcing=fp)
        assert beq(s1, s2)
