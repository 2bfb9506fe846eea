"""GPU parity, exact mode: the sm_100a kernels called through the C ABI reproduce the
reference CPU implementation BITWISE, on the same inputs.

Every comparison is against oracle/_ref (the compiled, unmodified reference) or, for
meshes the reference generators cannot produce (reversed faces), against the C
restatement oracle/swdg_port.c, which test_oracle.py pins bitwise to the reference.
"""
import math

import numpy as np
import pytest

from oracle import port, ref
from paper_1804_02221_b200 import swdg
from paper_1804_02221_b200.driver import run_simulation, run_simulation_device
from tests.conftest import gpu_available
from tests.helpers import (MESHES, beq, build, random_state, reversed_mesh, scenario_params,
                           smooth_state)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def cfg_from(p, mode=swdg.MODE_EXACT):
    return swdg.RunConfig(
        phys=swdg.PhysicsParams(p.g, p.h_tol, p.h_des, p.h_ref),
        visc=swdg.ViscosityConfig(bool(p.visc_enabled), p.epsilon0, p.sigma_min, p.sigma_max),
        limiter_enabled=bool(p.limiter_enabled), mode=mode)


def S(arrs):
    return swdg.State(*[a.copy() for a in arrs])


@pytest.mark.parametrize("name", sorted(MESHES))
def test_assemble_rhs_bitwise(name):
    m = build(name)
    p = ref.params(g=9.81)
    integ = swdg.TimeIntegrator(m, cfg_from(p))
    rng = np.random.default_rng(3)
    for dry in (0.0, 0.2):
        s = random_state(m.n_nodes, rng, dry_prob=dry)
        out = integ.assemble_rhs(S(s))
        assert beq(out.arrays(), ref.assemble_rhs(m, p, s))


@pytest.mark.parametrize("degree", list(range(1, 16)))
def test_assemble_rhs_all_degrees(degree):
    m = ref.build_mesh("wavy", degree, 3, 2, periodic_x=True, periodic_y=True).bathymetry("smooth")
    p = ref.params(g=9.81)
    s = random_state(m.n_nodes, np.random.default_rng(degree), dry_prob=0.1)
    out = swdg.TimeIntegrator(m, cfg_from(p)).assemble_rhs(S(s))
    assert beq(out.arrays(), ref.assemble_rhs(m, p, s))


def test_reversed_faces_against_port():
    base = build("wavy_N4")
    m, _, _ = reversed_mesh(base)
    assert m.faces[:, 4].any()
    p = ref.params(g=9.81, visc=True, epsilon0=0.1, sigma_min=-6.5, sigma_max=-5.0)
    s = random_state(m.n_nodes, np.random.default_rng(5), dry_prob=0.1)
    integ = swdg.TimeIntegrator(m, cfg_from(p))
    r_gpu = integ.evaluate_rhs(S(s))
    r_port, eps = port.evaluate_rhs(m, p, s)
    assert beq(r_gpu.arrays(), r_port)
    assert beq([integ.last_eps()], [eps])


@pytest.mark.parametrize("name", ["wavy_N4", "dam_N4", "wavy_N7", "cart_1x1_periodic_N2",
                                  "cart_N3_walls"])
def test_evaluate_rhs_viscous_bitwise(name):
    m = build(name)
    N = m.degree
    smin = -(4.0 + 4.25 * math.log10(N)) - 1.0
    rng = np.random.default_rng(17)
    for state in (random_state(m.n_nodes, rng, dry_prob=0.05), smooth_state(m, 0.3)):
        for band in ((smin, smin + 2.0), (-6.5, -5.0)):
            p = ref.params(g=9.81, visc=True, epsilon0=0.1, sigma_min=band[0], sigma_max=band[1])
            ri = ref.Integrator(m, p)
            r_ref = ri.evaluate_rhs(state)
            gi = swdg.TimeIntegrator(m, cfg_from(p))
            r_gpu = gi.evaluate_rhs(S(state))
            assert beq(r_gpu.arrays(), r_ref)
            assert beq([gi.last_eps()], [ri.last_eps()])


@pytest.mark.parametrize("sid,kx,deg", [("wetdry_dambreak", 10, 3), ("parabolic_dam_dry", 8, 3),
                                        ("oscillating_lake", 12, 4), ("three_mound", 10, 2),
                                        ("parabolic_dam_wet", 8, 7)])
def test_try_step_sequence_bitwise(sid, kx, deg):
    m, st = ref.scenario_mesh(sid, kx, kx, deg)
    p, cfg = scenario_params(sid, deg)
    ri = ref.Integrator(m, p)
    gi = swdg.TimeIntegrator(m, cfg_from(p))
    s1 = [a.copy() for a in st]
    s2 = S(st)
    t = 0.0
    for _ in range(10):
        dt = ref.compute_dt(m, p, s1, cfg["cfl"])
        assert gi.compute_dt(s2, cfg["cfl"]) == dt
        a = ri.try_step(s1, t, dt)
        ok = gi.try_step(s2, t, dt)
        assert ok == bool(a.accepted)
        assert gi.last_limited_count() == a.n_limited
        assert gi.last_max_eps() == a.max_eps
        assert gi.last_min_stage_h() == a.min_stage_h
        assert beq(s2.arrays(), s1)
        t += dt
    d_ref, d_gpu = ref.diagnostics(m, p, s1), gi.diagnostics(s2)
    assert d_gpu.min_h == d_ref.min_h
    assert abs(d_gpu.mass - d_ref.mass) <= 1e-13 * abs(d_ref.mass)
    assert abs(d_gpu.entropy - d_ref.entropy) <= 1e-13 * abs(d_ref.entropy)
    assert abs(d_gpu.positivity_dt - d_ref.positivity_dt) <= 1e-13 * d_ref.positivity_dt


def test_reject_leaves_state_and_abort_raises():
    m, st = ref.scenario_mesh("wetdry_dambreak", 8, 8, 3)
    p, cfg = scenario_params("wetdry_dambreak")
    dt = 20 * ref.compute_dt(m, p, st, cfg["cfl"])
    gi = swdg.TimeIntegrator(m, cfg_from(p))
    s = S(st)
    assert gi.try_step(s, 0.0, dt) is False
    assert beq(s.arrays(), st)
    p0 = scenario_params("wetdry_dambreak", limiter_enabled=0.0)[0]
    with pytest.raises(swdg.NumericalAbort):
        swdg.TimeIntegrator(m, cfg_from(p0)).try_step(S(st), 0.0, dt)


@pytest.mark.parametrize("sid,kx,T,steps,fp", [
    ("wetdry_dambreak", 12, 0.2, 12, "b7a50b5a3ff22ec4"),
    ("parabolic_dam_dry", 8, 0.1, 13, "a57e2e67759014a6"),
])
def test_full_run_fingerprints(sid, kx, T, steps, fp):
    """Chaotic wet/dry runs: only a bitwise path reproduces these."""
    m, st = ref.scenario_mesh(sid, kx, kx, 0)
    p, cfg = scenario_params(sid)
    gi = swdg.TimeIntegrator(m, cfg_from(p))
    res = run_simulation(gi, S(st), T, cfg["cfl"], diagnostics=False)
    assert res.steps == steps
    assert ref.fnv1a_state(res.state.arrays()) == fp


@pytest.mark.parametrize("mode", [swdg.MODE_EXACT, swdg.MODE_FAST])
@pytest.mark.parametrize("sid,kx,T,steps,fp", [
    ("wetdry_dambreak", 12, 0.2, 12, "b7a50b5a3ff22ec4"),
    ("parabolic_dam_dry", 8, 0.1, 13, "a57e2e67759014a6"),
])
def test_device_driver_matches_host_driver(mode, sid, kx, T, steps, fp):
    """The device-resident driver (state uploaded once, reject-and-halve rolled back
    on the device, snapshots downloaded on the way) takes the same decisions as the
    host-state driver: bitwise the same trajectory, step count and diagnostics; in
    exact mode that is the reference's fingerprint."""
    m, st = ref.scenario_mesh(sid, kx, kx, 0)
    p, cfg = scenario_params(sid)
    host = run_simulation(swdg.TimeIntegrator(m, cfg_from(p, mode)), S(st), T, cfg["cfl"],
                          snapshot_times=(0.5 * T,))
    snaps = []
    dev = run_simulation_device(swdg.TimeIntegrator(m, cfg_from(p, mode)), S(st), T, cfg["cfl"],
                                snapshot_times=(0.5 * T,),
                                on_snapshot=lambda t, s: snaps.append((t, s.copy())))
    assert dev.steps == host.steps and dev.t == host.t
    assert beq(dev.state.arrays(), host.state.arrays())
    assert [(a.step, a.dt, a.mass, a.entropy, a.min_h, a.n_limited) for a in dev.series] == \
        [(a.step, a.dt, a.mass, a.entropy, a.min_h, a.n_limited) for a in host.series]
    assert len(snaps) == 1 and snaps[0][0] == 0.5 * T
    if mode == swdg.MODE_EXACT:  # without the snapshot event: the reference's fingerprint
        plain = run_simulation_device(swdg.TimeIntegrator(m, cfg_from(p, mode)), S(st), T,
                                      cfg["cfl"], diagnostics=False)
        assert plain.steps == steps and ref.fnv1a_state(plain.state.arrays()) == fp


def test_forcing_callback_bitwise():
    m = ref.build_mesh("cartesian", 3, 6, 6, periodic_x=True, periodic_y=True)
    p = ref.params(g=9.81)
    h0, amp, u0, v0, k, g = 2.0, 0.2, 0.7, 0.3, 2 * math.pi, 9.81
    omega = k * (u0 + v0)

    def forcing(x, y, t):  # validate.hpp:549-556, vectorised
        hx = amp * k * np.cos(k * (x + y) - omega * t)
        hh = h0 + amp * np.sin(k * (x + y) - omega * t)
        f = g * hh * hx
        return np.zeros_like(x), f, f

    x, y = m.arrays["x"], m.arrays["y"]
    hh = 2.0 + 0.2 * np.sin(2 * math.pi * (x + y))
    st = [hh, hh * 0.7, hh * 0.3]
    gi = swdg.TimeIntegrator(m, cfg_from(p))
    gi.forcing = forcing
    s_gpu, s_port = S(st), [a.copy() for a in st]
    for step in range(3):
        dt = ref.compute_dt(m, p, s_port, 0.4)
        gi.try_step(s_gpu, step * dt, dt)
        port.try_step(m, p, s_port, step * dt, dt, forcing=(h0, amp, u0, v0, k, g))
        # numpy sin/cos may differ from glibc's by an ulp: normwise, not bitwise
        err = max(np.abs(a - b).max() for a, b in zip(s_gpu.arrays(), s_port))
        assert err <= 1e-13 * max(np.abs(b).max() for b in s_port)
