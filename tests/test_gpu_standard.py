"""GPU parity, standard scheme (SchemeMode::standard, dg_rhs.hpp:14): the standard DGSEM
volume term (standard_volume_element dg_rhs.hpp:75-117) with the local Lax-Friedrichs
interface flux in strong form (llf_surface_flux fluxes.hpp:192-202, surface_terms
dg_rhs.hpp:228-246) — the paper's comparison scheme and the `entropy_glitch` scenario.
It runs on the exact-mode kernels and must match the reference BITWISE."""
import numpy as np
import pytest

from oracle import ref
from paper_1804_02221_b200 import swdg
from tests.conftest import gpu_available
from tests.helpers import MESHES, beq, build, random_state, scenario_params

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]

STD = swdg.SCHEME_STANDARD


def cfg_from(p, mode=swdg.MODE_EXACT, scheme=STD):
    return swdg.RunConfig(
        phys=swdg.PhysicsParams(p.g, p.h_tol, p.h_des, p.h_ref),
        visc=swdg.ViscosityConfig(bool(p.visc_enabled), p.epsilon0, p.sigma_min, p.sigma_max),
        limiter_enabled=bool(p.limiter_enabled), mode=mode, scheme=scheme)


def S(arrs):
    return swdg.State(*[a.copy() for a in arrs])


@pytest.mark.parametrize("name", sorted(MESHES))
def test_standard_assemble_rhs_bitwise(name):
    m = build(name)
    p = ref.params(g=9.81)
    integ = swdg.TimeIntegrator(m, cfg_from(p))
    rng = np.random.default_rng(11)
    for dry in (0.0, 0.2):
        s = random_state(m.n_nodes, rng, dry_prob=dry)
        out = integ.assemble_rhs(S(s))
        assert beq(out.arrays(), ref.assemble_rhs(m, p, s, mode=1))


@pytest.mark.parametrize("degree", [1, 2, 5, 9, 15])
def test_standard_all_degrees_bitwise(degree):
    m = ref.build_mesh("wavy", degree, 3, 2, periodic_x=True, periodic_y=True).bathymetry("smooth")
    p = ref.params(g=9.81)
    s = random_state(m.n_nodes, np.random.default_rng(degree), dry_prob=0.1)
    out = swdg.TimeIntegrator(m, cfg_from(p)).assemble_rhs(S(s))
    assert beq(out.arrays(), ref.assemble_rhs(m, p, s, mode=1))


def test_standard_differs_from_es():
    """The scheme switch reaches the kernels (a state away from rest)."""
    m = build("wavy_N4")
    p = ref.params(g=9.81)
    s = random_state(m.n_nodes, np.random.default_rng(2), dry_prob=0.0)
    es = swdg.TimeIntegrator(m, cfg_from(p, scheme=swdg.SCHEME_ES)).assemble_rhs(S(s)).arrays()
    sd = swdg.TimeIntegrator(m, cfg_from(p)).assemble_rhs(S(s)).arrays()
    assert max(np.abs(a - b).max() for a, b in zip(es, sd)) > 1e-6


@pytest.mark.parametrize("mode", [swdg.MODE_EXACT, swdg.MODE_FAST])
def test_entropy_glitch_try_steps_bitwise(mode):
    """The reference's standard-scheme scenario (scenarios.hpp:41-52) for 10 steps of
    try_step: state, limiter counts and min stage height bitwise.  A FAST-mode request
    runs the same exact kernels (the standard scheme has no fast path)."""
    m, st = ref.scenario_mesh("entropy_glitch", 20, 20, 1)
    p, cfg = scenario_params("entropy_glitch", 1)
    p.scheme = 1
    ri = ref.Integrator(m, p)
    gi = swdg.TimeIntegrator(m, cfg_from(p, mode=mode))
    s1 = [a.copy() for a in st]
    s2 = S(st)
    t = 0.0
    for _ in range(10):
        dt = ref.compute_dt(m, p, s1, cfg["cfl"])
        assert gi.compute_dt(s2, cfg["cfl"]) == dt
        a = ri.try_step(s1, t, dt)
        assert gi.try_step(s2, t, dt) == bool(a.accepted)
        assert gi.last_limited_count() == a.n_limited
        assert gi.last_min_stage_h() == a.min_stage_h
        assert beq(s2.arrays(), s1)
        t += dt


def test_standard_ignores_viscosity_like_the_reference():
    """evaluate_rhs adds artificial viscosity for SchemeMode::es only (timeloop.hpp:178)."""
    m = build("dam_N4")
    p = ref.params(g=9.81, epsilon0=0.1, sigma_min=-3.0, sigma_max=-1.0, visc=True)
    s = random_state(m.n_nodes, np.random.default_rng(4), dry_prob=0.0)
    out = swdg.TimeIntegrator(m, cfg_from(p)).assemble_rhs(S(s))
    p0 = ref.params(g=9.81)
    assert beq(out.arrays(), ref.assemble_rhs(m, p0, s, mode=1))
