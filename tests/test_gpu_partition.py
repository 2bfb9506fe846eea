"""Partitioned stepping on the GPU: several element partitions (ghost elements, halo
pack/unpack kernels, split-step C ABI) in one process on cuda:0, exchanged through
the loopback exchanger, reproduce the unpartitioned run — bitwise in exact mode
(hence the reference) and bitwise against the single-partition fast run."""
import numpy as np
import pytest

from oracle import ref
from paper_1804_02221_b200 import partition as part
from paper_1804_02221_b200 import swdg
from paper_1804_02221_b200.distributed import (GpuPartition, LoopbackExchanger,
                                               compute_dt_distributed, try_step_loopback)
from tests.conftest import gpu_available
from tests.helpers import beq, build, random_state, scenario_params

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def cfg_from(p, mode):
    return swdg.RunConfig(
        phys=swdg.PhysicsParams(p.g, p.h_tol, p.h_des, p.h_ref),
        visc=swdg.ViscosityConfig(bool(p.visc_enabled), p.epsilon0, p.sigma_min, p.sigma_max),
        limiter_enabled=bool(p.limiter_enabled), mode=mode)


def run_parts(m, cfg, st, P, dt, steps):
    import torch
    lms = [part.local_mesh(m, P, r) for r in range(P)]
    bs = [GpuPartition(lm, cfg) for lm in lms]
    for lm, b in zip(lms, bs):
        b.upload(part.scatter_state(st, lm))
    ex = LoopbackExchanger(bs, lambda n: torch.zeros(n, dtype=torch.float64, device="cuda"))
    acc = []
    for k in range(steps):
        acc.append(try_step_loopback(bs, ex, k * dt, dt))
    np_ = m.n1 * m.n1
    out = [np.zeros(m.n_nodes) for _ in range(3)]
    for lm, b in zip(lms, bs):
        w = b.download()
        sel = (lm.global_ids[: lm.n_owned, None] * np_ + np.arange(np_)).ravel()
        for o, a in zip(out, w):
            o[sel] = a[: lm.n_owned * np_]
    return out, acc


@pytest.mark.parametrize("mode", [swdg.MODE_EXACT, swdg.MODE_FAST])
@pytest.mark.parametrize("sid,kx,deg,P", [("wetdry_dambreak", 8, 3, 2),
                                          ("parabolic_dam_dry", 8, 3, 3),
                                          ("oscillating_lake", 10, 4, 4)])
def test_partitioned_equals_single(mode, sid, kx, deg, P):
    m, st = ref.scenario_mesh(sid, kx, kx, deg)
    p, cfg = scenario_params(sid, deg)
    dt = ref.compute_dt(m, p, st, cfg["cfl"])
    single = swdg.TimeIntegrator(m, cfg_from(p, mode))
    want = swdg.State(*[a.copy() for a in st])
    acc_ref = [single.try_step(want, k * dt, dt) for k in range(4)]
    got, acc = run_parts(m, cfg_from(p, mode), st, P, dt, 4)
    assert acc == acc_ref
    assert beq(got, want.arrays())
    if mode == swdg.MODE_EXACT:  # and therefore the reference itself
        ri = ref.Integrator(m, p)
        s = [a.copy() for a in st]
        for k in range(4):
            ri.try_step(s, k * dt, dt)
        assert beq(got, s)


@pytest.mark.parametrize("mode", [swdg.MODE_EXACT, swdg.MODE_FAST])
@pytest.mark.parametrize("sid,kx,deg,P", [("wetdry_dambreak", 12, 3, 2),
                                          ("oscillating_lake", 16, 4, 3),
                                          ("parabolic_dam_dry", 12, 2, 2)])
def test_partitioned_overlap_inviscid(mode, sid, kx, deg, P):
    """Inviscid partitions with an interior run each stage as interior (before the
    exchange) + the halo-adjacent rest (after it): still bitwise the single run."""
    m, st = ref.scenario_mesh(sid, kx, kx, deg)
    p, cfg = scenario_params(sid, deg, visc_enabled=0.0)
    dt = ref.compute_dt(m, p, st, cfg["cfl"])
    lo, hi = part.interior_range(part.local_mesh(m, P, 0).faces, part.local_mesh(m, P, 0).n_owned)
    assert hi - lo >= 2  # the split path is the one exercised
    single = swdg.TimeIntegrator(m, cfg_from(p, mode))
    want = swdg.State(*[a.copy() for a in st])
    acc_ref = [single.try_step(want, k * dt, dt) for k in range(4)]
    got, acc = run_parts(m, cfg_from(p, mode), st, P, dt, 4)
    assert acc == acc_ref
    assert beq(got, want.arrays())


def test_structured_partitions_match_global_mesh():
    """Device-generated partitions (owned + ghost elements by global id) carry exactly
    the global mesh's geometry, and partitioned fast stepping equals the global run."""
    import torch
    spec = swdg.structured_spec("wavy", 4, 12, 10, periodic_x=True, periodic_y=True,
                                bathy="smooth")
    cfg = swdg.RunConfig(phys=swdg.PhysicsParams(9.81), mode=swdg.MODE_FAST)
    glob = swdg.TimeIntegrator.structured(spec, cfg)
    np_ = 25
    P = 3
    bs = [GpuPartition.structured(spec, cfg, P, r) for r in range(P)]
    for b in bs:
        sel = (b.lm.global_ids[:, None] * np_ + np.arange(np_)).ravel()
        for k in ("x", "y", "x_xi", "y_eta", "jac", "b"):
            assert np.array_equal(b.integ.geometry(k), glob.geometry(k)[sel]), k
    x, y = glob.geometry("x"), glob.geometry("y")
    h = 1.0 + 0.1 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y)
    st = [h, 0.3 * h, -0.2 * h]
    s_glob = swdg.State(*[a.copy() for a in st])
    glob.upload(s_glob)
    dt = 0.3 * glob.compute_dt_device(0.5)
    glob.run_steps(3, 0.0, dt)
    glob.download(s_glob)
    for b in bs:
        b.upload(part.scatter_state(st, b.lm))
    ex = LoopbackExchanger(bs, lambda n: torch.zeros(n, dtype=torch.float64, device="cuda"))
    for k in range(3):
        assert try_step_loopback(bs, ex, k * dt, dt)
    got = [np.zeros(len(h)) for _ in range(3)]
    for b in bs:
        w = b.download()
        sel = (b.lm.global_ids[: b.lm.n_owned, None] * np_ + np.arange(np_)).ravel()
        for o, a in zip(got, w):
            o[sel] = a[: b.lm.n_owned * np_]
    assert beq(got, s_glob.arrays())


def test_distributed_dt_matches():
    m = build("wavy_N4")
    p = ref.params(g=9.81)
    st = random_state(m.n_nodes, np.random.default_rng(4), h=(0.5, 1.5))
    cfg = cfg_from(p, swdg.MODE_EXACT)
    lms = [part.local_mesh(m, 3, r) for r in range(3)]
    bs = [GpuPartition(lm, cfg) for lm in lms]
    for lm, b in zip(lms, bs):
        b.upload(part.scatter_state(st, lm))

    class MinEx:  # all-min over the in-process partitions
        def __init__(self, bs):
            self.vals = [b.dt_candidates() for b in bs]

        def all_min(self, v):
            return [min(x[0] for x in self.vals), min(x[1] for x in self.vals)]

    dt = compute_dt_distributed(bs[0], MinEx(bs), 0.5, m.degree, cfg.phys)
    assert dt == ref.compute_dt(m, p, st, 0.5)


def test_visc_interior_pass_touches_only_its_range():
    """The interior viscous pre-pass (run during the state exchange) computes eps and
    the flux pairs of the interior range only; the halo-adjacent elements keep their
    previous values until the boundary pass (a pre-kernel that ignored the range would
    redo, and for the boundary elements miscompute, the whole partition)."""
    sid, kx, deg, P = "wetdry_dambreak", 12, 3, 2
    m, st = ref.scenario_mesh(sid, kx, kx, deg)
    p, _ = scenario_params(sid, deg)
    lm = part.local_mesh(m, P, 0)
    b = GpuPartition(lm, cfg_from(p, swdg.MODE_FAST))
    lo, hi = part.interior_range(lm.faces, lm.n_owned)
    lo, hi = (lo + 1) & ~1, hi & ~1  # swdg_gpu_set_interior's even bounds
    assert hi - lo >= 2 and (lo > 0 or hi < lm.n_owned)
    n = lm.n_elem * lm.n1 * lm.n1
    lake = [np.full(n, 2.0), np.zeros(n), np.zeros(n)]  # no modal energy: eps = 0
    rough = random_state(n, np.random.default_rng(5))
    b.upload(lake)
    b.step_begin()
    b.stage_visc(0, 0.0, 1e-4)
    assert not b.integ.last_eps()[: lm.n_owned].any()
    b.upload(rough)
    b.step_begin()
    b.stage_visc_part(0, 0.0, 1e-4, 1)  # interior only
    e1 = b.integ.last_eps()[: lm.n_owned]
    outside = np.r_[0:lo, hi:lm.n_owned]
    assert e1[lo:hi].any()
    assert not e1[outside].any()
    b.stage_visc_part(0, 0.0, 1e-4, 2)  # the rest
    e2 = b.integ.last_eps()[: lm.n_owned]
    b.step_begin()
    b.stage_visc(0, 0.0, 1e-4)  # everything at once
    assert beq([e2], [b.integ.last_eps()[: lm.n_owned]])
