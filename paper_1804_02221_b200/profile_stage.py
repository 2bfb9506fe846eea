"""Small driver for ncu captures of the stage kernels: a wavy periodic mesh, smooth
state, fixed dt, a few device-resident SSPRK3 steps.

    python -m paper_1804_02221_b200.profile_stage --degree 7 --kx 200 --steps 2
"""
from __future__ import annotations

import argparse

import numpy as np

from . import swdg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--degree", type=int, default=7)
    ap.add_argument("--kx", type=int, default=200)
    ap.add_argument("--ky", type=int, default=0, help="elements in y (default: kx)")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--viscous", action="store_true")
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--time", type=int, default=0, help="time this many extra steps")
    ap.add_argument("--diag", action="store_true",
                    help="also run the step reductions (run_steps with reductions, step_device)")
    a = ap.parse_args()
    N = a.degree
    visc = swdg.ViscosityConfig(False)
    if a.viscous:
        smin, smax = swdg.default_sigma_band(N)
        visc = swdg.ViscosityConfig(True, 0.1, smin, smax)
    cfg = swdg.RunConfig(phys=swdg.PhysicsParams(9.81), visc=visc,
                         mode=swdg.MODE_EXACT if a.exact else swdg.MODE_FAST)
    spec = swdg.structured_spec("wavy", N, a.kx, a.ky or a.kx, periodic_x=True, periodic_y=True,
                                bathy="smooth")
    integ = swdg.TimeIntegrator.structured(spec, cfg)
    x, y = integ.geometry("x"), integ.geometry("y")
    h = 1.0 + 0.1 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y)
    st = swdg.State(h, 0.3 * h, -0.2 * h)
    integ.upload(st)
    dt = 0.1 * integ.compute_dt_device(0.5)
    integ.run_steps(a.steps, 0.0, dt, reductions=a.diag)
    if a.diag:
        integ.step_device(a.steps * dt, dt, 0.5)
    integ.synchronize()
    if a.time:
        import time
        reps = a.time
        t0 = time.perf_counter()
        # ends with a flag read (host sync); with --diag every step also runs the
        # per-step reductions
        integ.run_steps(reps, 0.0, dt, reductions=a.diag)
        el = time.perf_counter() - t0
        dofs = 3 * integ.mesh.n_nodes
        print(f"N={N} kx={a.kx} visc={a.viscous} diag={a.diag} stage_ms={el / reps / 3 * 1e3:.3f} "
              f"step_ms={el / reps * 1e3:.3f} dof_per_s={dofs * reps * 3 / el:.4e} "
              f"accepted={integ.last_info().accepted}")
    else:
        print("ok", integ.last_info().accepted, integ.launch_count())


if __name__ == "__main__":
    main()
