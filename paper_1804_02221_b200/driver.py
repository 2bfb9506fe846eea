"""Step loop around the GPU TimeIntegrator, mirroring run_simulation (driver.hpp:62-142).

CFL step from compute_dt (timeloop.hpp:53), snapping to the final time and snapshot
events with the reference's t_eps, reject-and-halve up to 10 times
(driver.hpp:101-111), and the per-step StepDiagnostics fields (driver.hpp:115-127,
computed on the device).  The reference-format output files (io.hpp) are written by
the C++ device driver, include/swdg_gpu_driver.hpp.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .swdg import NumericalAbort, State, TimeIntegrator


@dataclass
class StepDiagnostics:
    """timeloop.hpp:131-142"""
    step: int
    t: float
    dt: float
    mass: float
    entropy: float
    min_h: float
    n_limited: int
    max_eps: float
    min_stage_h: float
    positivity_dt: float


@dataclass
class RunResult:
    state: State
    t: float = 0.0
    steps: int = 0
    series: list = field(default_factory=list)
    mass_initial: float = 0.0
    entropy_initial: float = 0.0
    worst_limiter_entropy_jump: float = 0.0  # only with track_limiter_entropy


def run_simulation(integ: TimeIntegrator, state: State, final_time: float, cfl: float,
                   snapshot_times=(), keep_series: bool = True, diagnostics: bool = True,
                   max_steps: int | None = None,
                   track_limiter_entropy: bool = False) -> RunResult:
    out = RunResult(state=state)
    if track_limiter_entropy:
        integ.track_limiter_entropy = True
    if diagnostics:
        d0 = integ.diagnostics(state)
        out.mass_initial, out.entropy_initial = d0.mass, d0.entropy
    snaps = sorted(set(float(s) for s in snapshot_times if s <= final_time + 1e-12))
    next_snap = 0
    t = 0.0
    t_eps = 1e-12 * max(1.0, final_time)
    while t < final_time - t_eps:
        if max_steps is not None and out.steps >= max_steps:
            break
        dt = integ.compute_dt(state, cfl)
        t_event = final_time
        if next_snap < len(snaps):
            t_event = min(t_event, snaps[next_snap])
        hit_event = False
        if t + dt >= t_event - t_eps:
            dt = t_event - t
            hit_event = True
        rejections = 0
        while not integ.try_step(state, t, dt):
            dt *= 0.5
            hit_event = False
            rejections += 1
            if rejections >= 10:
                raise NumericalAbort(f"step rejected 10 times at t={t}")
        t = t_event if hit_event else t + dt
        out.steps += 1
        if diagnostics:
            d = integ.diagnostics(state)
            sd = StepDiagnostics(out.steps, t, dt, d.mass, d.entropy, d.min_h,
                                 integ.last_limited_count(), integ.last_max_eps(),
                                 integ.last_min_stage_h(), d.positivity_dt)
            if keep_series:
                out.series.append(sd)
        while next_snap < len(snaps) and t >= snaps[next_snap] - t_eps:
            next_snap += 1
    out.t = t
    if track_limiter_entropy:
        out.worst_limiter_entropy_jump = integ.worst_limiter_entropy_jump()
    return out


def run_simulation_device(integ: TimeIntegrator, state: State, final_time: float, cfl: float,
                          snapshot_times=(), keep_series: bool = True, diagnostics: bool = True,
                          max_steps: int | None = None, on_snapshot=None,
                          track_limiter_entropy: bool = False) -> RunResult:
    """run_simulation (driver.hpp:62-142) with the state resident on the device
    (SURVEY §8f row 1): the state is uploaded once and downloaded at snapshot
    events and at the end.  Each step is one `step_device` call: the three stages,
    then (queued behind them) the step diagnostics and the next compute_dt of the
    new state, read back with one host synchronisation.  Reject-and-halve rolls
    back on the device (W^n stays until a step is accepted; the next dt is only
    used after an accepted step, exactly where driver.hpp:92 recomputes it).
    Same decisions, same kernels, hence bitwise the same trajectory as
    run_simulation.  `on_snapshot(t, state)` receives the downloaded state."""
    out = RunResult(state=state)
    integ.upload(state)
    if track_limiter_entropy:
        integ.track_limiter_entropy = True
    if diagnostics:
        d0 = integ.diagnostics_device()
        out.mass_initial, out.entropy_initial = d0.mass, d0.entropy
    snaps = sorted(set(float(s) for s in snapshot_times if s <= final_time + 1e-12))
    next_snap = 0
    t = 0.0
    t_eps = 1e-12 * max(1.0, final_time)
    next_dt = None
    while t < final_time - t_eps:
        if max_steps is not None and out.steps >= max_steps:
            break
        dt = integ.compute_dt_device(cfl) if next_dt is None else next_dt
        t_event = final_time
        if next_snap < len(snaps):
            t_event = min(t_event, snaps[next_snap])
        hit_event = False
        if t + dt >= t_event - t_eps:
            dt = t_event - t
            hit_event = True
        rejections = 0
        while True:
            rep = integ.step_device(t, dt, cfl)
            if rep.info.accepted:
                break
            dt *= 0.5
            hit_event = False
            rejections += 1
            if rejections >= 10:
                raise NumericalAbort(f"step rejected 10 times at t={t}")
        next_dt = rep.next_dt
        t = t_event if hit_event else t + dt
        out.steps += 1
        if diagnostics:
            d = rep.diag
            sd = StepDiagnostics(out.steps, t, dt, d.mass, d.entropy, d.min_h,
                                 integ.last_limited_count(), integ.last_max_eps(),
                                 integ.last_min_stage_h(), d.positivity_dt)
            if keep_series:
                out.series.append(sd)
        while next_snap < len(snaps) and t >= snaps[next_snap] - t_eps:
            if on_snapshot is not None:
                integ.download(state)
                on_snapshot(snaps[next_snap], state)
            next_snap += 1
    integ.download(state)
    out.t = t
    if track_limiter_entropy:
        out.worst_limiter_entropy_jump = integ.worst_limiter_entropy_jump()
    return out
