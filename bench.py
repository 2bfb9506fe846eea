#!/usr/bin/env python3
"""Throughput benchmark: FP64 DOF-updates/s per SSPRK3 stage on the synthetic
curvilinear mesh of BASELINE.json config 5.

Workload (per GPU, weak scaling): build_wavy_mesh(N, 1000, 1000) periodic on [0,1]^2,
amp 0.04, bathymetry b = 0.1 + 0.05 sin(2 pi x) sin(2 pi y), smooth state
h = 1 + 0.1 sin(2 pi x) cos(2 pi y), hu = 0.3 h, hv = -0.2 h, g = 9.81, fixed
dt = 0.1 * compute_dt (no rejections; checked).  A bench "step" is one SSPRK3 time
step = 3 RK stages; value = 3 * DOFs * steps / time, DOFs = 3 K (N+1)^2
(bench.hpp:259).  Inputs (>= 5 GB of geometry+state) exceed the 126 MB L2, so no
flush is needed between iterations.

  python bench.py [--gpus N --steps K --warmup W] [--degree N] [--no-sweep] [--viscous]

On one GPU the line also carries the N=1..15 sweep (the BASELINE metric is "vs
N=1..15"): per degree the DOF-updates/s, the frozen roofline and its fraction.
  python bench.py --impl reference ...   # the reference CPU solver, same config
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 DOF-updates/sec per RK stage"
UNIT = "DOF-updates/s"
KX = int(os.environ.get("SWDG_BENCH_KX", "1000"))  # smaller meshes: debugging only


def frozen_counts(N: int, viscous: bool):
    """SURVEY §8(d) algorithmic bytes/flops per node and stage (frozen contract)."""
    n1 = N + 1
    bytes_node = 112.0 + (128.0 if viscous else 0.0)  # stage average (96, 120, 120)
    flops_elem = 51 * N * n1 * n1 + (12 * n1 + 35) * n1 * n1 + 276 * n1
    if viscous:
        flops_elem += (28 * n1 + 20) * n1 * n1
    return bytes_node, flops_elem / (n1 * n1)


def stage_kernel(N: int, viscous: bool) -> str:
    """the fused stage kernel(s) launch_fast_stage / launch_fast_visc_pre pick for
    this degree (kernels_fast.cu launch_n)"""
    n1 = N + 1
    if viscous:
        main = ("k_stage_node<%d,..,visc> (node per thread)" % n1 if n1 <= 3
                else "k_stage_hl<%d,..,visc> (half-line)" % n1)
        return main + " + k_visc_lines<%d> (viscous pre-kernel)" % n1
    if n1 <= 3:
        return "k_stage_elem<%d> (element per thread)" % n1
    if n1 == 4:
        return "k_stage_node<%d> (node per thread)" % n1
    return "k_stage_hl<%d> (half-line)" % n1


NCU_TRAFFIC_FILES = ("r02_ncu_traffic.json", "r01_ncu_traffic.json")


def ncu_traffic(N: int, viscous: bool):
    """DRAM bytes per launch of the stage kernel from the newest committed ncu
    --set full capture of this configuration (profiles/r0*_ncu_traffic.json; the
    captured launch is a stage-2 launch, which reads W^n: 120 B/node
    algorithmic, +128 viscous), or None"""
    for name in NCU_TRAFFIC_FILES:
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                d = json.load(f)
        except Exception:
            continue
        e = d.get("%s_N%d" % ("visc" if viscous else "inv", N))
        if e is not None:
            return float(e["dram_bytes_per_launch"]), name
    return None, None


def peaks():
    p = {"hbm_gbs": 6541.8, "fp64_tflops": 36.8, "hbm_src": "fallback", "fp64_src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p["hbm_gbs"] = float(m["hbm_gbs"])
        p["hbm_src"] = "MEASURED_PEAKS.json"
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as f:
            p["fp64_tflops"] = float(json.load(f)["dfma_tflops"])
            p["fp64_src"] = "profiles/r01_fp64_peak.json (DFMA microbenchmark on this pool)"
    except Exception:
        pass
    return p


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 2 + k and s[2 + k].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.samples[0][1]),
                "reasons": reasons, "samples": len(self.samples)}


def spec_for(N: int, kx: int = KX):
    from paper_1804_02221_b200 import swdg
    return swdg.structured_spec("wavy", N, kx, kx, periodic_x=True, periodic_y=True,
                                extra=0.04, bathy="smooth")


def run_config(N: int, viscous: bool):
    from paper_1804_02221_b200 import swdg
    visc = swdg.ViscosityConfig(False)
    if viscous:
        smin, smax = swdg.default_sigma_band(N)
        visc = swdg.ViscosityConfig(True, 0.1, smin, smax)
    return swdg.RunConfig(phys=swdg.PhysicsParams(9.81, 1e-4, 1e-8, 1.0), visc=visc,
                          mode=swdg.MODE_FAST)


def smooth_state(x, y):
    import numpy as np
    h = 1.0 + 0.1 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y)
    return h, 0.3 * h, -0.2 * h


def memcpy_d2d_gbs(nbytes: int = 4 << 30, reps: int = 10) -> float:
    """cudaMemcpy device-to-device bandwidth (read + write bytes / time), the
    paper's memory reference (bench.hpp:216-229 memcopy_baseline)"""
    import torch
    a = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    gbs = 2 * nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    del a, b
    torch.cuda.empty_cache()
    return gbs


def measure_gpu(N: int, steps: int, warmup: int, viscous: bool, rank: int, world: int,
                e2e_steps: int = 50):
    import numpy as np
    import torch
    from paper_1804_02221_b200 import swdg

    spec = spec_for(N)
    cfg = run_config(N, viscous)
    integ = swdg.TimeIntegrator.structured(spec, cfg, device=torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    integ.set_stream(stream.cuda_stream)
    nn = integ.mesh.n_nodes
    dofs = 3 * nn
    # initial state built on the host from the device-generated coordinates, pinned
    x, y = integ.geometry("x"), integ.geometry("y")
    host = [torch.empty(nn, dtype=torch.float64).pin_memory() for _ in range(3)]
    for hbuf, val in zip(host, smooth_state(x, y)):
        hbuf.numpy()[:] = val
    del x, y
    st = swdg.State(*(hb.numpy() for hb in host))
    integ.upload(st)
    dt = 0.1 * integ.compute_dt_device(0.5)

    # warm-up, then K timed device-resident steps: the metric as BASELINE.md
    # defines it (every step: 3 stages + the per-step dt and diagnostics
    # reductions on the device), then the same K steps stages-only (the stage
    # kernels' own time, what the roofline fraction is computed from)
    integ.run_steps(warmup, 0.0, dt, reductions=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = integ.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        ev0.record(stream)
        ok = integ.run_steps(steps, warmup * dt, dt, reductions=True)
        ev1.record(stream)
        torch.cuda.synchronize()
        launches = integ.launch_count() - l0
        # re-warm the stages-only path (captures its CUDA graph outside the timing)
        ok2 = integ.run_steps(4, (warmup + steps) * dt, dt)
        ev2.record(stream)
        ok2 = integ.run_steps(steps, (warmup + steps + 4) * dt, dt) and ok2
        ev3.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    ms_stages = ev2.elapsed_time(ev3)
    if not (ok and ok2):
        raise RuntimeError("a stage was rejected during the timed run (invalid measurement)")
    if world > 1:
        t = torch.tensor([ms, ms_stages], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, ms_stages = float(t[0].item()), float(t[1].item())

    # e2e through the public driver API (driver.run_simulation_device, the
    # run_simulation loop of driver.hpp:62-142 with the state resident on the
    # device): the initial state uploaded from pinned host memory, per step
    # compute_dt + try_step (reject-and-halve) + the step diagnostics read back,
    # the final state downloaded — all inside the timed region
    from paper_1804_02221_b200.driver import run_simulation_device
    e2e_s = e2e_host_s = float("nan")
    h2d = d2h = 0
    if e2e_steps > 0:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res_run = run_simulation_device(integ, st, 1e30, 0.05, max_steps=e2e_steps,
                                        keep_series=False)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / res_run.steps
        # per step: the step report (flags, diagnostics, next dt: ~100 B) + the
        # state upload/download amortised over the run
        h2d = (3 * nn * 8) // res_run.steps
        d2h = (3 * nn * 8) // res_run.steps + 128
        # the reference-API form (host State in, host State out every step)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(2):
            integ.try_step(st, s * dt, dt)
        torch.cuda.synchronize()
        e2e_host_s = (time.perf_counter() - t0) / 2
    res = dict(ms=ms, ms_stages=ms_stages, dofs=dofs, nn=nn, launches=launches,
               clocks=clk.summary(),
               e2e_s=e2e_s, h2d=h2d, d2h=d2h, e2e_host_s=e2e_host_s, e2e_steps=e2e_steps)
    integ.close()
    return res


def measure_gpu_distributed(N: int, steps: int, warmup: int, viscous: bool, rank: int,
                            world: int, e2e_steps: int = 2, halo: str = "nccl"):
    """Strong scaling over `world` ranks (one GPU each) of the same 1M-element mesh:
    rank r owns a band of element rows, generates its owned + ghost geometry on its
    device, and exchanges face-trace halos between stages: NCCL point-to-point, or
    (halo="ipc") direct peer-memory stores through CUDA IPC."""
    import numpy as np
    import torch
    from paper_1804_02221_b200 import swdg
    from paper_1804_02221_b200.distributed import (GpuPartition, GraphStepper, IpcExchanger,
                                                   TorchExchanger, compute_dt_distributed,
                                                   run_steps_distributed, try_step_distributed)

    spec = spec_for(N)
    cfg = run_config(N, viscous)
    dev = torch.cuda.current_device()
    b = GpuPartition.structured(spec, cfg, world, rank, dev)
    integ = b.integ
    stream = torch.cuda.current_stream()
    nn_local = integ.mesh.n_nodes
    x, y = integ.geometry("x"), integ.geometry("y")
    host = [torch.empty(nn_local, dtype=torch.float64).pin_memory() for _ in range(3)]
    for hbuf, val in zip(host, smooth_state(x, y)):
        hbuf.numpy()[:] = val
    st = swdg.State(*(hb.numpy() for hb in host))
    integ.upload(st)
    ex = IpcExchanger(b) if halo == "ipc" else TorchExchanger(b, "cuda")
    dt = 0.1 * compute_dt_distributed(b, ex, 0.5, N, cfg.phys)
    if halo == "ipc":  # the steps replay a captured graph (GraphStepper)
        stepper = GraphStepper(b, ex, 0.0, dt)
        stepper.begin()
        stepper.run(warmup)
        if not stepper.accepted():
            raise RuntimeError("a warm-up step was rejected")
    else:
        run_steps_distributed(b, ex, warmup, 0.0, dt)
    torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = integ.launch_count()
    r0 = stepper.replays if halo == "ipc" else 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        ev0.record(stream)
        if halo == "ipc":
            stepper.run(steps)
            ev1.record(stream)
            torch.cuda.synchronize()
            ok = stepper.accepted()
        else:
            ok = run_steps_distributed(b, ex, steps, warmup * dt, dt)
            ev1.record(stream)
            torch.cuda.synchronize()
    if not ok:
        raise RuntimeError("a step was rejected during the timed run (invalid measurement)")
    launches = integ.launch_count() - l0
    if halo == "ipc":  # kernels replayed from the graph are not API calls: count them
        launches += (stepper.replays - r0) * stepper.replay_launches
    t = torch.tensor([ev0.elapsed_time(ev1)], device="cuda", dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    # e2e: every rank uploads its partition from pinned host memory, steps, downloads
    torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for s in range(e2e_steps):
        integ.upload(st)
        try_step_distributed(b, ex, s * dt, dt)
        integ.download(st)
    torch.cuda.synchronize()
    e2e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    torch.distributed.all_reduce(e2e, op=torch.distributed.ReduceOp.MAX)
    np1 = (N + 1) ** 2
    return dict(ms=ms, dofs=3 * spec.kx * spec.ky * np1, nn=b.lm.n_owned * np1,
                launches=launches, clocks=clk.summary(), e2e_s=float(e2e.item()) / e2e_steps,
                h2d=3 * nn_local * 8, d2h=3 * nn_local * 8, halo_peers=len(b.plan.peers))


def cpu_reference(N: int, viscous: bool, budget_s: float = 15.0, kx: int = 64, steps=None,
                  warmup: int = 0):
    """The reference's own try_step (oracle/_ref, single-threaded like the reference) on
    a bounded sample of the C5 workload: the same mesh family, state and params on a
    kx*kx element patch.  Returns DOF-updates/s per stage."""
    import numpy as np
    from oracle import ref
    m = ref.build_mesh("wavy", N, kx, kx, periodic_x=True, periodic_y=True,
                       extra=0.04).bathymetry("smooth")
    smin = -(4.0 + 4.25 * np.log10(max(N, 1))) - 1.0
    p = ref.params(g=9.81, visc=viscous, epsilon0=0.1, sigma_min=smin, sigma_max=smin + 2.0)
    st = list(smooth_state(m.arrays["x"], m.arrays["y"]))
    dt = 0.1 * ref.compute_dt(m, p, st, 0.5)
    integ = ref.Integrator(m, p)
    L = ref.lib()
    runner = L.ref_runner_create(integ.h, *(ref.ptr(a) for a in st))
    if warmup:
        assert L.ref_runner_steps(runner, warmup, 0.0, dt) == warmup, "reference rejected a step"
    t0 = time.perf_counter()
    n = 0
    while True:
        acc = L.ref_runner_steps(runner, 1, (warmup + n) * dt, dt)
        assert acc == 1, "reference rejected a step"
        n += 1
        el = time.perf_counter() - t0
        if (steps is not None and n >= steps) or (steps is None and el >= budget_s):
            break
    L.ref_runner_free(runner)
    dofs = 3 * m.n_nodes
    return dict(value=3 * dofs * n / el, seconds=el, steps=n, kx=kx, dofs=dofs)


def _ref_worker(args):
    N, viscous, steps, budget, barrier, warmup = args
    barrier.wait()
    if steps is None:
        return cpu_reference(N, viscous, budget_s=budget, warmup=warmup)
    return cpu_reference(N, viscous, steps=steps, warmup=warmup)


def cpu_reference_parallel(N: int, viscous: bool, steps, procs: int, budget_s: float = 15.0,
                           warmup: int = 0):
    """P concurrent processes of cpu_reference (each its own patch, released
    together by a barrier): the aggregate DOF-updates/s of the host."""
    if procs <= 1:
        r = (cpu_reference(N, viscous, budget_s=budget_s, warmup=warmup) if steps is None
             else cpu_reference(N, viscous, steps=steps, warmup=warmup))
        r["procs"] = 1
        return r
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Manager() as man:
        barrier = man.Barrier(procs)
        with ctx.Pool(procs) as pool:
            rs = pool.map(_ref_worker, [(N, viscous, steps, budget_s, barrier, warmup)] * procs)
    secs = max(r["seconds"] for r in rs)
    return dict(value=sum(r["value"] for r in rs), seconds=secs, steps=rs[0]["steps"],
                kx=rs[0]["kx"], dofs=rs[0]["dofs"], procs=procs)


def cpu_model():
    """The host CPU as /proc/cpuinfo reports it (a VM may hide the marketing name:
    family/model/stepping and the vector ISA are added)."""
    info = {}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if ":" in line:
                    k, v = line.split(":", 1)
                    info.setdefault(k.strip(), v.strip())
    except Exception:
        return "unknown"
    flags = info.get("flags", "").split()
    isa = [f for f in ("avx512f", "avx2", "fma") if f in flags]
    return (f"{info.get('model name', 'unknown')} (family {info.get('cpu family', '?')}, model "
            f"{info.get('model', '?')}, stepping {info.get('stepping', '?')}; "
            f"{'/'.join(isa)}; {os.cpu_count()} logical CPUs)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--degree", type=int, default=7)
    ap.add_argument("--viscous", action="store_true")
    ap.add_argument("--no-sweep", dest="sweep", action="store_false",
                    help="skip the N=1..15 sweep (single GPU)")
    ap.add_argument("--distributed", action="store_true",
                    help="use the partitioned (NCCL halo) path even on one GPU")
    ap.add_argument("--halo", default="nccl", choices=["nccl", "ipc"],
                    help="partitioned path: halo exchange by NCCL or by CUDA IPC peer stores")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    N = args.degree
    workload = f"C5 synthetic wavy curvilinear mesh {KX}x{KX} ({KX * KX} elements) over " \
               f"{world} GPU(s), N={N}, " \
               f"{'viscous' if args.viscous else 'inviscid'} ES-DGSEM SSPRK3 stage"
    config = {"workload": workload, "elements": KX * KX, "elements_per_gpu": KX * KX // world,
              "degree": N,
              "viscosity": bool(args.viscous), "state": "smooth", "dt": "0.1*CFL fixed",
              "l2": "inputs > L2 (no flush needed)", "mode": "fast"}

    if args.impl == "reference":
        if world > 1 and rank != 0:
            return
        # the reference is single-threaded: on all host cores it is P independent
        # processes, each stepping its own patch of the workload at the same time
        # W untimed warm-up steps, then K timed steps (the same K, W as our arm)
        P = int(os.environ.get("SWDG_REF_PROCS", "0")) or max(1, len(os.sched_getaffinity(0)))
        r = cpu_reference_parallel(N, args.viscous, args.steps, P, warmup=args.warmup)
        config = dict(config, workload=(
            f"C5 synthetic wavy curvilinear mesh, N={N}, "
            f"{'viscous' if args.viscous else 'inviscid'} ES-DGSEM SSPRK3 stage: the reference "
            f"CPU solver on {r['procs']} concurrent {r['kx']}x{r['kx']}-element patches "
            f"({r['procs'] * r['kx'] ** 2} elements; the 1000x1000 mesh would take ~80 GB and "
            f"minutes per step on one core), {r['steps']} steps each"),
            elements=r["procs"] * r["kx"] ** 2, elements_per_gpu=None)
        line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
                "n_gpus": args.gpus, "steps": r["steps"], "warmup": args.warmup,
                "ms_per_step": 1e3 * r["seconds"] / r["steps"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config,
                "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["procs"],
                                 "kind": "reference",
                                 "sample": f"{r['procs']} concurrent single-threaded processes of the "
                                           f"reference TimeIntegrator::try_step (oracle/_ref), each on "
                                           f"a {r['kx']}x{r['kx']} patch of the same mesh family, "
                                           f"{r['steps']} steps, {r['seconds']:.1f} s",
                                 "cpu": cpu_model()},
                "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    # NCCL's version banner goes to stdout: keep the one-JSON-line contract
    os.environ["NCCL_DEBUG"] = os.environ.get("SWDG_NCCL_DEBUG", "WARN")
    import torch
    distributed = world > 1 or args.distributed
    if distributed:
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        if not torch.distributed.is_initialized():
            if "MASTER_ADDR" not in os.environ:  # single-process check of the path
                os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29531", RANK="0",
                                  WORLD_SIZE="1")
            torch.distributed.init_process_group("nccl")
        r = measure_gpu_distributed(N, args.steps, args.warmup, args.viscous, rank, world,
                                    halo=args.halo)
        config.update(parallelism=f"element partition over {world} GPU(s), "
                                  f"{'CUDA IPC peer-memory' if args.halo == 'ipc' else 'NCCL'} halos",
                      scaling="strong: the same 1M-element mesh for every N")
    else:
        r = measure_gpu(N, args.steps, args.warmup, args.viscous, rank, world)
    # value: DOF-updates of the whole job per second, per-step dt + diagnostics
    # amortised over the step's 3 stages (BASELINE.md "Metric")
    stage_s = r["ms"] * 1e-3 / (3 * args.steps)
    value = (r["dofs"] if distributed else world * r["dofs"]) / stage_s
    # the stage kernels alone (roofline): stages-only timing of the same steps
    kstage_s = r.get("ms_stages", r["ms"]) * 1e-3 / (3 * args.steps)
    value_stages = (r["dofs"] if distributed else world * r["dofs"]) / kstage_s
    bytes_node, flops_node = frozen_counts(N, args.viscous)
    pk = peaks()
    achieved_gbs = bytes_node * r["nn"] / kstage_s / 1e9
    achieved_tf = flops_node * r["nn"] / kstage_s / 1e12
    traffic, traffic_src = ncu_traffic(N, args.viscous)
    stage2_bytes = (120.0 + (128.0 if args.viscous else 0.0)) * r["nn"]
    roof_dofs = min(pk["hbm_gbs"] * 1e9 / (bytes_node / 3.0),
                    pk["fp64_tflops"] * 1e12 / (flops_node / 3.0))
    bound = "hbm" if pk["hbm_gbs"] * 1e9 / (bytes_node / 3.0) <= \
        pk["fp64_tflops"] * 1e12 / (flops_node / 3.0) else "fp64"
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["ms"] / args.steps, "higher_is_better": True,
        # the same 1M-element mesh at every GPU count: N=1 is the first point of
        # the strong-scaling series (BASELINE config 5)
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config,
        "value_stages_only": value_stages,
        "ms_per_step_stages_only": r.get("ms_stages", r["ms"]) / args.steps,
        "roofline": {
            "bound": bound,
            "achieved": achieved_gbs if bound == "hbm" else achieved_tf,
            "peak": pk["hbm_gbs"] if bound == "hbm" else pk["fp64_tflops"],
            "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
            "frac": (achieved_gbs / pk["hbm_gbs"]) if bound == "hbm"
            else achieved_tf / pk["fp64_tflops"],
            "traffic": traffic,
            "traffic_unit": "bytes per launch (ncu dram__bytes_read+write of one stage-2 "
                            "launch, cold L2)",
            "traffic_source": traffic_src and "profiles/" + traffic_src,
            "traffic_vs_same_stage_algorithmic": traffic / stage2_bytes if traffic else None,
            "algorithmic_bytes_per_launch": bytes_node * r["nn"],
            "algorithmic_bytes_stage2_launch": stage2_bytes,
            "timing": "achieved = stage-average algorithmic bytes / the stage kernels' own "
                      "time per stage (CUDA events over K stages-only steps)",
            "kernel": stage_kernel(N, args.viscous),
            "algorithmic_bytes_per_node": bytes_node, "algorithmic_flops_per_node": flops_node,
            "achieved_fp64_tflops": achieved_tf, "achieved_gbs": achieved_gbs,
            "roof_dof_per_s": roof_dofs, "frac_of_roof": value_stages / world / roof_dofs,
            "peak_sources": {"hbm": pk["hbm_src"], "fp64": pk["fp64_src"]},
        },
        "clocks": r["clocks"],
        "gpu_launches": r["launches"],
        "e2e": {"value": (1 if distributed else world) * 3 * r["dofs"] / r["e2e_s"], "unit": UNIT,
                "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"],
                "path": ("per rank: swdg_gpu_upload_state + split-step C ABI with halo exchanges + "
                         "download (pinned)") if distributed else
                        (f"driver.run_simulation_device, {r['e2e_steps']} steps: state uploaded "
                         "from pinned memory once, per step one swdg_gpu_step_device (3 stages + "
                         "diagnostics + next compute_dt, one D2H of the step report), final "
                         "state downloaded; bytes amortised per step"),
                **({} if distributed else {
                    "host_state_per_step": {
                        "value": 3 * r["dofs"] / r["e2e_host_s"], "unit": UNIT,
                        "h2d_bytes_per_step": 3 * r["nn"] * 8,
                        "d2h_bytes_per_step": 3 * r["nn"] * 8,
                        "path": "TimeIntegrator.try_step with a host State (upload + step + "
                                "download every step, PCIe-bound)"}})},
    }
    if distributed:
        out["halo_peers_rank0"] = r.get("halo_peers")
    if rank == 0 and not distributed:
        out["roofline"]["memcpy_d2d_gbs"] = memcpy_d2d_gbs()
    if rank == 0:
        procs = int(os.environ.get("SWDG_REF_PROCS", "0")) or max(1, len(os.sched_getaffinity(0)))
        cb = cpu_reference_parallel(N, args.viscous, None, procs, budget_s=args.cpu_budget)
        c1 = cpu_reference(N, args.viscous, budget_s=min(5.0, args.cpu_budget))
        out["cpu_baseline"] = {
            "value": cb["value"], "unit": UNIT, "cores": cb["procs"], "kind": "reference",
            "sample": f"{cb['procs']} concurrent single-threaded processes of oracle/_ref "
                      f"TimeIntegrator::try_step, each on a {cb['kx']}x{cb['kx']} patch of the "
                      f"same mesh family, {cb['steps']} steps in {cb['seconds']:.1f} s",
            "value_1core": c1["value"],
            "sample_1core": f"one process, {c1['kx']}x{c1['kx']} patch, {c1['steps']} steps in "
                            f"{c1['seconds']:.1f} s (the reference is single-threaded)",
            "cpu": cpu_model()}
        if args.sweep and not distributed:
            sweep, sweep_s, roof, frac = {}, {}, {}, {}
            for n in range(1, 16):
                if args.viscous and n < 2:
                    continue
                if n == N:
                    v, vs = value, value_stages
                else:
                    ks = max(3, args.steps // 4)
                    rr = measure_gpu(n, ks, 3, args.viscous, rank, 1, e2e_steps=0)
                    v = rr["dofs"] / (rr["ms"] * 1e-3 / (3 * ks))
                    vs = rr["dofs"] / (rr["ms_stages"] * 1e-3 / (3 * ks))
                bn, fn = frozen_counts(n, args.viscous)
                rf = min(pk["hbm_gbs"] * 1e9 / (bn / 3.0), pk["fp64_tflops"] * 1e12 / (fn / 3.0))
                sweep[n], sweep_s[n], roof[n], frac[n] = v, vs, rf, vs / rf
            # the metric (per-step dt + diagnostics amortised) and the stage kernels
            # alone; the roofline fraction is the stage kernels' (frozen bytes/flops)
            out["sweep_dof_per_s_by_degree"] = sweep
            out["sweep_dof_per_s_stages_only_by_degree"] = sweep_s
            out["sweep_roof_dof_per_s_by_degree"] = roof
            out["sweep_frac_of_roof_by_degree"] = frac
        print(json.dumps(out), flush=True)
    if distributed:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
