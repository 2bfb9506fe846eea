"""Two processes exchanging halos through peer memory (IpcExchanger: CUDA IPC
mailboxes, device-side flags, no NCCL) reproduce the single-GPU run.  Both ranks
share cuda:0 (one B200 per gpurun box): the same kernels, handles and flags as
between GPUs, the stores landing in the other process's device memory instead of
crossing NVLink.  Exact mode bitwise (hence the reference); fast mode bitwise
against the single-GPU fast run, as for the in-process partitions."""
import os
import socket

import numpy as np
import pytest

from oracle import ref
from tests.conftest import gpu_available
from tests.helpers import beq, scenario_params

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _cfg(p, mode):
    from paper_1804_02221_b200 import swdg
    return swdg.RunConfig(phys=swdg.PhysicsParams(p.g, p.h_tol, p.h_des, p.h_ref),
                          visc=swdg.ViscosityConfig(bool(p.visc_enabled), p.epsilon0,
                                                    p.sigma_min, p.sigma_max),
                          limiter_enabled=bool(p.limiter_enabled), mode=mode)


def _worker(rank, world, port_no, scen, mode, steps, path):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_no}", rank=rank,
                            world_size=world)
    from paper_1804_02221_b200 import partition as part
    from paper_1804_02221_b200.distributed import (GpuPartition, IpcExchanger,
                                                   step_report_distributed,
                                                   try_step_distributed)
    sid, k, N, visc = scen
    m, st = ref.scenario_mesh(sid, k, k, N)
    p, c = scenario_params(sid, N, **({} if visc else {"visc_enabled": 0.0}))
    lm = part.local_mesh(m, world, rank)
    b = GpuPartition(lm, _cfg(p, mode), device=0)
    b.upload(part.scatter_state(st, lm))
    ex = IpcExchanger(b, timeout_s=20.0)
    dt = ref.compute_dt(m, p, st, c["cfl"])
    acc, reps = [], []
    for s in range(steps):
        acc.append(try_step_distributed(b, ex, s * dt, dt))
        reps.append(step_report_distributed(b, ex) if acc[-1] else None)
    np_ = lm.n1 * lm.n1
    mine = np.stack([w[: lm.n_owned * np_] for w in b.download()])
    out = [None] * world
    dist.all_gather_object(out, (lm.global_ids[: lm.n_owned].tolist(), mine, acc, reps,
                                 b.has_interior, ex.seq))
    if rank == 0:
        np.save(path, np.array(out, dtype=object), allow_pickle=True)
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("scen", [("wetdry_dambreak", 12, 3, True),
                                  ("oscillating_lake", 16, 4, False)])
def test_two_processes_peer_memory_halo(tmp_path, mode, scen):
    import torch.multiprocessing as mp
    from paper_1804_02221_b200 import swdg
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    path = os.path.join(tmp_path, "res.npy")
    steps = 4
    mp.spawn(_worker, args=(2, port_no, scen, mode, steps, path), nprocs=2, join=True)
    res = np.load(path, allow_pickle=True)
    sid, k, N, visc = scen
    m, st = ref.scenario_mesh(sid, k, k, N)
    p, c = scenario_params(sid, N, **({} if visc else {"visc_enabled": 0.0}))
    single = swdg.TimeIntegrator(m, _cfg(p, mode))
    dt = ref.compute_dt(m, p, st, c["cfl"])
    want = swdg.State(*[a.copy() for a in st])
    acc_ref = [single.try_step(want, s * dt, dt) for s in range(steps)]
    np_ = m.n1 * m.n1
    got = [np.zeros(m.n_nodes) for _ in range(3)]
    for gids, mine, acc, reps, has_interior, seq in res:
        assert acc == acc_ref
        assert has_interior  # the overlapped schedule (interior during the exchange) ran
        # state exchange per stage (+ flux pairs when viscous) + one per step report
        assert seq == steps * 3 * (2 if visc else 1) + sum(acc)
        sel = (np.array(gids)[:, None] * np_ + np.arange(np_)).ravel()
        for j in range(3):
            got[j][sel] = mine[j]
    assert beq(got, want.arrays())
    d = single.diagnostics(want)
    last = res[0][3][-1]
    assert last["min_h"] == d.min_h
    assert abs(last["mass"] - d.mass) <= 1e-13 * abs(d.mass)


def _graph_worker(rank, world, port_no, N, visc, steps, path):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_no}", rank=rank,
                            world_size=world)
    from paper_1804_02221_b200 import swdg
    from paper_1804_02221_b200.distributed import (GpuPartition, IpcExchanger,
                                                   run_steps_distributed_graph)
    spec, cfg, dt = _graph_case(N, visc)
    b = GpuPartition.structured(spec, cfg, world, rank, 0)
    x, y = b.integ.geometry("x"), b.integ.geometry("y")
    b.upload([1.0 + 0.1 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y),
              0.3 * np.ones_like(x), -0.2 * np.ones_like(x)])
    ex = IpcExchanger(b, timeout_s=20.0)
    if steps == 5:
        ok = run_steps_distributed_graph(b, ex, steps, 0.0, dt)
    else:  # several run() calls with odd counts: the ping-pong must stay aligned
        from paper_1804_02221_b200.distributed import GraphStepper
        stp = GraphStepper(b, ex, 0.0, dt)
        stp.begin()
        for n in (4, 3, 1, 2):
            stp.run(n)
        ok = stp.accepted()
    np_ = (N + 1) ** 2
    n_own = b.lm.n_owned
    mine = np.stack([w[: n_own * np_] for w in b.download()])
    out = [None] * world
    dist.all_gather_object(out, (b.lm.global_ids[:n_own].tolist(), mine, ok, ex.seq))
    if rank == 0:
        np.save(path, np.array(out, dtype=object), allow_pickle=True)
    dist.destroy_process_group()


def _graph_case(N, visc):
    from paper_1804_02221_b200 import swdg
    v = swdg.ViscosityConfig(False)
    if visc:
        smin, smax = swdg.default_sigma_band(N)
        v = swdg.ViscosityConfig(True, 0.1, smin, smax)
    cfg = swdg.RunConfig(phys=swdg.PhysicsParams(9.81), visc=v, mode=swdg.MODE_FAST)
    spec = swdg.structured_spec("wavy", N, 24, 24, periodic_x=True, periodic_y=True,
                                bathy="smooth")
    return spec, cfg, 5e-5


@pytest.mark.parametrize("N,visc,steps", [(4, False, 5), (3, True, 5), (4, False, 10)])
def test_two_processes_graph_replayed_steps(tmp_path, N, visc, steps):
    """run_steps_distributed_graph: one eager step, two captured steps replayed twice
    (the device-resident sequence base advancing per replay): the same state as the
    single-GPU fixed-dt stepping of the same mesh."""
    import torch.multiprocessing as mp
    from paper_1804_02221_b200 import swdg
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    path = os.path.join(tmp_path, "res.npy")
    mp.spawn(_graph_worker, args=(2, port_no, N, visc, steps, path), nprocs=2, join=True)
    res = np.load(path, allow_pickle=True)
    spec, cfg, dt = _graph_case(N, visc)
    single = swdg.TimeIntegrator.structured(spec, cfg)
    x, y = single.geometry("x"), single.geometry("y")
    single.upload(swdg.State(1.0 + 0.1 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y),
                             0.3 * np.ones_like(x), -0.2 * np.ones_like(x)))
    assert single.run_steps(steps, 0.0, dt)
    want = [np.empty(single.mesh.n_nodes) for _ in range(3)]
    single.download(swdg.State(*want))
    np_ = (N + 1) ** 2
    got = [np.zeros(single.mesh.n_nodes) for _ in range(3)]
    per_step = 3 * (2 if visc else 1)
    for gids, mine, ok, seq in res:
        assert ok
        assert seq == steps * per_step
        sel = (np.array(gids)[:, None] * np_ + np.arange(np_)).ravel()
        for j in range(3):
            got[j][sel] = mine[j]
    assert beq(got, want)


def test_flag_wait_times_out_instead_of_hanging():
    """A peer that never raises its flag: the device-side wait gives up after its
    timeout, the stream moves on, and halo_status reports it (once)."""
    import time
    from paper_1804_02221_b200 import partition as part
    from paper_1804_02221_b200.distributed import GpuPartition
    sid, k, N = "oscillating_lake", 8, 3
    m, st = ref.scenario_mesh(sid, k, k, N)
    p, _ = scenario_params(sid, N, visc_enabled=0.0)
    lm = part.local_mesh(m, 2, 0)
    b = GpuPartition(lm, _cfg(p, 1))
    base, handle = b.ipc_alloc(4 * 8)
    assert len(handle) == 64
    t0 = time.perf_counter()
    b.wait_flags(base, 2, 1, 0.2)  # nobody will store 1 there
    assert b.halo_timed_out()
    assert time.perf_counter() - t0 < 10.0
    assert not b.halo_timed_out()  # the report is cleared
    b.wait_flags(base, 2, 0, 0.2)  # already satisfied (flags start at 0)
    assert not b.halo_timed_out()
