"""Two ranks over NCCL, one B200 each (skipped on boxes with fewer than 2 GPUs):
the partitioned step of paper_1804_02221_b200.distributed with real NCCL halo
exchanges -- interior/boundary overlap, the SM reserve of the interior launch --
and the §8(e) per-step reductions reproduce the single-GPU run: exact mode
bitwise (hence the reference), fast mode bitwise against the single-GPU fast run
of the same partition-free kernels is not required (different launch ranges), so
fast mode is held to 1e-12 normwise after the steps."""
import os
import socket

import numpy as np
import pytest

from oracle import ref
from tests.helpers import beq, normwise, scenario_params

pytestmark = [pytest.mark.gpu]


def _gpus():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


SCEN = ("wetdry_dambreak", 12, 3)  # wet/dry fronts, viscosity, limiter


def _worker(rank, world, port_no, mode, path):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port_no}", rank=rank,
                            world_size=world)
    from paper_1804_02221_b200 import partition as part
    from paper_1804_02221_b200 import swdg
    from paper_1804_02221_b200.distributed import (GpuPartition, TorchExchanger,
                                                   step_report_distributed,
                                                   try_step_distributed)
    sid, k, N = SCEN
    m, st = ref.scenario_mesh(sid, k, k, N)
    p, c = scenario_params(sid, N)
    cfg = swdg.RunConfig(phys=swdg.PhysicsParams(p.g, p.h_tol, p.h_des, p.h_ref),
                         visc=swdg.ViscosityConfig(bool(p.visc_enabled), p.epsilon0,
                                                   p.sigma_min, p.sigma_max),
                         limiter_enabled=bool(p.limiter_enabled), mode=mode)
    lm = part.local_mesh(m, world, rank)
    b = GpuPartition(lm, cfg, device=rank)
    b.upload(part.scatter_state(st, lm))
    ex = TorchExchanger(b, f"cuda:{rank}")
    dt = ref.compute_dt(m, p, st, c["cfl"])
    acc, reps = [], []
    for s in range(4):
        acc.append(try_step_distributed(b, ex, s * dt, dt))
        reps.append(step_report_distributed(b, ex) if acc[-1] else None)
    np_ = lm.n1 * lm.n1
    mine = np.stack([w[: lm.n_owned * np_] for w in b.download()])
    out = [None] * world
    dist.all_gather_object(out, (lm.global_ids[: lm.n_owned].tolist(), mine, acc, reps))
    if rank == 0:
        np.save(path, np.array(out, dtype=object), allow_pickle=True)
    dist.destroy_process_group()


@pytest.mark.skipif(_gpus() < 2, reason="needs two CUDA devices (one per rank)")
@pytest.mark.parametrize("mode", [0, 1])
def test_two_ranks_nccl(tmp_path, mode):
    import torch.multiprocessing as mp
    from paper_1804_02221_b200 import swdg
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    path = os.path.join(tmp_path, "res.npy")
    mp.spawn(_worker, args=(2, port_no, mode, path), nprocs=2, join=True)
    res = np.load(path, allow_pickle=True)
    sid, k, N = SCEN
    m, st = ref.scenario_mesh(sid, k, k, N)
    p, c = scenario_params(sid, N)
    cfg = swdg.RunConfig(phys=swdg.PhysicsParams(p.g, p.h_tol, p.h_des, p.h_ref),
                         visc=swdg.ViscosityConfig(bool(p.visc_enabled), p.epsilon0,
                                                   p.sigma_min, p.sigma_max),
                         limiter_enabled=bool(p.limiter_enabled), mode=mode)
    single = swdg.TimeIntegrator(m, cfg)
    dt = ref.compute_dt(m, p, st, c["cfl"])
    want = swdg.State(*[a.copy() for a in st])
    acc_ref = [single.try_step(want, s * dt, dt) for s in range(4)]
    np_ = m.n1 * m.n1
    got = [np.zeros(m.n_nodes) for _ in range(3)]
    for gids, mine, acc, reps in res:
        assert acc == acc_ref
        sel = (np.array(gids)[:, None] * np_ + np.arange(np_)).ravel()
        for j in range(3):
            got[j][sel] = mine[j]
    if mode == 0:
        assert beq(got, want.arrays())
        d = ref.diagnostics(m, p, want.arrays())
        last = res[0][3][-1]
        assert last["min_h"] == d.min_h and last["positivity_dt"] == d.positivity_dt
        assert abs(last["mass"] - d.mass) <= 1e-13 * abs(d.mass)
    else:
        assert normwise(got, want.arrays()) <= 1e-12
