"""Multi-GPU decomposition on the CPU: the partitioner and halo plans are pure,
deterministic functions of the face list, and a partitioned run of the oracle —
in one process (loopback) and across two gloo ranks — reproduces the global run
bitwise (the same exchange schedule drives the GPU partitions)."""
import os

import numpy as np
import pytest

from oracle import port, ref
from paper_1804_02221_b200 import partition as part
from paper_1804_02221_b200.distributed import (LoopbackExchanger, TorchExchanger,
                                               try_step_distributed, try_step_loopback)
from tests.helpers import beq, build, random_state, reversed_mesh, scenario_params, smooth_state
from tests.port_partition import PortPartition

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def test_ranges_and_owner_are_inverse():
    for K in (1, 7, 100, 1001):
        for P in (1, 2, 3, 8):
            if P > K:
                continue
            rs = part.ranges(K, P)
            assert rs[0][0] == 0 and rs[-1][1] == K
            e = np.arange(K)
            o = part.owner(e, K, P)
            for r, (a, b) in enumerate(rs):
                assert np.all(o[a:b] == r)


@pytest.mark.parametrize("name,P", [("wavy_N4", 2), ("wavy_N4", 3), ("dam_N4", 4),
                                    ("cart_N3_walls", 2)])
def test_plan_consistency(name, P):
    m = build(name)
    plans = [part.build_plan(m.faces, m.n_elem, m.degree, P, r) for r in range(P)]
    n1 = m.degree + 1
    # every global face appears in the local lists of exactly the ranks it touches
    seen = np.zeros(len(m.faces), int)
    for gids, n_owned, lf, ords, plan in plans:
        seen[ords] += 1
        assert np.all(np.diff(ords) > 0), "local faces keep the global order"
        # local ids resolve back to the global faces
        for f, o in zip(lf, ords):
            g = m.faces[o]
            assert gids[f[0]] == g[0] and f[1] == g[1]
            if g[5] == 0:
                assert gids[f[2]] == g[2] and f[3] == g[3]
    for fi, f in enumerate(m.faces):
        ranks = {int(part.owner(f[0], m.n_elem, P))}
        if f[5] == 0:
            ranks.add(int(part.owner(f[2], m.n_elem, P)))
        assert seen[fi] == len(ranks)
    # pairwise: what r sends to s is what s expects from r
    for r in range(P):
        for s in plans[r][4].peers:
            assert len(plans[r][4].send_idx[s]) == len(plans[s][4].recv_idx[r])
            assert len(plans[r][4].send_idx[s]) % n1 == 0
    # deterministic
    again = part.build_plan(m.faces, m.n_elem, m.degree, P, P - 1)
    assert np.array_equal(again[2], plans[-1][2])


def _global_run(m, p, st, dt, steps):
    s = [a.copy() for a in st]
    for k in range(steps):
        info = port.try_step(m, p, s, k * dt, dt)
        assert info.accepted
    return s


def _gather(lms, backends, n_nodes):
    out = [np.zeros(n_nodes) for _ in range(3)]
    for lm, b in zip(lms, backends):
        np_ = lm.n1 * lm.n1
        sel = (lm.global_ids[: lm.n_owned, None] * np_ + np.arange(np_)).ravel()
        for o, w in zip(out, b.W):
            o[sel] = w[: lm.n_owned * np_]
    return out


@pytest.mark.parametrize("name,P,visc", [("wavy_N4", 2, False), ("wavy_N4", 3, True),
                                         ("dam_N4", 4, True), ("cart_N3_walls", 2, True),
                                         ("wavy_N7", 3, True)])
def test_loopback_partitioned_oracle_is_bitwise(name, P, visc):
    m = build(name)
    N = m.degree
    smin = -(4.0 + 4.25 * np.log10(N)) - 1.0
    p = ref.params(g=9.81, visc=visc, epsilon0=0.1, sigma_min=smin, sigma_max=smin + 2.0)
    st = random_state(m.n_nodes, np.random.default_rng(2), h=(0.5, 1.5), vel=0.5)
    dt = 0.3 * port.compute_dt(m, p, st, 0.5)
    want = _global_run(m, p, st, dt, 3)
    lms = [part.local_mesh(m, P, r) for r in range(P)]
    bs = [PortPartition(lm, p) for lm in lms]
    for lm, b in zip(lms, bs):
        b.upload(part.scatter_state(st, lm))
    ex = LoopbackExchanger(bs, lambda n: np.zeros(n))
    for k in range(3):
        assert try_step_loopback(bs, ex, k * dt, dt)
    assert beq(_gather(lms, bs, m.n_nodes), want)


def test_loopback_reversed_faces():
    m, _, _ = reversed_mesh(build("wavy_N4"))
    p = ref.params(g=9.81, visc=True, epsilon0=0.1, sigma_min=-6.5, sigma_max=-5.0)
    st = smooth_state(m, 0.2)
    dt = 0.3 * port.compute_dt(m, p, st, 0.5)
    want = _global_run(m, p, st, dt, 2)
    lms = [part.local_mesh(m, 3, r) for r in range(3)]
    bs = [PortPartition(lm, p) for lm in lms]
    for lm, b in zip(lms, bs):
        b.upload(part.scatter_state(st, lm))
    ex = LoopbackExchanger(bs, lambda n: np.zeros(n))
    for k in range(2):
        assert try_step_loopback(bs, ex, k * dt, dt)
    assert beq(_gather(lms, bs, m.n_nodes), want)


@pytest.mark.parametrize("name,P,visc", [("wavy_N4", 3, True), ("cart_N3_walls", 2, True)])
def test_loopback_step_reports_match_global(name, P, visc):
    """SURVEY §8(e) per-step reductions: mass/entropy/n_limited sums, min h /
    positivity / min stage h minima, max eps maximum over the partitions equal the
    single-mesh step report (sums to rounding: a different summation order)."""
    from paper_1804_02221_b200.distributed import step_report_loopback
    m = build(name)
    N = m.degree
    smin = -(4.0 + 4.25 * np.log10(N)) - 1.0
    p = ref.params(g=9.81, visc=visc, epsilon0=0.1, sigma_min=smin, sigma_max=smin + 2.0)
    st = random_state(m.n_nodes, np.random.default_rng(4), h=(0.0, 1.5), vel=0.5, dry_prob=0.1)
    dt = 0.1 * port.compute_dt(m, p, st, 0.5)
    lms = [part.local_mesh(m, P, r) for r in range(P)]
    bs = [PortPartition(lm, p) for lm in lms]
    for lm, b in zip(lms, bs):
        b.upload(part.scatter_state(st, lm))
    ex = LoopbackExchanger(bs, lambda n: np.zeros(n))
    s = [a.copy() for a in st]
    for k in range(3):
        info = port.try_step(m, p, s, k * dt, dt)
        assert try_step_loopback(bs, ex, k * dt, dt) == bool(info.accepted)
        if not info.accepted:  # the driver reads the report of accepted steps only
            continue
        rep = step_report_loopback(bs, ex)
        d = port.diagnostics(m, p, s)
        assert rep["n_limited"] == info.n_limited
        assert rep["min_stage_h"] == info.min_stage_h
        assert rep["max_eps"] == info.max_eps
        assert rep["min_h"] == d.min_h
        assert rep["positivity_dt"] == d.positivity_dt
        assert abs(rep["mass"] - d.mass) <= 1e-13 * abs(d.mass)
        assert abs(rep["entropy"] - d.entropy) <= 1e-13 * abs(d.entropy)


def _gloo_worker(rank, world, port_no, result_path):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_no}", rank=rank,
                            world_size=world)
    m, st = ref.scenario_mesh("wetdry_dambreak", 8, 8, 3)
    p, cfg = scenario_params("wetdry_dambreak")
    dt = port.compute_dt(m, p, st, cfg["cfl"])
    lm = part.local_mesh(m, world, rank)
    b = PortPartition(lm, p)
    b.upload(part.scatter_state(st, lm))
    ex = TorchExchanger(b, "cpu")
    from paper_1804_02221_b200.distributed import step_report_distributed
    acc, reps = [], []
    for k in range(4):
        acc.append(try_step_distributed(b, ex, k * dt, dt))
        reps.append(step_report_distributed(b, ex))
    np_ = lm.n1 * lm.n1
    mine = np.stack([w[: lm.n_owned * np_] for w in b.W])
    gathered = [None] * world
    dist.all_gather_object(gathered, (lm.global_ids[: lm.n_owned].tolist(), mine, acc, reps))
    if rank == 0:
        np.save(result_path, np.array(gathered, dtype=object), allow_pickle=True)
    dist.destroy_process_group()


def test_gloo_two_ranks_bitwise(tmp_path):
    """world_size-2 gloo run of the partitioned stepping (wet/dry dam break with
    viscosity and limiter) equals the single-process oracle run bitwise."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    path = os.path.join(tmp_path, "res.npy")
    mp.spawn(_gloo_worker, args=(2, port_no, path), nprocs=2, join=True)
    res = np.load(path, allow_pickle=True)
    m, st = ref.scenario_mesh("wetdry_dambreak", 8, 8, 3)
    p, cfg = scenario_params("wetdry_dambreak")
    dt = port.compute_dt(m, p, st, cfg["cfl"])
    want = [a.copy() for a in st]
    acc_ref, infos = [], []
    for k in range(4):
        info = port.try_step(m, p, want, k * dt, dt)
        acc_ref.append(bool(info.accepted))
        infos.append((info.n_limited, info.min_stage_h, port.diagnostics(m, p, want)))
    np_ = m.n1 * m.n1
    got = [np.zeros(m.n_nodes) for _ in range(3)]
    for gids, mine, acc, reps in res:
        assert acc == acc_ref
        for rep, (nl, msh, d) in zip(reps, infos):  # the same report on every rank
            assert rep["n_limited"] == nl and rep["min_stage_h"] == msh
            assert rep["min_h"] == d.min_h and rep["positivity_dt"] == d.positivity_dt
            assert abs(rep["mass"] - d.mass) <= 1e-13 * abs(d.mass)
        sel = (np.array(gids)[:, None] * np_ + np.arange(np_)).ravel()
        for j in range(3):
            got[j][sel] = mine[j]
    assert beq(got, want)


@pytest.mark.parametrize("kx,ky,P", [(8, 12, 3), (10, 10, 2), (6, 20, 4)])
def test_interior_range_is_halo_free(kx, ky, P):
    """interior_range (the part of a stage that runs while the halo is in flight):
    no element in [lo, hi) has a face to a ghost, and for a band partition it is the
    band minus its first and last element row."""
    from paper_1804_02221_b200 import swdg
    faces = swdg.structured_faces(kx, ky, True, True)
    for r in range(P):
        _, n_owned, lf, _, _ = part.build_plan(faces, kx * ky, 3, P, r)
        lo, hi = part.interior_range(lf, n_owned)
        f = np.asarray(lf).reshape(-1, 6)
        inter = f[:, 5] == 0
        for a, b in ((f[:, 0], f[:, 2]), (f[:, 2], f[:, 0])):
            sel = inter & (a >= lo) & (a < hi)
            assert not np.any(b[sel] >= n_owned)
        if n_owned // kx >= 3:
            assert (lo, hi) == (kx, n_owned - kx)


def test_bench_frozen_roofline():
    """bench.py's frozen counts: 112 B/node, the flop model, and the
    roof per degree (HBM-bound up to N=8, FP64 above, 1.10e11 DOF/s at N=15)."""
    import bench
    b, f = bench.frozen_counts(7, False)
    assert b == 112.0 and abs(f / 3 - 174.2) < 0.1
    b, f = bench.frozen_counts(15, False)
    assert abs(f / 3 - 336.4) < 0.1
    roof = lambda n: min(6541.8e9 / (bench.frozen_counts(n, False)[0] / 3),
                         36.8e12 / (bench.frozen_counts(n, False)[1] / 3))
    assert abs(roof(7) - 1.752e11) < 1e9 and abs(roof(15) - 1.094e11) < 1e9
    assert "half-line" in bench.stage_kernel(7, False)
    assert "element" in bench.stage_kernel(1, False)
