"""Partitioned SSPRK3 stepping across ranks: one element partition per
GPU, face-trace halos exchanged between stages, one flag reduction per step.

    step_begin
    for k in 0..2:
        exchange stage-k input state at the halo face nodes      (3 doubles / node)
        stage_visc k            (viscosity on: eps, BR1, flux pairs)
        exchange the viscous flux pairs at the halo face nodes   (4 doubles / node)
        stage_run k             (fused stage kernel, limiter, reject flags)
    all-reduce (reject, abort) -> step_commit(accept)

The stepping logic is backend-agnostic: `GpuPartition` drives the sm_100a kernels
through the split-step C ABI; tests drive the same loop with the CPU oracle.  The
exchanger is torch.distributed point-to-point (NCCL between GPUs, gloo on CPU),
direct peer-memory stores through CUDA IPC (`IpcExchanger`), or an in-process
loopback for several partitions in one process.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import swdg
from .partition import LocalMesh


class Backend:
    """Interface of one rank's partition."""
    visc: bool
    plan = None  # HaloPlan

    def step_begin(self): ...
    def pack(self, what: int, k: int, buf): ...
    def unpack(self, what: int, k: int, buf): ...
    def stage_visc(self, k: int, t: float, dt: float): ...
    def stage_run(self, k: int, t: float, dt: float): ...
    def step_flags(self): ...
    def step_commit(self, accept: bool): ...
    def dt_candidates(self): ...
    def step_report(self) -> dict: ...  # REPORT_KEYS of the owned elements, this rank


def _offsets(plan, which):
    off, out = 0, {}
    for p in plan.peers:
        n = len(getattr(plan, which)[p])
        out[p] = (off, n)
        off += n
    return out, off


class TorchExchanger:
    """Halo exchange with torch.distributed point-to-point ops (NCCL or gloo)."""

    def __init__(self, backend: Backend, device):
        import torch
        self.torch = torch
        self.b = backend
        plan = backend.plan
        self.soff, ns = _offsets(plan, "send_idx")
        self.roff, nr = _offsets(plan, "recv_idx")
        self.send = torch.zeros(max(ns, 1) * 4, dtype=torch.float64, device=device)
        self.recv = torch.zeros(max(nr, 1) * 4, dtype=torch.float64, device=device)
        self._ops = {}  # what -> the P2P op list (same buffers every stage: built once)

    def _p2p_ops(self, what: int):
        ops = self._ops.get(what)
        if ops is None:
            dist = self.torch.distributed
            nf = 4 if what else 3
            ops = []
            for p in self.b.plan.peers:
                o, n = self.soff[p]
                if n:
                    ops.append(dist.P2POp(dist.isend, self.send[o * nf:(o + n) * nf], p))
                o, n = self.roff[p]
                if n:
                    ops.append(dist.P2POp(dist.irecv, self.recv[o * nf:(o + n) * nf], p))
            self._ops[what] = ops
        return ops

    def exchange(self, what: int, k: int):
        self.finish(self.start(what, k))

    def start(self, what: int, k: int):
        """pack + post the sends/receives; NCCL runs them on its own stream, after
        the pack on the current stream.  Returns the handle `finish` takes."""
        self.b.pack(what, k, self.send)
        ops = self._p2p_ops(what)
        return what, k, (self.torch.distributed.batch_isend_irecv(ops) if ops else [])

    def finish(self, handle):
        """the current stream waits for the transfers, then unpacks"""
        what, k, works = handle
        for r in works:
            r.wait()
        self.b.unpack(what, k, self.recv)

    def all_max(self, vals):
        t = self.torch.tensor(vals, dtype=self.torch.float64, device=self.send.device)
        self.torch.distributed.all_reduce(t, op=self.torch.distributed.ReduceOp.MAX)
        return t.tolist()

    def all_min(self, vals):
        return [-v for v in self.all_max([-v for v in vals])]

    def all_gather(self, vals):
        """every rank's `vals`, in rank order (for order-fixed sums)"""
        torch = self.torch
        t = torch.tensor(vals, dtype=torch.float64, device=self.send.device)
        out = [torch.empty_like(t) for _ in range(torch.distributed.get_world_size())]
        torch.distributed.all_gather(out, t)
        return [o.tolist() for o in out]


class IpcExchanger:
    """Halo exchange through peer memory, no NCCL: every rank exports a mailbox
    (two receive slots -- exchanges alternate between them -- and one sequence
    flag per peer) by CUDA IPC and maps its peers'.  `start` queues, per peer, one
    kernel that packs this rank's send entries straight into the peer's slot (NVLink
    / NVSwitch stores between GPUs) and then raises this rank's flag there;
    `finish` queues a device-side wait on this rank's own flags and the unpack from
    its slot.  Both are stream-ordered with the stage kernels: no host
    synchronisation and no separate communication stream per exchange, and the
    interior stage kernel queued between them overlaps the transfer.  Slot reuse is
    safe without acknowledgements: a rank writes slot s&1 of exchange s only after
    its wait for exchange s-1 saw the peer's flag, which the peer raised after
    unpacking exchange s-2 (its own stream order).  torch.distributed (any backend,
    CPU tensors) carries the setup and the per-step reductions.  Ranks may share a
    GPU (the mapping is then plain device memory of the other process)."""

    def __init__(self, backend: "GpuPartition", timeout_s: float = 30.0):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.b = backend
        self.timeout_s = timeout_s
        plan = backend.plan
        self.peers = list(plan.peers)
        self.soff, ns = _offsets(plan, "send_idx")
        self.roff, nr = _offsets(plan, "recv_idx")
        self.slot = max(nr, 1) * 4  # doubles per receive slot
        nflag = max(len(self.peers), 1)
        # mailbox: 2 receive slots, the peers' flags, and this rank's device-resident
        # sequence base (graph replays; local use only)
        self.base, handle = backend.ipc_alloc((2 * self.slot + nflag + 1) * 8)
        self.flags = self.base + 2 * self.slot * 8
        self.seq_base = self.flags + nflag * 8
        self.dev_base = 0   # host mirror of *seq_base
        self.capturing = None  # exchange count inside a capture
        me = dist.get_rank()
        info = dict(handle=handle, slot=self.slot,
                    at={p: (self.roff[p][0], self.roff[p][1], j) for j, p in enumerate(self.peers)})
        allinfo = [None] * dist.get_world_size()
        dist.all_gather_object(allinfo, info)
        self.dst, self.flag_at = {}, {}
        for p in self.peers:
            o, n, j = allinfo[p]["at"][me]
            assert n == self.soff[p][1], "halo plans disagree between ranks"
            base = backend.ipc_open(allinfo[p]["handle"])
            self.dst[p] = (base, allinfo[p]["slot"], o)
            self.flag_at[p] = base + (2 * allinfo[p]["slot"] + j) * 8
        self.seq = 0

    def start(self, what: int, k: int):
        if self.capturing is None:  # eager: absolute sequence numbers
            self.seq += 1
            seq, off, base = self.seq, self.seq, None
        else:  # captured: offsets from the device-resident base
            self.capturing += 1
            seq, off, base = self.seq + self.capturing, self.capturing, self.seq_base
        s, nf = seq & 1, (4 if what else 3)
        for p in self.peers:
            pbase, slot, o = self.dst[p]
            first, n = self.soff[p]
            self.b.push(what, k, first, n, pbase + (s * slot + o * nf) * 8, self.flag_at[p],
                        off, base)
        return what, k, seq, off, base

    def finish(self, handle):
        what, k, seq, off, base = handle
        self.b.wait_flags(self.flags, len(self.peers), off, self.timeout_s, base)
        self.b.unpack_at(what, k, self.base + (seq & 1) * self.slot * 8)

    # CUDA-graph capture of whole steps: the captured pushes and waits carry
    # sequence offsets from the device base, and the replay's last kernel advances
    # the base by the replay's exchange count (even, so every exchange keeps its
    # receive slot from replay to replay)
    def sync_base(self):
        """bring the device base to the host count (eagerly, before a capture)"""
        if self.dev_base != self.seq:
            self.b.seq_advance(self.seq_base, self.seq - self.dev_base)
            self.dev_base = self.seq

    def capture_begin(self):
        if self.dev_base != self.seq:
            raise RuntimeError("sync_base() before the capture")
        self.capturing = 0

    def capture_end(self) -> int:
        n, self.capturing = self.capturing, None
        if n % 2:
            raise ValueError("a captured replay needs an even number of exchanges")
        self.b.seq_advance(self.seq_base, n)
        self.per_replay = n
        return n

    def replayed(self):
        self.seq += self.per_replay
        self.dev_base += self.per_replay

    def exchange(self, what: int, k: int):
        self.finish(self.start(what, k))

    def _check(self):
        if self.b.halo_timed_out():
            raise RuntimeError("peer-memory halo exchange timed out (a peer never raised its flag)")

    def _dev(self):
        # the reductions ride on whatever process group carries the setup: NCCL
        # needs device tensors, gloo takes host ones
        return "cuda" if self.dist.get_backend() == "nccl" else "cpu"

    def all_max(self, vals):
        self._check()
        t = self.torch.tensor(vals, dtype=self.torch.float64, device=self._dev())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.tolist()

    def all_min(self, vals):
        return [-v for v in self.all_max([-v for v in vals])]

    def all_gather(self, vals):
        self._check()
        t = self.torch.tensor(vals, dtype=self.torch.float64, device=self._dev())
        out = [self.torch.empty_like(t) for _ in range(self.dist.get_world_size())]
        self.dist.all_gather(out, t)
        return [o.tolist() for o in out]


class LoopbackExchanger:
    """Several partitions in one process: halo buffers copied directly."""

    def __init__(self, backends, make_buffer):
        self.bs = backends
        self.bufs = []
        for b in backends:
            soff, ns = _offsets(b.plan, "send_idx")
            roff, nr = _offsets(b.plan, "recv_idx")
            self.bufs.append((soff, roff, make_buffer(max(ns, 1) * 4), make_buffer(max(nr, 1) * 4)))

    def exchange_all(self, what: int, k: int):
        nf = 4 if what else 3
        for b, (_, _, send, _) in zip(self.bs, self.bufs):
            b.pack(what, k, send)
        for r, (b, (_, roff, _, recv)) in enumerate(zip(self.bs, self.bufs)):
            for p in b.plan.peers:
                o, n = roff[p]
                so, sn = self.bufs[p][0][r]
                assert sn == n, "halo plans disagree between ranks"
                recv[o * nf:(o + n) * nf] = self.bufs[p][2][so * nf:(so + n) * nf]
        for b, (_, _, _, recv) in zip(self.bs, self.bufs):
            b.unpack(what, k, recv)


INTERIOR, BOUNDARY = 1, 2


def _overlap(b: Backend) -> bool:
    """partitions with an interior run each stage in two parts, the interior one
    while a halo is in flight: inviscid, the stage kernel during the state
    exchange; viscous, the pre-kernel during the state exchange and the stage
    kernel during the flux-pair exchange"""
    return getattr(b, "has_interior", False)


def _stage_overlapped(b: Backend, ex, k: int, t: float, dt: float):
    h = ex.start(0, k)
    if b.visc:
        b.stage_visc_part(k, t, dt, INTERIOR)
        ex.finish(h)
        b.stage_visc_part(k, t, dt, BOUNDARY)
        h = ex.start(1, k)
    b.stage_run_part(k, t, dt, INTERIOR)
    ex.finish(h)
    b.stage_run_part(k, t, dt, BOUNDARY)


def try_step_distributed(b: Backend, ex, t: float, dt: float) -> bool:
    """One SSPRK3 step of this rank's partition, in lock step with the other ranks."""
    b.step_begin()
    for k in range(3):
        if _overlap(b) and hasattr(ex, "start"):
            _stage_overlapped(b, ex, k, t, dt)
            continue
        ex.exchange(0, k)
        if b.visc:
            b.stage_visc(k, t, dt)
            ex.exchange(1, k)
        b.stage_run(k, t, dt)
    rej, ab = b.step_flags()
    rej, ab = ex.all_max([float(rej), float(ab)])
    if ab:
        raise swdg.NumericalAbort("negative water height without limiter")
    accept = not rej
    b.step_commit(accept)
    return accept


def _step_stages(b: Backend, ex, t: float, dt: float):
    for k in range(3):
        if _overlap(b) and hasattr(ex, "start"):
            _stage_overlapped(b, ex, k, t, dt)
            continue
        ex.exchange(0, k)
        if b.visc:
            b.stage_visc(k, t, dt)
            ex.exchange(1, k)
        b.stage_run(k, t, dt)


class GraphStepper:
    """Fixed-dt partitioned stepping replayed from a captured CUDA graph.  With the
    peer-memory exchanger a whole step is stream-ordered device work (pushes,
    device-side flag waits, unpacks, interior/boundary stage kernels), so two steps
    -- the W/A ping-pong returns to its start -- are captured once and replayed: no
    Python and no host synchronisation per stage or per step.  The first step runs
    eagerly (first-launch attributes and occupancy queries stay out of the
    capture), and so does an odd remainder.  No forcing (the captured stage
    arguments are those of the captured steps)."""

    def __init__(self, b: "GpuPartition", ex: "IpcExchanger", t: float, dt: float):
        self.b, self.ex, self.t, self.dt = b, ex, t, dt
        self.g = None
        self.replays = 0
        self.replay_launches = 0  # kernels per replay (counted while capturing)

    def _eager(self):
        _step_stages(self.b, self.ex, self.t, self.dt)
        self.b.step_commit(True)

    def _capture(self):
        import torch
        b, ex = self.b, self.ex
        ex.sync_base()
        self.g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        l0 = b.integ.launch_count()
        with torch.cuda.graph(self.g, stream=side, capture_error_mode="thread_local"):
            b.set_stream(torch.cuda.current_stream().cuda_stream)
            ex.capture_begin()
            for _ in range(2):
                _step_stages(b, ex, self.t, self.dt)
                b.step_commit(True)
            ex.capture_end()
        self.replay_launches = b.integ.launch_count() - l0
        b.set_stream(torch.cuda.current_stream().cuda_stream)

    def run(self, nsteps: int):
        """queue nsteps steps (no host synchronisation)"""
        if self.g is None and nsteps > 0:
            self._eager()
            nsteps -= 1
            if nsteps >= 2:
                self._capture()
                self.phase = 0  # eager steps since the capture, mod 2
        if self.g is None:
            for _ in range(nsteps):
                self._eager()
            return
        # the graph holds the buffers of an even step: after an odd number of
        # eager steps one more eager step re-aligns the W/A ping-pong with it
        if self.phase and nsteps > 0:
            self._eager()
            self.phase, nsteps = 0, nsteps - 1
        # eager steps advanced the host sequence count: the device base follows
        # (an even number of eager steps since the capture, so the receive-slot
        # parity the graph carries still holds), else the replay's flags would
        # fall behind values the eager exchanges already stored
        if nsteps >= 2:
            self.ex.sync_base()
        for _ in range(nsteps // 2):
            self.g.replay()
            self.ex.replayed()
            self.replays += 1
        if nsteps % 2:
            self._eager()
            self.phase ^= 1

    def accepted(self) -> bool:
        """the stage flags of every step since begin(), reduced over the ranks"""
        rej, ab = self.b.step_flags()
        rej, ab = self.ex.all_max([float(rej), float(ab)])
        if ab:
            raise swdg.NumericalAbort("negative water height without limiter")
        return not rej

    def begin(self):
        self.b.step_begin()


def run_steps_distributed_graph(b: "GpuPartition", ex: "IpcExchanger", nsteps: int, t: float,
                                dt: float) -> bool:
    """run_steps_distributed over GraphStepper (peer-memory exchanger)."""
    st = GraphStepper(b, ex, t, dt)
    st.begin()
    st.run(nsteps)
    return st.accepted()


def run_steps_distributed(b: Backend, ex, nsteps: int, t: float, dt: float) -> bool:
    """Device-resident stepping for throughput runs (the partitioned counterpart of
    swdg_gpu_run_steps): no per-step host synchronisation; the stage flags
    accumulate over the run and are reduced over the ranks once at the end.
    Returns False if any stage of any rank signalled a reject (the caller treats
    the run as invalid)."""
    b.step_begin()
    for s in range(nsteps):
        ts = t + s * dt
        for k in range(3):
            if _overlap(b) and hasattr(ex, "start"):
                _stage_overlapped(b, ex, k, ts, dt)
                continue
            ex.exchange(0, k)
            if b.visc:
                b.stage_visc(k, ts, dt)
                ex.exchange(1, k)
            b.stage_run(k, ts, dt)
        b.step_commit(True)
    rej, ab = b.step_flags()
    rej, ab = ex.all_max([float(rej), float(ab)])
    if ab:
        raise swdg.NumericalAbort("negative water height without limiter")
    return not rej


def try_step_loopback(bs, ex: LoopbackExchanger, t: float, dt: float) -> bool:
    """All partitions of one process, one SSPRK3 step (the same schedule)."""
    for b in bs:
        b.step_begin()
    for k in range(3):
        if all(_overlap(b) for b in bs):  # interior before each exchange, like NCCL ranks
            if bs[0].visc:
                for b in bs:
                    b.stage_visc_part(k, t, dt, INTERIOR)
                ex.exchange_all(0, k)
                for b in bs:
                    b.stage_visc_part(k, t, dt, BOUNDARY)
                for b in bs:
                    b.stage_run_part(k, t, dt, INTERIOR)
                ex.exchange_all(1, k)
            else:
                for b in bs:
                    b.stage_run_part(k, t, dt, INTERIOR)
                ex.exchange_all(0, k)
            for b in bs:
                b.stage_run_part(k, t, dt, BOUNDARY)
            continue
        ex.exchange_all(0, k)
        if bs[0].visc:
            for b in bs:
                b.stage_visc(k, t, dt)
            ex.exchange_all(1, k)
        for b in bs:
            b.stage_run(k, t, dt)
    flags = [b.step_flags() for b in bs]
    if any(a for _, a in flags):
        raise swdg.NumericalAbort("negative water height without limiter")
    accept = not any(r for r, _ in flags)
    for b in bs:
        b.step_commit(accept)
    return accept


# StepDiagnostics fields a step produces per rank (driver.hpp:115-127)
REPORT_KEYS = ("mass", "entropy", "min_h", "positivity_dt", "n_limited", "min_stage_h",
               "max_eps")


def combine_reports(rows) -> dict:
    """sums of mass, entropy and n_limited (in rank order, so the
    result is independent of the collective's reduction order), minima of min_h,
    the positivity bound and min_stage_h, maximum of max_eps."""
    cols = list(zip(*rows))
    out = {}
    for k, col in zip(REPORT_KEYS, cols):
        if k in ("mass", "entropy", "n_limited"):
            acc = 0.0
            for v in col:
                acc += v
            out[k] = int(acc) if k == "n_limited" else acc
        elif k == "max_eps":
            out[k] = max(col)
        else:
            out[k] = min(col)
    return out


def step_report_distributed(b: Backend, ex) -> dict:
    """The step diagnostics of the whole partitioned mesh (field.hpp:39-68,
    limiter.hpp:135-166 and the try_step report timeloop.hpp:192-195).  The
    positivity bound of a cut face needs the neighbour's NEW state: the committed
    state's halo is exchanged first (the ghosts still hold stage-3 inputs)."""
    ex.exchange(0, 0)
    loc = b.step_report()
    return combine_reports(ex.all_gather([float(loc[k]) for k in REPORT_KEYS]))


def step_report_loopback(bs, ex) -> dict:
    ex.exchange_all(0, 0)
    return combine_reports([[float(b.step_report()[k]) for k in REPORT_KEYS] for b in bs])


def run_simulation_distributed(b: Backend, ex, final_time: float, cfl: float, degree: int,
                               phys, max_steps=None, keep_series=True):
    """run_simulation's loop (driver.hpp:91-138) over the ranks: the global CFL dt,
    reject-and-halve in lock step, and the global step diagnostics per step."""
    t, steps, series = 0.0, 0, []
    t_eps = 1e-12 * max(1.0, final_time)
    while t < final_time - t_eps:
        if max_steps is not None and steps >= max_steps:
            break
        dt = compute_dt_distributed(b, ex, cfl, degree, phys)
        hit = False
        if t + dt >= final_time - t_eps:
            dt, hit = final_time - t, True
        rej = 0
        while not try_step_distributed(b, ex, t, dt):
            dt *= 0.5
            hit = False
            rej += 1
            if rej >= 10:
                raise swdg.NumericalAbort(f"step rejected 10 times at t={t}")
        t = final_time if hit else t + dt
        steps += 1
        rep = step_report_distributed(b, ex)
        if keep_series:
            series.append(dict(step=steps, t=t, dt=dt, **rep))
    return t, steps, series


def compute_dt_distributed(b: Backend, ex, cfl: float, degree: int, phys) -> float:
    """compute_dt (timeloop.hpp:53-75) over all ranks: min of both reductions, then
    the all-dry fallback, exactly as on one device."""
    if not (cfl > 0.0) or cfl > 1.0:
        raise swdg.SwdgError("compute_dt: cfl must be in (0, 1]")
    d, ml = b.dt_candidates()
    d, ml = ex.all_min([d, ml])
    if not math.isfinite(d):
        order = 2.0 * degree + 1.0
        d = ml / (order * math.sqrt(phys.g * max(phys.h_ref, 1e-12)))
    return cfl * d


class GpuPartition(Backend):
    """One rank's partition on the GPU through the split-step C ABI."""

    def __init__(self, lm: LocalMesh, cfg: swdg.RunConfig, device: int = 0, integ=None):
        self.lm = lm
        self.plan = lm.halo
        self.visc = bool(cfg.visc.enabled)
        if integ is None:
            mesh = swdg.Mesh(lm.degree, lm.n_elem, lm.arrays, lm.faces, n_owned=lm.n_owned)
            integ = swdg.TimeIntegrator(mesh, cfg, device=device)
        self.integ = integ
        L = swdg.lib()
        vp, i32p = C.c_void_p, C.POINTER(C.c_int32)
        for name, args in (("swdg_gpu_halo_setup", [vp, C.c_int64, i32p, C.c_int64, i32p]),
                           ("swdg_gpu_halo_pack", [vp, C.c_int, C.c_int, C.c_void_p]),
                           ("swdg_gpu_halo_unpack", [vp, C.c_int, C.c_int, C.c_void_p]),
                           ("swdg_gpu_step_begin", [vp]),
                           ("swdg_gpu_stage_visc", [vp, C.c_int, C.c_double, C.c_double]),
                           ("swdg_gpu_stage_run", [vp, C.c_int, C.c_double, C.c_double]),
                           ("swdg_gpu_set_interior", [vp, C.c_int32, C.c_int32]),
                           ("swdg_gpu_stage_visc_part", [vp, C.c_int, C.c_double, C.c_double,
                                                         C.c_int]),
                           ("swdg_gpu_stage_run_part", [vp, C.c_int, C.c_double, C.c_double,
                                                        C.c_int]),
                           ("swdg_gpu_step_flags", [vp, i32p, i32p]),
                           ("swdg_gpu_step_commit", [vp, C.c_int, C.POINTER(swdg.StepInfoC)]),
                           ("swdg_gpu_dt_candidates", [vp, C.POINTER(C.c_double),
                                                       C.POINTER(C.c_double)]),
                           ("swdg_gpu_ipc_alloc", [vp, C.c_int64, C.POINTER(C.c_void_p),
                                                   C.c_void_p]),
                           ("swdg_gpu_ipc_open", [vp, C.c_void_p, C.POINTER(C.c_void_p)]),
                           ("swdg_gpu_halo_push", [vp, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                                   C.c_void_p, C.c_void_p, C.c_void_p,
                                                   C.c_uint64]),
                           ("swdg_gpu_halo_wait", [vp, C.c_void_p, C.c_int32, C.c_void_p,
                                                   C.c_uint64, C.c_double]),
                           ("swdg_gpu_seq_advance", [vp, C.c_void_p, C.c_uint64]),
                           ("swdg_gpu_halo_status", [vp, i32p])):
            f = getattr(L, name)
            f.restype = C.c_int
            f.argtypes = args
        self.L = L
        send = np.concatenate([self.plan.send_idx[p] for p in self.plan.peers] or
                              [np.zeros(0, np.int32)]).astype(np.int32)
        recv = np.concatenate([self.plan.recv_idx[p] for p in self.plan.peers] or
                              [np.zeros(0, np.int32)]).astype(np.int32)
        self._keep = (send, recv)
        self._chk(L.swdg_gpu_halo_setup(self.integ._h, len(send), send.ctypes.data_as(i32p),
                                        len(recv), recv.ctypes.data_as(i32p)))
        self.info = swdg.StepInfoC()
        from .partition import interior_range
        lo, hi = interior_range(lm.faces, lm.n_owned)
        self._chk(L.swdg_gpu_set_interior(self.integ._h, lo, hi))
        self.has_interior = hi - lo >= 2
        # halo buffers are torch tensors moved by torch (NCCL / copies): order the
        # context's kernels on torch's current stream
        import torch
        self.integ.set_stream(torch.cuda.current_stream().cuda_stream)

    @classmethod
    def structured(cls, spec, cfg: swdg.RunConfig, P: int, rank: int, device: int = 0):
        """Rank `rank` of P of a device-generated structured mesh: the host builds only
        the face list and the partition plan; geometry is generated on the device for
        the owned and ghost elements."""
        from .partition import build_plan
        K = spec.kx * spec.ky
        faces = swdg.structured_faces(spec.kx, spec.ky, spec.periodic_x, spec.periodic_y)
        gids, n_owned, lf, ords, plan = build_plan(faces, K, spec.degree, P, rank)
        lm = LocalMesh(spec.degree, len(gids), n_owned, gids, lf, ords, {}, plan)
        integ = swdg.TimeIntegrator.structured_part(spec, cfg, gids, n_owned, lf, device)
        return cls(lm, cfg, device, integ=integ)

    def _chk(self, rc):
        self.integ._check(rc)

    def set_stream(self, handle):
        self.integ.set_stream(handle)

    def upload(self, state):
        self.integ.upload(swdg.State(*state))

    def download(self):
        out = [np.empty(self.lm.n_nodes) for _ in range(3)]
        self.integ.download(swdg.State(*out))
        return out

    def step_begin(self):
        self._chk(self.L.swdg_gpu_step_begin(self.integ._h))

    def pack(self, what, k, buf):
        self._chk(self.L.swdg_gpu_halo_pack(self.integ._h, what, k, C.c_void_p(buf.data_ptr())))

    def unpack(self, what, k, buf):
        self._chk(self.L.swdg_gpu_halo_unpack(self.integ._h, what, k, C.c_void_p(buf.data_ptr())))

    def unpack_at(self, what, k, ptr: int):
        self._chk(self.L.swdg_gpu_halo_unpack(self.integ._h, what, k, C.c_void_p(ptr)))

    # direct peer-memory exchange (IpcExchanger)
    def ipc_alloc(self, nbytes: int):
        p, h = C.c_void_p(), (C.c_char * 64)()
        self._chk(self.L.swdg_gpu_ipc_alloc(self.integ._h, nbytes, C.byref(p), h))
        return p.value, bytes(h)

    def ipc_open(self, handle: bytes) -> int:
        p, h = C.c_void_p(), (C.c_char * 64).from_buffer_copy(handle)
        self._chk(self.L.swdg_gpu_ipc_open(self.integ._h, h, C.byref(p)))
        return p.value

    def push(self, what, k, first, count, dst: int, flag: int, seq: int, base: int | None = None):
        self._chk(self.L.swdg_gpu_halo_push(self.integ._h, what, k, first, count,
                                            C.c_void_p(dst), C.c_void_p(flag), C.c_void_p(base),
                                            seq))

    def wait_flags(self, flags: int, n: int, seq: int, timeout_s: float,
                   base: int | None = None):
        self._chk(self.L.swdg_gpu_halo_wait(self.integ._h, C.c_void_p(flags), n,
                                            C.c_void_p(base), seq, timeout_s))

    def seq_advance(self, base: int, by: int):
        self._chk(self.L.swdg_gpu_seq_advance(self.integ._h, C.c_void_p(base), by))

    def halo_timed_out(self) -> bool:
        v = C.c_int32()
        self._chk(self.L.swdg_gpu_halo_status(self.integ._h, C.byref(v)))
        return bool(v.value)

    def stage_visc(self, k, t, dt):
        self._chk(self.L.swdg_gpu_stage_visc(self.integ._h, k, t, dt))

    def stage_run(self, k, t, dt):
        self._chk(self.L.swdg_gpu_stage_run(self.integ._h, k, t, dt))

    def stage_run_part(self, k, t, dt, part):
        self._chk(self.L.swdg_gpu_stage_run_part(self.integ._h, k, t, dt, part))

    def stage_visc_part(self, k, t, dt, part):
        self._chk(self.L.swdg_gpu_stage_visc_part(self.integ._h, k, t, dt, part))

    def step_flags(self):
        r, a = C.c_int32(), C.c_int32()
        self._chk(self.L.swdg_gpu_step_flags(self.integ._h, C.byref(r), C.byref(a)))
        return r.value, a.value

    def step_commit(self, accept):
        self._chk(self.L.swdg_gpu_step_commit(self.integ._h, int(accept), C.byref(self.info)))

    def dt_candidates(self):
        d, m = C.c_double(), C.c_double()
        self._chk(self.L.swdg_gpu_dt_candidates(self.integ._h, C.byref(d), C.byref(m)))
        return d.value, m.value

    def step_report(self):
        """this rank's owned-element diagnostics of the committed state and its
        stage report (reduced over ranks by step_report_distributed)"""
        d = self.integ.diagnostics_device()
        return dict(mass=d.mass, entropy=d.entropy, min_h=d.min_h,
                    positivity_dt=d.positivity_dt, n_limited=self.info.n_limited,
                    min_stage_h=self.info.min_stage_h, max_eps=self.info.max_eps)
