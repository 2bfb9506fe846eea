"""The peer-memory halo protocol of distributed.IpcExchanger on the CPU: two gloo
ranks run the partitioned oracle stepping with the real exchanger over a backend
whose "device memory" is POSIX shared memory -- mailboxes exported and mapped by
name, packs written straight into the peer's receive slot, sequence flags stored
after the data and polled by the receiver.  Eager exchanges and the device-base
offsets of captured replays (executed directly here: capture_end's base advance
runs at once, like the end of a replay) must reproduce the single-process oracle
run bitwise, which pins the slot alternation, the flag ordering and the sequence
arithmetic that the GPU kernels implement."""
import os
import socket
import time

import numpy as np

from oracle import port, ref
from paper_1804_02221_b200 import partition as part
from tests.helpers import beq, scenario_params
from tests.port_partition import PortPartition

_SEG = 40  # address = segment id << _SEG | byte offset


class ShmPartition(PortPartition):
    """PortPartition plus the IPC entry points, over multiprocessing shared memory."""

    def __init__(self, lm, p):
        super().__init__(lm, p)
        self.segs = {}
        self.own = []
        self.timed_out = False

    def _view(self, addr, nbytes):
        seg = self.segs[addr >> _SEG]
        off = addr & ((1 << _SEG) - 1)
        return np.ndarray(nbytes // 8, dtype=np.float64, buffer=seg.buf, offset=off)

    def _u64(self, addr, n=1):
        seg = self.segs[addr >> _SEG]
        return np.ndarray(n, dtype=np.uint64, buffer=seg.buf, offset=addr & ((1 << _SEG) - 1))

    def ipc_alloc(self, nbytes):
        from multiprocessing import shared_memory
        seg = shared_memory.SharedMemory(create=True, size=nbytes)
        seg.buf[:nbytes] = bytes(nbytes)
        sid = os.getpid() * 16 + len(self.own) + 1  # unique across the ranks
        self.segs[sid] = seg
        self.own.append(seg)
        return sid << _SEG, (f"{sid}:{seg.name}".encode()).ljust(64, b"\0")

    def ipc_open(self, handle):
        from multiprocessing import shared_memory
        sid, name = handle.rstrip(b"\0").decode().split(":")
        seg = shared_memory.SharedMemory(name=name)
        self.segs[int(sid)] = seg
        return int(sid) << _SEG

    def push(self, what, k, first, count, dst, flag, seq, base=None):
        f = self._fields(what, k)
        nf = len(f)
        if count:
            idx = self.send[first:first + count]
            self._view(dst, count * nf * 8)[:] = np.stack([a[idx] for a in f], axis=1).ravel()
        self._u64(flag)[0] = (int(self._u64(base)[0]) if base else 0) + seq  # after the data

    def wait_flags(self, flags, n, seq, timeout_s, base=None):
        want = (int(self._u64(base)[0]) if base else 0) + seq
        t0 = time.monotonic()
        while n and not (self._u64(flags, n) >= want).all():
            if time.monotonic() - t0 > timeout_s:
                self.timed_out = True
                return
            time.sleep(1e-4)

    def unpack_at(self, what, k, addr):
        nf = 4 if what else 3
        self.unpack(what, k, self._view(addr, max(len(self.recv), 1) * nf * 8))

    def seq_advance(self, base, by):
        self._u64(base)[0] += np.uint64(by)

    def halo_timed_out(self):
        v, self.timed_out = self.timed_out, False
        return v

    def close(self):
        for seg in self.segs.values():
            seg.close()
        for seg in self.own:  # the exporting rank removes the name (after the barrier)
            seg.unlink()


def _worker(rank, world, port_no, path):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_no}", rank=rank,
                            world_size=world)
    from paper_1804_02221_b200.distributed import (IpcExchanger, _step_stages,
                                                   step_report_distributed,
                                                   try_step_distributed)
    m, st = ref.scenario_mesh("wetdry_dambreak", 8, 8, 3)
    p, cfg = scenario_params("wetdry_dambreak")
    dt = port.compute_dt(m, p, st, cfg["cfl"])
    lm = part.local_mesh(m, world, rank)
    b = ShmPartition(lm, p)
    b.upload(part.scatter_state(st, lm))
    ex = IpcExchanger(b, timeout_s=30.0)
    acc, reps = [], []
    for k in range(3):  # eager steps with the step reports' extra exchange
        acc.append(try_step_distributed(b, ex, k * dt, dt))
        reps.append(step_report_distributed(b, ex))
    for r in range(2):  # "replays": two steps in capture mode, base advanced at the end
        ex.sync_base()
        ex.capture_begin()
        for s in range(2):
            b.step_begin()
            _step_stages(b, ex, (3 + 2 * r + s) * dt, dt)
            b.step_commit(True)
        ex.capture_end()
        ex.replayed()
    timed_out = b.halo_timed_out()
    np_ = lm.n1 * lm.n1
    mine = np.stack([w[: lm.n_owned * np_] for w in b.W])
    gathered = [None] * world
    dist.all_gather_object(gathered, (lm.global_ids[: lm.n_owned].tolist(), mine, acc, reps,
                                      ex.seq, timed_out))
    dist.barrier()
    b.close()
    if rank == 0:
        np.save(path, np.array(gathered, dtype=object), allow_pickle=True)
    dist.destroy_process_group()


def test_ipc_protocol_two_ranks_bitwise(tmp_path):
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    path = os.path.join(tmp_path, "res.npy")
    mp.spawn(_worker, args=(2, port_no, path), nprocs=2, join=True)
    res = np.load(path, allow_pickle=True)
    m, st = ref.scenario_mesh("wetdry_dambreak", 8, 8, 3)
    p, cfg = scenario_params("wetdry_dambreak")
    dt = port.compute_dt(m, p, st, cfg["cfl"])
    want = [a.copy() for a in st]
    acc_ref = []
    for k in range(7):
        acc_ref.append(bool(port.try_step(m, p, want, k * dt, dt).accepted))
    assert all(acc_ref)
    np_ = m.n1 * m.n1
    got = [np.zeros(m.n_nodes) for _ in range(3)]
    for gids, mine, acc, reps, seq, timed_out in res:
        assert acc == acc_ref[:3] and not timed_out
        assert seq == 3 * (6 + 1) + 2 * 2 * 6  # eager steps + reports, two 2-step replays
        sel = (np.array(gids)[:, None] * np_ + np.arange(np_)).ravel()
        for j in range(3):
            got[j][sel] = mine[j]
    assert beq(got, want)
