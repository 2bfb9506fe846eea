"""TEST INFRASTRUCTURE: the distributed stepping loop's compute backend on the CPU
oracle (oracle/swdg_port.c).  A partitioned oracle run must reproduce the global
oracle run bitwise, which pins the partitioner, the halo plans and the exchange
schedule that the GPU backend (paper_1804_02221_b200.distributed.GpuPartition) uses."""
from __future__ import annotations

import numpy as np

from oracle import port
from paper_1804_02221_b200.distributed import Backend

CA = (0.0, 3.0 / 4.0, 1.0 / 3.0)
CB = (1.0, 1.0 / 4.0, 2.0 / 3.0)


class PortPartition(Backend):
    def __init__(self, lm, p):
        self.lm = lm
        self.plan = lm.halo
        self.p = p
        self.visc = bool(p.visc_enabled)
        self.view = port.View(lm)
        nn = lm.n_nodes
        z = lambda: [np.zeros(nn) for _ in range(3)]  # noqa: E731
        self.W, self.A, self.B = z(), z(), z()
        self.flux = [np.zeros(nn) for _ in range(4)]
        self.send = np.concatenate([self.plan.send_idx[q] for q in self.plan.peers] or
                                   [np.zeros(0, np.int32)])
        self.recv = np.concatenate([self.plan.recv_idx[q] for q in self.plan.peers] or
                                   [np.zeros(0, np.int32)])
        self.max_eps = 0.0

    def upload(self, state):
        self.W = [np.array(a, copy=True) for a in state]

    def inputs(self, k):
        return (self.W, self.A, self.B)[k]

    def _fields(self, what, k):
        return self.flux if what else self.inputs(k)

    def pack(self, what, k, buf):
        f = self._fields(what, k)
        nf = len(f)
        b = buf.numpy() if hasattr(buf, "numpy") else buf
        b[: len(self.send) * nf] = np.stack([a[self.send] for a in f], axis=1).ravel()

    def unpack(self, what, k, buf):
        f = self._fields(what, k)
        nf = len(f)
        b = buf.numpy() if hasattr(buf, "numpy") else buf
        vals = np.asarray(b[: len(self.recv) * nf]).reshape(-1, nf)
        for j, a in enumerate(f):
            a[self.recv] = vals[:, j]

    def step_begin(self):
        self.stage_flags = []
        self.stage_nl = []
        self.stage_mh = []
        self.max_eps = 0.0

    def stage_visc(self, k, t, dt):
        s = self.inputs(k)
        eps = port.compute_viscosity(self.view, self.p, s[0])
        self.max_eps = max(self.max_eps, float(eps[: self.lm.n_owned].max(initial=0.0)))
        u, v = port.velocities(self.view, self.p, s)
        grads = port.br1_gradients(self.view, u, v)
        self.flux = list(port.viscous_fluxes(self.view, s[0], grads, eps))

    def stage_run(self, k, t, dt):
        s = self.inputs(k)
        vis = port.viscous_lhs(self.view, self.flux) if self.visc else None
        r = port.assemble_rhs(self.view, self.p, s, visc=vis)
        out = []
        for a, ra, w in zip(s, r, self.W):
            o = a.copy()
            o += dt * ra  # StateVec::axpy
            if k > 0:
                o = CA[k] * w + CB[k] * o  # StateVec::combine
            out.append(np.ascontiguousarray(o))
        ok, nl, mh = port.post_stage(self.view, self.p, out)
        self.stage_flags.append(ok)
        self.stage_nl.append(nl)
        self.stage_mh.append(mh)
        if k == 1:
            self.B = out
        else:
            self.A = out

    def step_flags(self):
        for ok in self.stage_flags:
            if ok < 0:
                return 0, 1
            if ok == 0:
                return 1, 0
        return 0, 0

    def step_commit(self, accept):
        if accept:
            self.W = [a.copy() for a in self.A]

    def step_report(self):
        d = port.diagnostics(self.view, self.p, self.W)
        return dict(mass=d.mass, entropy=d.entropy, min_h=d.min_h,
                    positivity_dt=d.positivity_dt,
                    n_limited=self.stage_nl[-1] if self.p.limiter_enabled else 0,
                    min_stage_h=min(self.stage_mh), max_eps=self.max_eps)
