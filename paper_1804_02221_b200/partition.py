"""Element partitioning and face-trace halo plans for multi-GPU runs.

The reference has no decomposition (one process holds the whole mesh); this module
adds one.  It is a pure function of (face list, K, P):

* ranks own contiguous element ranges [r K / P, (r+1) K / P) — for the structured
  generators (e = ey kx + ex, mesh.hpp:241) these are bands of element rows;
* each rank's local mesh is its owned elements (local ids 0..n_owned-1, global order)
  followed by ghost copies of every off-rank neighbour (sorted by global id);
* the local face list is the subsequence of MeshTopology::faces touching an owned
  element, in global order, so every face keeps its ordinal rank — exact mode then
  accumulates corner contributions in the reference order and a partitioned run is
  bitwise the single-GPU run;
* halo plans list, per peer and in global-face order, the owner-side face nodes the
  peer needs (sender local node ids) and where they land (receiver ghost node ids).

Per stage the halo carries the stage-input state at those nodes (3 doubles per face
node); with viscosity a second exchange carries the viscous flux pairs (4 doubles).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

NODE_ARRAYS = ("x", "y", "x_xi", "x_eta", "y_xi", "y_eta", "jac", "b")
FACE_ARRAYS = ("face_jsurf", "face_nx", "face_ny", "face_a")
OP_ARRAYS = ("weights", "deriv", "deriv_modified", "deriv_weak", "vandermonde_inv")


def ranges(K: int, P: int):
    """Owned element range of every rank (balanced, integer arithmetic)."""
    return [(r * K // P, (r + 1) * K // P) for r in range(P)]


def owner(e: np.ndarray, K: int, P: int) -> np.ndarray:
    """Rank owning global element e (inverse of `ranges`)."""
    e = np.asarray(e, np.int64)
    r = (e * P) // K
    # r*K//P <= e < (r+1)*K//P; the estimate can be one too high or low
    lo = (r * K) // P
    r = np.where(e < lo, r - 1, r)
    hi = ((r + 1) * K) // P
    r = np.where(e >= hi, r + 1, r)
    return r


def face_node(n1: int, face: np.ndarray, t: np.ndarray) -> np.ndarray:
    """core.hpp:53-61 face_node_index, vectorised."""
    face = np.asarray(face)
    t = np.asarray(t)
    return np.select([face == 0, face == 1, face == 2],
                     [t * n1, (n1 - 1) * n1 + t, t * n1 + (n1 - 1)], t)


@dataclass
class HaloPlan:
    peers: list = field(default_factory=list)        # peer ranks, ascending
    send_idx: dict = field(default_factory=dict)     # peer -> local node ids (owner side)
    recv_idx: dict = field(default_factory=dict)     # peer -> local ghost node ids


@dataclass
class LocalMesh:
    """A rank's partition in the swdg_mesh_view layout (owned first, then ghosts)."""
    degree: int
    n_elem: int
    n_owned: int
    global_ids: np.ndarray            # local -> global element id
    faces: np.ndarray                 # (F, 6) int32, local ids, global order
    face_ordinals: np.ndarray         # global ordinal of each local face
    arrays: dict = field(default_factory=dict)
    halo: HaloPlan = field(default_factory=HaloPlan)

    @property
    def n1(self):
        return self.degree + 1

    @property
    def n_nodes(self):
        return self.n_elem * self.n1 * self.n1


def build_plan(faces: np.ndarray, K: int, degree: int, P: int, rank: int):
    """Local element ids, local faces and halo plan for `rank` (no geometry)."""
    faces = np.asarray(faces, np.int64).reshape(-1, 6)
    n1 = degree + 1
    np_ = n1 * n1
    e0, e1 = ranges(K, P)[rank]
    em, fm, ep, fp, rev, tag = (faces[:, k] for k in range(6))
    interior = tag == 0
    own_m = (em >= e0) & (em < e1)
    own_p = interior & (ep >= e0) & (ep < e1)
    keep = own_m | own_p
    # ghosts: off-rank neighbours of owned elements
    ghost_m = keep & ~own_m
    ghost_p = keep & interior & ~own_p
    ghosts = np.unique(np.concatenate([em[ghost_m], ep[ghost_p]]))
    n_owned = e1 - e0
    global_ids = np.concatenate([np.arange(e0, e1, dtype=np.int64), ghosts])
    g2l = {int(g): n_owned + i for i, g in enumerate(ghosts)}

    def to_local(e):
        e = np.asarray(e, np.int64)
        out = e - e0
        off = (e < e0) | (e >= e1)
        if off.any():
            out = out.copy()
            out[off] = [g2l[int(x)] for x in e[off]]
        return out

    lf = faces[keep].copy()
    lf[:, 0] = to_local(lf[:, 0])
    inter = lf[:, 5] == 0
    lf[inter, 2] = to_local(lf[inter, 2])
    ordinals = np.nonzero(keep)[0]

    # halo: every cut face of the global list, in global order, contributes the
    # minus side's face nodes to the plus side's rank and vice versa; both ranks of
    # a pair enumerate the same faces in the same order
    plan = HaloPlan()
    t = np.arange(n1)
    send, recv = {}, {}
    ranks_m = owner(em, K, P)
    ranks_p = owner(np.where(interior, ep, 0), K, P)
    for fi in np.nonzero(interior & (ranks_m != ranks_p))[0]:
        ra, rb = int(ranks_m[fi]), int(ranks_p[fi])
        if rank not in (ra, rb):
            continue
        for src_rank, dst_rank, e, f in ((ra, rb, em[fi], fm[fi]), (rb, ra, ep[fi], fp[fi])):
            nodes = face_node(n1, np.full(n1, f), t)
            if src_rank == rank:
                send.setdefault(dst_rank, []).append(to_local([e])[0] * np_ + nodes)
            if dst_rank == rank:
                recv.setdefault(src_rank, []).append(to_local([e])[0] * np_ + nodes)
    plan.peers = sorted(set(send) | set(recv))
    for p in plan.peers:
        plan.send_idx[p] = np.concatenate(send.get(p, [np.zeros(0, np.int64)])).astype(np.int32)
        plan.recv_idx[p] = np.concatenate(recv.get(p, [np.zeros(0, np.int64)])).astype(np.int32)
    return global_ids, n_owned, lf.astype(np.int32), ordinals, plan


def local_mesh(mesh, P: int, rank: int) -> LocalMesh:
    """Partition a host mesh (object with degree, n_elem, faces, arrays)."""
    gids, n_owned, lf, ords, plan = build_plan(mesh.faces, mesh.n_elem, mesh.degree, P, rank)
    n1 = mesh.degree + 1
    np_ = n1 * n1
    a = mesh.arrays
    arrays = {}
    node_sel = (gids[:, None] * np_ + np.arange(np_)).ravel()
    face_sel = (gids[:, None] * 4 * n1 + np.arange(4 * n1)).ravel()
    for k in NODE_ARRAYS:
        if k in a:
            arrays[k] = np.ascontiguousarray(a[k][node_sel])
    for k in FACE_ARRAYS:
        arrays[k] = np.ascontiguousarray(a[k][face_sel])
    for k in OP_ARRAYS:
        arrays[k] = a[k]
    return LocalMesh(mesh.degree, len(gids), n_owned, gids, lf, ords, arrays, plan)


def interior_range(faces: np.ndarray, n_owned: int):
    """The longest run [lo, hi) of owned elements none of whose faces touches a
    ghost (local id >= n_owned): the part of a stage that needs no halo data and
    can run while the exchange is in flight."""
    f = np.asarray(faces, np.int64).reshape(-1, 6)
    inter = f[:, 5] == 0
    em, ep = f[:, 0], np.where(inter, f[:, 2], f[:, 0])
    touch = np.zeros(n_owned + 1, bool)
    cut = inter & ((em >= n_owned) | (ep >= n_owned))
    for a, b in ((em, ep), (ep, em)):
        sel = cut & (a < n_owned)
        touch[a[sel]] = True
    best, lo = (0, 0), None
    for e in range(n_owned + 1):
        if e < n_owned and not touch[e]:
            if lo is None:
                lo = e
        elif lo is not None:
            if e - lo > best[1] - best[0]:
                best = (lo, e)
            lo = None
    return best


def scatter_state(state, lm: LocalMesh):
    """Global state -> this rank's local arrays (owned + ghosts)."""
    np_ = lm.n1 * lm.n1
    sel = (lm.global_ids[:, None] * np_ + np.arange(np_)).ravel()
    return [np.ascontiguousarray(s[sel]) for s in state]


def owned_slice(lm: LocalMesh):
    np_ = lm.n1 * lm.n1
    return slice(0, lm.n_owned * np_)
