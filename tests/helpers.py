"""Shared fixtures for the parity tests (test infrastructure; may use oracle/)."""
from __future__ import annotations

import numpy as np

from oracle import ref


def beq(a, b) -> bool:
    """Bitwise equality of sequences of float64 arrays (signed zeros/NaN payloads count)."""
    return all(np.array_equal(np.asarray(x, np.float64).view(np.uint64),
                              np.asarray(y, np.float64).view(np.uint64)) for x, y in zip(a, b))


def normwise(a, b) -> float:
    """max_{node,field} |a-b| / max |b| (normwise because dry nodes)."""
    scale = max(float(np.max(np.abs(y))) for y in b) or 1.0
    return max(float(np.max(np.abs(x - y))) for x, y in zip(a, b)) / scale


def random_state(n, rng, h=(0.3, 2.0), vel=1.5, dry_prob=0.0):
    hh = rng.uniform(*h, n)
    if dry_prob:
        hh[rng.uniform(0, 1, n) < dry_prob] = 0.0
    return [hh, hh * rng.uniform(-vel, vel, n), hh * rng.uniform(-vel, vel, n)]


def smooth_state(m, amp=0.1):
    x, y = m.arrays["x"], m.arrays["y"]
    h = 1.0 + amp * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y)
    return [h, 0.3 * h, -0.2 * h]


def scenario_params(sid, degree=0, **over):
    c = ref.scenario_config(sid, degree)
    c.update(over)
    return ref.params(g=c["g"], h_tol=c["h_tol"], h_des=c["h_des"], h_ref=c["h_ref"],
                      epsilon0=c["epsilon0"], sigma_min=c["sigma_min"],
                      sigma_max=c["sigma_max"], visc=bool(c["visc_enabled"]),
                      limiter=bool(c["limiter_enabled"])), c


# Mesh configurations covering the hot-path inputs: curved periodic, walls, reversed
# orientation is absent from the structured generators (covered by synthetic meshes).
MESHES = {
    "wavy_N4": dict(kind="wavy", degree=4, kx=6, ky=5, periodic_x=True, periodic_y=True),
    "wavy_N1": dict(kind="wavy", degree=1, kx=5, ky=4, periodic_x=True, periodic_y=True),
    "wavy_N7": dict(kind="wavy", degree=7, kx=3, ky=3, periodic_x=True, periodic_y=True),
    "dam_N4": dict(kind="curved_dam", degree=4, kx=6, ky=5),
    "cart_N3_walls": dict(kind="cartesian", degree=3, kx=4, ky=3, x0=-1.0, x1=1.0,
                          y0=0.0, y1=1.5),
    "cart_1x1_periodic_N2": dict(kind="cartesian", degree=2, kx=1, ky=1, periodic_x=True,
                                 periodic_y=True),
}


def build(name, bathy=("smooth",)):
    spec = dict(MESHES[name])
    kind = spec.pop("kind")
    m = ref.build_mesh(kind, spec.pop("degree"), spec.pop("kx"), spec.pop("ky"), **spec)
    if bathy:
        m.bathymetry(*bathy)
    return m


def reversed_mesh(m):
    """Relabel a mesh so that every interior face's plus element stores its nodes in the
    opposite orientation: rotate the plus elements of the chosen faces by 180 degrees.

    Rotating an element's local frame by 180 degrees maps node (i,j) -> (N-i,N-j),
    faces S<->N, E<->W, negates all metric terms (x_xi, y_xi, x_eta, y_eta) and keeps
    J; face arrays move with their faces (t -> N-t).  Faces incident to a rotated
    element flip their `reversed` flag.  Used to exercise `reversed` and
    non-canonical face numbering, which the structured generators never produce.
    """
    import types
    n1 = m.degree + 1
    np_ = n1 * n1
    a = {k: v.copy() for k, v in m.arrays.items()}
    rot = np.zeros(m.n_elem, bool)
    rot[1::2] = True
    perm = np.arange(np_).reshape(n1, n1)[::-1, ::-1].ravel()
    node_keys = ("x", "y", "x_xi", "x_eta", "y_xi", "y_eta", "jac", "b",
                 "b_yeta", "b_yxi", "b_xeta", "b_xxi")
    for k in node_keys:
        v = a[k].reshape(m.n_elem, np_)
        v[rot] = v[rot][:, perm]
        if k in ("x_xi", "x_eta", "y_xi", "y_eta", "b_yeta", "b_yxi", "b_xeta", "b_xxi"):
            v[rot] = -v[rot]
    fswap = np.array([2, 3, 0, 1])
    for k in ("face_jsurf", "face_nx", "face_ny", "face_a"):
        v = a[k].reshape(m.n_elem, 4, n1)
        old = v[rot].copy()
        v[rot] = old[:, fswap, ::-1]
    faces = m.faces.copy()
    for f in faces:
        em, fm, ep, fp = f[0], f[1], f[2], f[3]
        flip = 0
        if rot[em]:
            f[1] = fswap[fm]
            flip ^= 1
        if f[5] == 0 and rot[ep]:
            f[3] = fswap[fp]
            flip ^= 1
        if f[5] == 0:
            f[4] ^= flip
    # a plain holder: a copy of the RefMesh would share (and double-free) its handle
    out = types.SimpleNamespace(degree=m.degree, n_elem=m.n_elem, n_owned=0, arrays=a,
                                faces=faces, n1=m.n1, n_nodes=m.n_nodes)
    return out, rot, perm
