"""oracle/port.py — TEST INFRASTRUCTURE ONLY: ctypes view of the plain-C restatement
(oracle/swdg_port.c -> oracle/_build/libswdg_port.so).

Mesh arguments are any object exposing ``degree``, ``n_elem``, ``faces`` ((F,6) int32),
``arrays`` (dict of numpy float64 arrays with the reference MeshGeometry/Operators1D
names) and optionally ``n_owned``.  Only tests/, smoke() and bench.py's cpu_baseline
leg may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .ref import Diagnostics, Params, StepInfo, params  # noqa: F401  (shared POD layouts)

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libswdg_port.so")
_dp = C.POINTER(C.c_double)
_lib = None


class FaceC(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("elem_minus", "face_minus", "elem_plus", "face_plus", "reversed", "tag")]


class MeshViewC(C.Structure):
    """swdg_mesh_view (include/swdg_gpu.h)."""

    _fields_ = [("n_elem", C.c_int32), ("degree", C.c_int32), ("n_owned", C.c_int32),
                ("n_faces", C.c_int32), ("faces", C.c_void_p)] + [
        (k, _dp) for k in ("weights", "deriv", "deriv_modified", "deriv_weak",
                           "vandermonde_inv", "x", "y", "x_xi", "x_eta", "y_xi", "y_eta",
                           "jac", "b", "face_jsurf", "face_nx", "face_ny", "face_a")]


def build():
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(PORT_SO):
            build()
        L = C.CDLL(PORT_SO)
        mv = C.POINTER(MeshViewC)
        pp = C.POINTER(Params)
        sig = {
            "port_last_error": (C.c_char_p, []),
            "port_assemble_rhs": (C.c_int, [mv, pp] + [_dp] * 11),
            "port_shock_indicator": (C.c_double, [C.c_int, _dp, _dp, C.POINTER(C.c_int)]),
            "port_viscosity_coefficient": (C.c_double, [C.c_double, pp, C.POINTER(C.c_int)]),
            "port_compute_viscosity": (C.c_int, [mv, pp, _dp, _dp]),
            "port_velocities": (None, [mv, pp] + [_dp] * 5),
            "port_br1_gradients": (C.c_int, [mv] + [_dp] * 6),
            "port_viscous_fluxes": (C.c_int, [mv] + [_dp] * 10),
            "port_viscous_lhs": (C.c_int, [mv] + [_dp] * 6),
            "port_evaluate_rhs": (C.c_int, [mv, pp] + [_dp] * 10),
            "port_element_average": (None, [mv, _dp, _dp, _dp, C.c_int, _dp, _dp]),
            "port_post_stage": (C.c_int, [mv, pp, _dp, _dp, _dp, C.POINTER(C.c_int), _dp]),
            "port_try_step": (C.c_int, [mv, pp, _dp, _dp, _dp, C.c_double, C.c_double,
                                        C.c_int, _dp, C.POINTER(StepInfo)]),
            "port_compute_dt": (C.c_int, [mv, pp, _dp, _dp, _dp, C.c_double, _dp]),
            "port_diagnostics": (C.c_int, [mv, pp, _dp, _dp, _dp, C.POINTER(Diagnostics)]),
            "port_es_flux": (C.c_int, [_dp, _dp, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_double, _dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(_dp)


def check(rc):
    if rc != 0:
        raise RuntimeError(f"port error {rc}: {lib().port_last_error().decode()}")


class View:
    """Keeps the numpy arrays alive behind a swdg_mesh_view."""

    def __init__(self, mesh):
        a = mesh.arrays
        self.faces = np.ascontiguousarray(mesh.faces, np.int32)
        self.keep = {k: np.ascontiguousarray(a[k], np.float64) for k in
                     ("weights", "deriv", "deriv_modified", "deriv_weak", "vandermonde_inv",
                      "x", "y", "x_xi", "x_eta", "y_xi", "y_eta", "jac", "b",
                      "face_jsurf", "face_nx", "face_ny", "face_a")}
        self.c = MeshViewC(mesh.n_elem, mesh.degree, getattr(mesh, "n_owned", 0) or 0,
                           len(self.faces), self.faces.ctypes.data,
                           *(ptr(self.keep[k]) for k in (
                               "weights", "deriv", "deriv_modified", "deriv_weak",
                               "vandermonde_inv", "x", "y", "x_xi", "x_eta", "y_xi", "y_eta",
                               "jac", "b", "face_jsurf", "face_nx", "face_ny", "face_a")))
        self.n_nodes = mesh.n_elem * (mesh.degree + 1) ** 2
        self.n_elem = mesh.n_elem


def _view(mesh):
    return mesh if isinstance(mesh, View) else View(mesh)


def _zeros(n, k=3):
    return [np.zeros(n) for _ in range(k)]


def assemble_rhs(mesh, p, state, visc=None, forcing=None):
    v = _view(mesh)
    out = _zeros(v.n_nodes)
    vh = visc if visc is not None else (None, None)
    fh = forcing if forcing is not None else (None, None, None)
    check(lib().port_assemble_rhs(C.byref(v.c), C.byref(p), *(ptr(a) for a in state),
                                  *(ptr(a) for a in vh), *(ptr(a) for a in fh),
                                  *(ptr(a) for a in out)))
    return out


def evaluate_rhs(mesh, p, state, forcing=None):
    v = _view(mesh)
    out = _zeros(v.n_nodes)
    eps = np.zeros(v.n_elem)
    fh = forcing if forcing is not None else (None, None, None)
    check(lib().port_evaluate_rhs(C.byref(v.c), C.byref(p), *(ptr(a) for a in state),
                                  *(ptr(a) for a in fh), *(ptr(a) for a in out), ptr(eps)))
    return out, eps


def compute_viscosity(mesh, p, h):
    v = _view(mesh)
    eps = np.zeros(v.n_elem)
    check(lib().port_compute_viscosity(C.byref(v.c), C.byref(p), ptr(h), ptr(eps)))
    return eps


def velocities(mesh, p, state):
    v = _view(mesh)
    u, w = _zeros(v.n_nodes, 2)
    lib().port_velocities(C.byref(v.c), C.byref(p), *(ptr(a) for a in state), ptr(u), ptr(w))
    return u, w


def br1_gradients(mesh, u, w):
    v = _view(mesh)
    out = _zeros(v.n_nodes, 4)
    check(lib().port_br1_gradients(C.byref(v.c), ptr(u), ptr(w), *(ptr(a) for a in out)))
    return out


def viscous_fluxes(mesh, h, grads, eps):
    v = _view(mesh)
    out = _zeros(v.n_nodes, 4)
    check(lib().port_viscous_fluxes(C.byref(v.c), ptr(h), *(ptr(a) for a in grads), ptr(eps),
                                    *(ptr(a) for a in out)))
    return out  # fvu, fvv, gvu, gvv


def viscous_lhs(mesh, fluxes):
    v = _view(mesh)
    out = _zeros(v.n_nodes, 2)
    check(lib().port_viscous_lhs(C.byref(v.c), *(ptr(a) for a in fluxes),
                                 *(ptr(a) for a in out)))
    return out


def post_stage(mesh, p, state):
    v = _view(mesh)
    nl, mh = C.c_int(0), C.c_double(np.inf)
    ok = lib().port_post_stage(C.byref(v.c), C.byref(p), *(ptr(a) for a in state),
                               C.byref(nl), C.byref(mh))
    return ok, nl.value, mh.value


def try_step(mesh, p, state, t, dt, forcing=None) -> StepInfo:
    v = _view(mesh)
    info = StepInfo()
    fp = np.zeros(8)
    fk = 0
    if forcing is not None:
        fk = 1
        fp[:6] = forcing
    rc = lib().port_try_step(C.byref(v.c), C.byref(p), *(ptr(a) for a in state), t, dt, fk,
                             ptr(fp), C.byref(info))
    if rc == 3:
        raise ArithmeticError(lib().port_last_error().decode())
    check(rc)
    return info


def compute_dt(mesh, p, state, cfl):
    v = _view(mesh)
    dt = C.c_double()
    check(lib().port_compute_dt(C.byref(v.c), C.byref(p), *(ptr(a) for a in state), cfl,
                                C.byref(dt)))
    return dt.value


def diagnostics(mesh, p, state) -> Diagnostics:
    v = _view(mesh)
    d = Diagnostics()
    check(lib().port_diagnostics(C.byref(v.c), C.byref(p), *(ptr(a) for a in state),
                                 C.byref(d)))
    return d


def es_flux(wm, wp, bm, bp, nx, ny, g, h_des=1e-8):
    out = np.zeros(3)
    a, b = np.asarray(wm, np.float64), np.asarray(wp, np.float64)
    check(lib().port_es_flux(ptr(a), ptr(b), bm, bp, nx, ny, g, h_des, ptr(out)))
    return out
