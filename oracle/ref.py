"""oracle/ref.py — TEST INFRASTRUCTURE ONLY: ctypes view of oracle/_ref/libswdg_ref.so.

The library is the UNMODIFIED reference (`/root/reference/proj/include/swdg`) behind
the C ABI in oracle/ref_capi.cpp.  Only tests/, __graft_entry__.smoke() and bench.py's
reference / cpu_baseline legs may import this module; the product
(`paper_1804_02221_b200`) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libswdg_ref.so")

_dp = C.POINTER(C.c_double)
_lib = None


class Face(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("elem_minus", "face_minus", "elem_plus", "face_plus", "reversed", "tag")]


class Params(C.Structure):
    _fields_ = [("g", C.c_double), ("h_tol", C.c_double), ("h_des", C.c_double),
                ("h_ref", C.c_double), ("epsilon0", C.c_double), ("sigma_min", C.c_double),
                ("sigma_max", C.c_double), ("visc_enabled", C.c_int32),
                ("limiter_enabled", C.c_int32), ("mode", C.c_int32), ("scheme", C.c_int32)]


class StepInfo(C.Structure):
    _fields_ = [("min_stage_h", C.c_double), ("max_eps", C.c_double),
                ("n_limited", C.c_int32), ("accepted", C.c_int32)]


class Diagnostics(C.Structure):
    _fields_ = [("mass", C.c_double), ("entropy", C.c_double), ("min_h", C.c_double),
                ("positivity_dt", C.c_double)]


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref`")
        L = C.CDLL(REF_SO)
        vp = C.c_void_p
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_operators": (C.c_int, [C.c_int] + [_dp] * 7),
            "ref_mesh_build": (vp, [C.c_int] * 4 + [C.c_double] * 4 + [C.c_int, C.c_int, C.c_double]),
            "ref_mesh_bathymetry": (None, [vp, C.c_int, _dp]),
            "ref_scenario_mesh": (vp, [C.c_char_p, C.c_int, C.c_int, C.c_int]),
            "ref_scenario_initial": (C.c_int, [C.c_char_p, vp, _dp, _dp, _dp]),
            "ref_scenario_config": (C.c_int, [C.c_char_p, C.c_int, _dp]),
            "ref_mesh_free": (None, [vp]),
            "ref_mesh_n_elem": (C.c_int, [vp]),
            "ref_mesh_degree": (C.c_int, [vp]),
            "ref_mesh_n_faces": (C.c_int, [vp]),
            "ref_mesh_array": (_dp, [vp, C.c_char_p]),
            "ref_mesh_faces": (None, [vp, C.POINTER(C.c_int32), _dp]),
            "ref_watertightness_gap": (C.c_double, [vp]),
            "ref_assemble_rhs": (C.c_int, [vp, C.POINTER(Params), C.c_int, _dp, _dp, _dp,
                                           C.c_double, _dp, _dp, _dp]),
            "ref_integ_create": (vp, [vp, C.POINTER(Params), C.c_int, _dp]),
            "ref_integ_free": (None, [vp]),
            "ref_integ_try_step": (C.c_int, [vp, _dp, _dp, _dp, C.c_double, C.c_double,
                                             C.POINTER(StepInfo)]),
            "ref_runner_create": (vp, [vp, _dp, _dp, _dp]),
            "ref_runner_steps": (C.c_int, [vp, C.c_int, C.c_double, C.c_double]),
            "ref_runner_free": (None, [vp]),
            "ref_integ_evaluate_rhs": (C.c_int, [vp, _dp, _dp, _dp, C.c_double, _dp, _dp, _dp]),
            "ref_integ_last_eps": (None, [vp, _dp]),
            "ref_compute_dt": (C.c_int, [vp, C.POINTER(Params), _dp, _dp, _dp, C.c_double, _dp]),
            "ref_diagnostics": (C.c_int, [vp, C.POINTER(Params), _dp, _dp, _dp,
                                          C.POINTER(Diagnostics)]),
            "ref_compute_viscosity": (C.c_int, [vp, C.POINTER(Params), _dp, _dp]),
            "ref_shock_indicator": (C.c_double, [C.c_int, _dp]),
            "ref_br1_gradients": (C.c_int, [vp, _dp, _dp, _dp, _dp, _dp, _dp]),
            "ref_viscous_lhs": (C.c_int, [vp] + [_dp] * 10),
            "ref_limit_all": (C.c_int, [vp, C.POINTER(Params), _dp, _dp, _dp, C.c_int, _dp]),
            "ref_mms_error": (C.c_int, [vp, C.POINTER(Params), C.c_double, C.c_double, _dp,
                                        _dp, C.POINTER(C.c_int64)]),
            "ref_volume_kernel": (C.c_int, [C.c_int, C.c_int, C.c_long, C.POINTER(_dp),
                                            C.POINTER(_dp), C.c_double]),
            "ref_count_ops": (C.c_int, [C.c_int, C.c_long, C.POINTER(C.c_uint64)]),
            "ref_bench_rough_state": (C.c_int, [C.c_int, C.c_long, _dp, _dp, _dp]),
            "ref_run_simulation": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_double,
                                             C.c_double, _dp, _dp, _dp,
                                             C.POINTER(C.c_int64), _dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def check(rc: int):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def params(g=9.81, h_tol=1e-4, h_des=1e-8, h_ref=1.0, epsilon0=0.0, sigma_min=0.0,
           sigma_max=0.0, visc=False, limiter=True, mode=0, scheme=0) -> Params:
    """scheme: 0 = SchemeMode::es, 1 = SchemeMode::standard (dg_rhs.hpp:14)."""
    return Params(g, h_tol, h_des, h_ref, epsilon0, sigma_min, sigma_max, int(visc),
                  int(limiter), mode, scheme)


NODE_ARRAYS = ("x", "y", "x_xi", "x_eta", "y_xi", "y_eta", "jac", "b",
               "b_yeta", "b_yxi", "b_xeta", "b_xxi")
FACE_ARRAYS = ("face_jsurf", "face_nx", "face_ny", "face_a")
OP_ARRAYS = ("nodes", "weights", "deriv", "deriv_modified", "deriv_weak", "vandermonde",
             "vandermonde_inv")

MESH_KINDS = {"cartesian": 0, "curved_dam": 1, "wavy": 2}
BATHY_KINDS = {"none": 0, "constant": 1, "linear": 2, "paraboloid": 3, "smooth": 4,
               "step": 5, "sine": 6}


@dataclass
class RefMesh:
    """A reference `swdg::Mesh` plus numpy copies of every array."""

    handle: int
    n_elem: int
    degree: int
    arrays: dict
    faces: np.ndarray  # (n_faces, 6) int32
    offsets: np.ndarray

    @property
    def n1(self):
        return self.degree + 1

    @property
    def n_nodes(self):
        return self.n_elem * self.n1 * self.n1

    def refresh(self):
        L = lib()
        nn, nf = self.n_nodes, 4 * self.n_elem * self.n1
        for k in NODE_ARRAYS:
            self.arrays[k] = np.ctypeslib.as_array(L.ref_mesh_array(self.handle, k.encode()),
                                                   (nn,)).copy()
        for k in FACE_ARRAYS:
            self.arrays[k] = np.ctypeslib.as_array(L.ref_mesh_array(self.handle, k.encode()),
                                                   (nf,)).copy()
        for k in OP_ARRAYS:
            n = self.n1 if k in ("nodes", "weights") else self.n1 * self.n1
            self.arrays[k] = np.ctypeslib.as_array(L.ref_mesh_array(self.handle, k.encode()),
                                                   (n,)).copy()
        nfc = L.ref_mesh_n_faces(self.handle)
        self.faces = np.zeros((nfc, 6), np.int32)
        self.offsets = np.zeros((nfc, 2), np.float64)
        L.ref_mesh_faces(self.handle, self.faces.ctypes.data_as(C.POINTER(C.c_int32)),
                         ptr(self.offsets))
        return self

    def bathymetry(self, kind: str, *p):
        prm = np.zeros(4)
        prm[: len(p)] = p
        lib().ref_mesh_bathymetry(self.handle, BATHY_KINDS[kind], ptr(prm))
        return self.refresh()

    def __del__(self):
        try:
            if self.handle and _lib is not None:
                _lib.ref_mesh_free(self.handle)
        except Exception:
            pass


def _wrap(handle) -> RefMesh:
    if not handle:
        raise RuntimeError(f"reference mesh build failed: {lib().ref_last_error().decode()}")
    L = lib()
    m = RefMesh(handle, L.ref_mesh_n_elem(handle), L.ref_mesh_degree(handle), {}, None, None)
    return m.refresh()


def build_mesh(kind: str, degree: int, kx: int, ky: int, x0=0.0, x1=1.0, y0=0.0, y1=1.0,
               periodic_x=False, periodic_y=False, extra=None) -> RefMesh:
    if extra is None:
        extra = 0.5 if kind == "curved_dam" else 0.04
    if kind == "curved_dam" and (x0, x1, y0, y1) == (0.0, 1.0, 0.0, 1.0):
        x0, x1, y0, y1 = -5.0, 7.5, -5.0, 5.0
    return _wrap(lib().ref_mesh_build(MESH_KINDS[kind], degree, kx, ky, x0, x1, y0, y1,
                                      int(periodic_x), int(periodic_y), extra))


def scenario_mesh(sid: str, kx=0, ky=0, degree=0):
    m = _wrap(lib().ref_scenario_mesh(sid.encode(), kx, ky, degree))
    h, hu, hv = (np.zeros(m.n_nodes) for _ in range(3))
    check(lib().ref_scenario_initial(sid.encode(), m.handle, ptr(h), ptr(hu), ptr(hv)))
    m.refresh()
    return m, (h, hu, hv)


def scenario_config(sid: str, degree=0) -> dict:
    out = np.zeros(12)
    check(lib().ref_scenario_config(sid.encode(), degree, ptr(out)))
    keys = ("g", "h_tol", "h_des", "h_ref", "epsilon0", "sigma_min", "sigma_max",
            "visc_enabled", "limiter_enabled", "cfl", "final_time", "orbital_period")
    return dict(zip(keys, out.tolist()))


def operators(degree: int) -> dict:
    n1 = degree + 1
    out = {k: np.zeros(n1 if k in ("nodes", "weights") else n1 * n1) for k in OP_ARRAYS}
    check(lib().ref_operators(degree, *(ptr(out[k]) for k in OP_ARRAYS)))
    return out


def assemble_rhs(m: RefMesh, p: Params, state, t=0.0, mode=0):
    out = [np.zeros(m.n_nodes) for _ in range(3)]
    check(lib().ref_assemble_rhs(m.handle, C.byref(p), mode, *(ptr(a) for a in state), t,
                                 *(ptr(a) for a in out)))
    return out


def limit_all(m: RefMesh, p: Params, state, zero_dry=True):
    """limit_element (limiter.hpp:43-84) on every element, in place; returns theta."""
    theta = np.zeros(m.n_elem)
    check(lib().ref_limit_all(m.handle, C.byref(p), *(ptr(a) for a in state), int(zero_dry),
                              ptr(theta)))
    return theta


MMS_WAVE = (2.0, 0.2, 0.7, 0.3, 2.0 * np.pi, 9.81)  # validate.hpp:543-546 (h0, amp, u0, v0, k, g)


def mms_error(m: RefMesh, p: Params, cfl=0.4, t_end=0.2, wave=MMS_WAVE):
    """crit_convergence's run (validate.hpp:560-595) on mesh m: (L2(h) error, steps)."""
    fp = np.array(wave, np.float64)
    err, steps = C.c_double(), C.c_int64()
    check(lib().ref_mms_error(m.handle, C.byref(p), cfl, t_end, ptr(fp), C.byref(err),
                              C.byref(steps)))
    return err.value, steps.value


def volume_kernel(kind: int, degree: int, k: int, inputs, g=9.81):
    """the reference's split (0) / standard (1) volume kernel, out = 0 + term"""
    ins = (_dp * 7)(*(ptr(a) for a in inputs))
    out = [np.zeros(k * (degree + 1) ** 2) for _ in range(3)]
    outs = (_dp * 3)(*(ptr(a) for a in out))
    check(lib().ref_volume_kernel(kind, degree, k, ins, outs, g))
    return out


def count_ops(degree: int, k: int):
    """bench::count_ops: (evals_split, evals_std, flops_split, flops_std)"""
    o = (C.c_uint64 * 4)()
    check(lib().ref_count_ops(degree, k, o))
    return tuple(int(x) for x in o)


def bench_rough_state(degree: int, n_elem: int):
    """bench.hpp:108-121: the mt19937(20250810) rough field the reference benchmarks on."""
    n = n_elem * (degree + 1) ** 2
    out = [np.zeros(n) for _ in range(3)]
    check(lib().ref_bench_rough_state(degree, n_elem, *(ptr(a) for a in out)))
    return out


def compute_dt(m: RefMesh, p: Params, state, cfl):
    dt = C.c_double()
    check(lib().ref_compute_dt(m.handle, C.byref(p), *(ptr(a) for a in state), cfl,
                               C.byref(dt)))
    return dt.value


def diagnostics(m: RefMesh, p: Params, state) -> Diagnostics:
    d = Diagnostics()
    check(lib().ref_diagnostics(m.handle, C.byref(p), *(ptr(a) for a in state), C.byref(d)))
    return d


class Integrator:
    """reference TimeIntegrator (timeloop.hpp:146) on a RefMesh."""

    def __init__(self, m: RefMesh, p: Params, forcing=None):
        self.mesh = m
        fk, fp = 0, np.zeros(8)
        if forcing is not None:
            fk = 1
            fp[:6] = forcing
        self._fp = fp
        self.h = lib().ref_integ_create(m.handle, C.byref(p), fk, ptr(fp))
        if not self.h:
            raise RuntimeError(lib().ref_last_error().decode())

    def try_step(self, state, t, dt) -> StepInfo:
        info = StepInfo()
        check(lib().ref_integ_try_step(self.h, *(ptr(a) for a in state), t, dt,
                                       C.byref(info)))
        return info

    def evaluate_rhs(self, state, t=0.0):
        out = [np.zeros(self.mesh.n_nodes) for _ in range(3)]
        check(lib().ref_integ_evaluate_rhs(self.h, *(ptr(a) for a in state), t,
                                           *(ptr(a) for a in out)))
        return out

    def last_eps(self):
        e = np.zeros(self.mesh.n_elem)
        lib().ref_integ_last_eps(self.h, ptr(e))
        return e

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.ref_integ_free(self.h)
        except Exception:
            pass


def run_simulation(sid: str, kx=0, ky=0, degree=0, final_time=0.0, cfl=0.0):
    m, _ = scenario_mesh(sid, kx, ky, degree)
    out = [np.zeros(m.n_nodes) for _ in range(3)]
    steps, t = C.c_int64(), C.c_double()
    check(lib().ref_run_simulation(sid.encode(), kx, ky, degree, final_time, cfl,
                                   *(ptr(a) for a in out), C.byref(steps), C.byref(t)))
    return out, steps.value, t.value


def fnv1a_state(state) -> str:
    """FNV-1a over the 64-bit words of h||hu||hv (the SURVEY fact-4 fingerprints)."""
    h = 1469598103934665603
    for a in state:
        for w in np.ascontiguousarray(a, np.float64).view(np.uint64).tolist():
            h ^= w
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"
