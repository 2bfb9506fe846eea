"""Python host side of the B200 stage path, mirroring the reference's C++ surface.

The reference (`/root/reference/proj/include/swdg`) is a header-only C++ library;
its stage-path seams are `TimeIntegrator` (timeloop.hpp:146-262), `assemble_rhs`
(dg_rhs.hpp:267), `compute_dt` (timeloop.hpp:53) and the diagnostics of
field.hpp:39-68 / limiter.hpp:135.  This module exposes the same names with the
same argument meaning and error behaviour (`SwdgError`, `NumericalAbort`), backed
by the sm_100a kernels through the C ABI in include/swdg_gpu.h
(`_lib/libswdg_gpu.so`).  There is no CPU fallback: without the built library or a
CUDA device every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SWDG_LIB") or os.path.join(_PKG, "_lib", "libswdg_gpu.so")
_dp = C.POINTER(C.c_double)

SWDG_OK, SWDG_ERR_CUDA, SWDG_ERR_INPUT, SWDG_ERR_ABORT = 0, 1, 2, 3
MODE_EXACT, MODE_FAST = 0, 1
SCHEME_ES, SCHEME_STANDARD = 0, 1  # SchemeMode (dg_rhs.hpp:14)
TAG_INTERIOR, TAG_WALL = 0, 1


class SwdgError(RuntimeError):
    """core.hpp:63 SwdgError (bad input/config)."""


class NumericalAbort(SwdgError):
    """timeloop.hpp:46 NumericalAbort (limiter off and a negative height)."""


class CudaError(RuntimeError):
    """Device/runtime failure (no reference counterpart)."""


# ---------------------------------------------------------------- C structs
class FaceC(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("elem_minus", "face_minus", "elem_plus", "face_plus", "reversed", "tag")]


_VIEW_PTRS = ("weights", "deriv", "deriv_modified", "deriv_weak", "vandermonde_inv",
              "x", "y", "x_xi", "x_eta", "y_xi", "y_eta", "jac", "b",
              "face_jsurf", "face_nx", "face_ny", "face_a")


class MeshViewC(C.Structure):
    _fields_ = [("n_elem", C.c_int32), ("degree", C.c_int32), ("n_owned", C.c_int32),
                ("n_faces", C.c_int32), ("faces", C.c_void_p)] + [(k, _dp) for k in _VIEW_PTRS]


class ParamsC(C.Structure):
    _fields_ = [("g", C.c_double), ("h_tol", C.c_double), ("h_des", C.c_double),
                ("h_ref", C.c_double), ("epsilon0", C.c_double), ("sigma_min", C.c_double),
                ("sigma_max", C.c_double), ("visc_enabled", C.c_int32),
                ("limiter_enabled", C.c_int32), ("mode", C.c_int32), ("scheme", C.c_int32)]


class StepInfoC(C.Structure):
    _fields_ = [("min_stage_h", C.c_double), ("max_eps", C.c_double),
                ("n_limited", C.c_int32), ("accepted", C.c_int32)]


class DiagnosticsC(C.Structure):
    _fields_ = [("mass", C.c_double), ("entropy", C.c_double), ("min_h", C.c_double),
                ("positivity_dt", C.c_double)]


class StepReportC(C.Structure):
    _fields_ = [("info", StepInfoC), ("diag", DiagnosticsC), ("next_dt", C.c_double)]


class StructuredSpecC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("degree", C.c_int32), ("kx", C.c_int32), ("ky", C.c_int32),
                ("periodic_x", C.c_int32), ("periodic_y", C.c_int32),
                ("bathy_kind", C.c_int32), ("reserved", C.c_int32),
                ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
                ("extra", C.c_double), ("bathy", C.c_double * 4)]


MESH_KINDS = {"cartesian": 0, "curved_dam": 1, "wavy": 2}
BATHY_KINDS = {"none": 0, "constant": 1, "linear": 2, "paraboloid": 3, "smooth": 4,
               "step": 5, "sine": 6}


def structured_spec(kind: str, degree: int, kx: int, ky: int, x0=0.0, x1=1.0, y0=0.0, y1=1.0,
                    periodic_x=False, periodic_y=False, extra=None, bathy="none",
                    bathy_params=()) -> StructuredSpecC:
    """Generator spec of build_cartesian/curved_dam/wavy_mesh (mesh.hpp:342-379)."""
    if extra is None:
        extra = 0.5 if kind == "curved_dam" else 0.04
    if kind == "curved_dam" and (x0, x1, y0, y1) == (0.0, 1.0, 0.0, 1.0):
        x0, x1, y0, y1 = -5.0, 7.5, -5.0, 5.0
    bp = (C.c_double * 4)(*(list(bathy_params) + [0.0] * (4 - len(bathy_params))))
    return StructuredSpecC(MESH_KINDS[kind], degree, kx, ky, int(periodic_x), int(periodic_y),
                           BATHY_KINDS[bathy], 0, x0, x1, y0, y1, extra, bp)


def operators(degree: int) -> dict:
    """make_operators (operators.hpp:148) from the host library (no device needed)."""
    n1 = degree + 1
    keys = ("nodes", "weights", "deriv", "deriv_modified", "deriv_weak", "vandermonde",
            "vandermonde_inv")
    out = {k: np.zeros(n1 if k in ("nodes", "weights") else n1 * n1) for k in keys}
    rc = lib().swdg_operators(degree, *(_ptr(out[k]) for k in keys))
    if rc != SWDG_OK:
        raise SwdgError("swdg_operators: degree must be in [1, 15]")
    return out


def structured_faces(kx: int, ky: int, periodic_x=False, periodic_y=False) -> np.ndarray:
    """structured_topology (mesh.hpp:237-290) as an (F, 6) int32 table."""
    n = lib().swdg_structured_face_count(kx, ky, int(periodic_x), int(periodic_y))
    out = np.zeros((n, 6), np.int32)
    lib().swdg_structured_faces(kx, ky, int(periodic_x), int(periodic_y), out.ctypes.data)
    return out


FORCING_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_double, C.c_int64, _dp, _dp, _dp, _dp, _dp)

_lib = None


def lib():
    """Load libswdg_gpu.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        sig = {
            "swdg_gpu_create": (C.c_int, [C.POINTER(MeshViewC), C.POINTER(ParamsC), C.c_int,
                                          C.POINTER(vp)]),
            "swdg_gpu_create_error": (C.c_char_p, []),
            "swdg_gpu_destroy": (None, [vp]),
            "swdg_gpu_last_error": (C.c_char_p, [vp]),
            "swdg_gpu_set_stream": (C.c_int, [vp, vp]),
            "swdg_gpu_synchronize": (C.c_int, [vp]),
            "swdg_gpu_upload_state": (C.c_int, [vp, _dp, _dp, _dp]),
            "swdg_gpu_download_state": (C.c_int, [vp, _dp, _dp, _dp]),
            "swdg_gpu_device_state": (C.c_int, [vp, C.POINTER(_dp), C.POINTER(_dp),
                                                C.POINTER(_dp)]),
            "swdg_gpu_evaluate_rhs": (C.c_int, [vp, C.c_double, _dp, _dp, _dp]),
            "swdg_gpu_assemble_rhs": (C.c_int, [vp, C.c_double, _dp, _dp, _dp]),
            "swdg_gpu_compute_dt": (C.c_int, [vp, C.c_double, _dp]),
            "swdg_gpu_try_step": (C.c_int, [vp, C.c_double, C.c_double, C.POINTER(StepInfoC)]),
            "swdg_gpu_run_steps": (C.c_int, [vp, C.c_int, C.c_double, C.c_double]),
            "swdg_gpu_last_info": (C.c_int, [vp, C.POINTER(StepInfoC)]),
            "swdg_gpu_last_eps": (C.c_int, [vp, _dp]),
            "swdg_gpu_diagnostics": (C.c_int, [vp, C.POINTER(DiagnosticsC)]),
            "swdg_gpu_set_forcing": (C.c_int, [vp, FORCING_FN, vp]),
            "swdg_gpu_launch_count": (C.c_int64, [vp]),
            "swdg_operators": (C.c_int, [C.c_int] + [_dp] * 7),
            "swdg_structured_face_count": (C.c_int64, [C.c_int] * 4),
            "swdg_structured_faces": (C.c_int, [C.c_int] * 4 + [vp]),
            "swdg_gpu_create_structured": (C.c_int, [C.POINTER(StructuredSpecC),
                                                     C.POINTER(ParamsC), C.c_int,
                                                     C.POINTER(vp)]),
            "swdg_gpu_download_geometry": (C.c_int, [vp, C.c_char_p, _dp]),
            "swdg_gpu_step_device": (C.c_int, [vp, C.c_double, C.c_double, C.c_double,
                                               C.POINTER(StepReportC)]),
            "swdg_gpu_set_track_limiter_entropy": (C.c_int, [vp, C.c_int]),
            "swdg_gpu_worst_limiter_entropy_jump": (C.c_int, [vp, _dp]),
            "swdg_gpu_upload_stage_input": (C.c_int, [vp, C.c_int, _dp, _dp, _dp]),
            "swdg_gpu_download_stage_output": (C.c_int, [vp, C.c_int, _dp, _dp, _dp]),
            "swdg_gpu_stage_info": (C.c_int, [vp, C.c_int, C.POINTER(StepInfoC)]),
            "swdg_gpu_step_begin": (C.c_int, [vp]),
            "swdg_gpu_stage_visc": (C.c_int, [vp, C.c_int, C.c_double, C.c_double]),
            "swdg_gpu_stage_run": (C.c_int, [vp, C.c_int, C.c_double, C.c_double]),
            "swdg_gpu_set_grid_cap": (C.c_int, [C.c_int32]),
            "swdg_gpu_run_steps_ex": (C.c_int, [vp, C.c_int, C.c_double, C.c_double, C.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    """Entry points declared in include/swdg_gpu.h."""
    import re
    hdr = os.path.join(os.path.dirname(_PKG), "include", "swdg_gpu.h")
    with open(hdr) as f:
        return sorted(set(re.findall(r"\b(swdg_gpu_\w+)\s*\(", f.read())))


def _ptr(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


# ---------------------------------------------------------------- config
@dataclass
class PhysicsParams:
    """physics.hpp:11-16"""
    g: float = 9.81
    h_tol: float = 1e-4
    h_des: float = 1e-8
    h_ref: float = 1.0


@dataclass
class ViscosityConfig:
    """viscosity.hpp:14-19"""
    enabled: bool = False
    epsilon0: float = 0.0
    sigma_min: float = 0.0
    sigma_max: float = 0.0


def default_sigma_band(degree: int):
    """viscosity.hpp:23-26"""
    smin = -(4.0 + 4.25 * np.log10(float(degree))) - 1.0
    return smin, smin + 2.0


@dataclass
class RunConfig:
    """The stage-relevant fields of timeloop.hpp:23-44 RunConfig (+ the GPU mode)."""
    phys: PhysicsParams = field(default_factory=PhysicsParams)
    visc: ViscosityConfig = field(default_factory=ViscosityConfig)
    limiter_enabled: bool = True
    mode: int = MODE_EXACT
    # SchemeMode (dg_rhs.hpp:14): SCHEME_ES, or SCHEME_STANDARD (standard DGSEM + LLF,
    # no artificial viscosity, always on the exact kernels)
    scheme: int = 0

    def c_params(self) -> ParamsC:
        return ParamsC(self.phys.g, self.phys.h_tol, self.phys.h_des, self.phys.h_ref,
                       self.visc.epsilon0, self.visc.sigma_min, self.visc.sigma_max,
                       int(self.visc.enabled), int(self.limiter_enabled), int(self.mode),
                       int(self.scheme))


# ---------------------------------------------------------------- mesh / state
class Mesh:
    """Host copy of a reference `swdg::Mesh` (mesh.hpp:101-112) in the reference layout.

    `arrays` carries Operators1D and MeshGeometry arrays by their reference names;
    `faces` is MeshTopology::faces as an (F, 6) int32 table
    (elem_minus, face_minus, elem_plus, face_plus, reversed, tag).
    """

    def __init__(self, degree: int, n_elem: int, arrays: dict, faces, n_owned: int = 0):
        self.degree = int(degree)
        self.n_elem = int(n_elem)
        self.n_owned = int(n_owned)
        self.arrays = {k: np.ascontiguousarray(v, np.float64) for k, v in arrays.items()}
        self.faces = np.ascontiguousarray(faces, np.int32).reshape(-1, 6)

    @classmethod
    def from_any(cls, m) -> "Mesh":
        if isinstance(m, Mesh):
            return m
        return cls(m.degree, m.n_elem, m.arrays, m.faces, getattr(m, "n_owned", 0) or 0)

    @property
    def n1(self):
        return self.degree + 1

    @property
    def np_(self):
        return self.n1 * self.n1

    @property
    def n_nodes(self):
        return self.n_elem * self.np_

    def view(self) -> MeshViewC:
        a = self.arrays
        missing = [k for k in _VIEW_PTRS if k not in a and k not in ("x", "y")]
        if missing:
            raise SwdgError(f"mesh is missing arrays {missing}")
        return MeshViewC(self.n_elem, self.degree, self.n_owned, len(self.faces),
                         self.faces.ctypes.data,
                         *(_ptr(a[k]) if k in a else None for k in _VIEW_PTRS))


class _DeviceMesh:
    """Shape-only stand-in for a mesh generated on the device; arrays download lazily."""

    def __init__(self, degree: int, n_elem: int):
        self.degree = degree
        self.n_elem = n_elem
        self.n_owned = 0
        self.owner = None
        self._arrays = {}

    @property
    def n1(self):
        return self.degree + 1

    @property
    def n_nodes(self):
        return self.n_elem * self.n1 * self.n1

    @property
    def arrays(self):
        class _Lazy(dict):
            def __missing__(d, k):
                d[k] = self.owner.geometry(k)
                return d[k]
        if not isinstance(self._arrays, _Lazy):
            self._arrays = _Lazy(self._arrays)
        return self._arrays


class State:
    """field.hpp:12-34: nodal (h, hu, hv), element-major."""

    def __init__(self, h, hu, hv):
        self.h = np.ascontiguousarray(h, np.float64)
        self.hu = np.ascontiguousarray(hu, np.float64)
        self.hv = np.ascontiguousarray(hv, np.float64)

    def arrays(self):
        return self.h, self.hu, self.hv

    def copy(self):
        return State(self.h.copy(), self.hu.copy(), self.hv.copy())


def _raise(code: int, msg: str):
    if code == SWDG_ERR_ABORT:
        raise NumericalAbort(msg)
    if code == SWDG_ERR_INPUT:
        raise SwdgError(msg)
    raise CudaError(msg)


# ---------------------------------------------------------------- integrator
class TimeIntegrator:
    """timeloop.hpp:146-262 on the GPU: one SSPRK3 step per `try_step`.

    `try_step(state, t, dt)` follows the reference contract: it returns False and
    leaves `state` untouched when a stage produces a negative element mean, raises
    NumericalAbort when the limiter is disabled and a stage goes negative, and
    otherwise overwrites `state` with the new one.  Every call uploads the caller's host
    state first, exactly like the reference reads its State argument; the
    device-resident throughput entry is `run_steps`.
    """

    def __init__(self, mesh, cfg: RunConfig, device: int = 0, _handle=None):
        self.cfg = cfg
        if _handle is None:
            self.mesh = Mesh.from_any(mesh)
            self._view = self.mesh.view()  # keeps pointers alive for the create call
            p = cfg.c_params()
            h = C.c_void_p()
            rc = lib().swdg_gpu_create(C.byref(self._view), C.byref(p), device, C.byref(h))
            if rc != SWDG_OK:
                _raise(rc, lib().swdg_gpu_create_error().decode())
            self._h = h
        else:
            self.mesh = mesh
            self._h = _handle
        self._resident = None  # id of the State mirrored on the device
        self._info = StepInfoC()
        self._forcing = None
        self._forcing_c = None
        self.forcing: Optional[Callable] = None

    @classmethod
    def structured(cls, spec: StructuredSpecC, cfg: RunConfig, device: int = 0):
        """Context over a device-generated structured mesh (swdg_gpu_create_structured)."""
        p = cfg.c_params()
        h = C.c_void_p()
        rc = lib().swdg_gpu_create_structured(C.byref(spec), C.byref(p), device, C.byref(h))
        if rc != SWDG_OK:
            _raise(rc, lib().swdg_gpu_create_error().decode())
        integ = cls(_DeviceMesh(spec.degree, spec.kx * spec.ky), cfg, device, _handle=h)
        integ.mesh.owner = integ
        return integ

    @classmethod
    def structured_part(cls, spec: StructuredSpecC, cfg: RunConfig, global_ids, n_owned: int,
                        local_faces, device: int = 0):
        """One partition of a device-generated structured mesh (owned + ghost elements)."""
        L = lib()
        f = L.swdg_gpu_create_structured_part
        f.restype = C.c_int
        f.argtypes = [C.POINTER(StructuredSpecC), C.POINTER(ParamsC), C.c_int, C.c_int32,
                      C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]
        gids = np.ascontiguousarray(global_ids, np.int32)
        faces = np.ascontiguousarray(local_faces, np.int32).reshape(-1, 6)
        p = cfg.c_params()
        h = C.c_void_p()
        rc = f(C.byref(spec), C.byref(p), device, len(gids), n_owned, gids.ctypes.data,
               len(faces), faces.ctypes.data, C.byref(h))
        if rc != SWDG_OK:
            _raise(rc, L.swdg_gpu_create_error().decode())
        m = _DeviceMesh(spec.degree, len(gids))
        m.n_owned = n_owned
        integ = cls(m, cfg, device, _handle=h)
        m.owner = integ
        return integ

    def geometry(self, name: str) -> np.ndarray:
        """Device geometry array (nodal or face layout) copied to host."""
        n = self.mesh.n_nodes
        if name.startswith("face_"):
            n = self.mesh.n_elem * 4 * (self.mesh.degree + 1)
        out = np.empty(n)
        self._check(lib().swdg_gpu_download_geometry(self._h, name.encode(), _ptr(out)))
        return out

    # -- plumbing
    def _check(self, rc):
        if rc != SWDG_OK:
            _raise(rc, lib().swdg_gpu_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            lib().swdg_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, state: State):
        self._check(lib().swdg_gpu_upload_state(self._h, *(_ptr(a) for a in state.arrays())))
        self._resident = id(state)

    def download(self, state: State):
        self._check(lib().swdg_gpu_download_state(self._h, *(_ptr(a) for a in state.arrays())))

    def _sync_forcing(self):
        if self.forcing is self._forcing:
            return
        self._forcing = self.forcing
        if self.forcing is None:
            self._forcing_c = None
            self._check(lib().swdg_gpu_set_forcing(self._h, FORCING_FN(), None))
            return
        fn = self.forcing
        x, y = self.mesh.arrays["x"], self.mesh.arrays["y"]

        def cb(user, t, count, xp, yp, fh, fhu, fhv):
            outs = [np.ctypeslib.as_array(p, (count,)) for p in (fh, fhu, fhv)]
            res = fn(x, y, t)  # vectorised ForcingFn: returns (fh, fhu, fhv) arrays
            for o, r in zip(outs, res):
                o[:] = r

        self._forcing_c = FORCING_FN(cb)
        self._check(lib().swdg_gpu_set_forcing(self._h, self._forcing_c, None))

    # -- reference surface
    def try_step(self, state: State, t: float, dt: float) -> bool:
        self._sync_forcing()
        self.upload(state)
        self._check(lib().swdg_gpu_try_step(self._h, t, dt, C.byref(self._info)))
        if self._info.accepted:
            self.download(state)
        return bool(self._info.accepted)

    def evaluate_rhs(self, state: State, t: float = 0.0) -> State:
        self._sync_forcing()
        self.upload(state)
        out = State(*(np.empty(self.mesh.n_nodes) for _ in range(3)))
        self._check(lib().swdg_gpu_evaluate_rhs(self._h, t, *(_ptr(a) for a in out.arrays())))
        return out

    def assemble_rhs(self, state: State, t: float = 0.0) -> State:
        self.upload(state)
        out = State(*(np.empty(self.mesh.n_nodes) for _ in range(3)))
        self._check(lib().swdg_gpu_assemble_rhs(self._h, t, *(_ptr(a) for a in out.arrays())))
        return out

    def compute_dt(self, state: State, cfl: float) -> float:
        self.upload(state)
        dt = C.c_double()
        self._check(lib().swdg_gpu_compute_dt(self._h, cfl, C.byref(dt)))
        return dt.value

    def diagnostics(self, state: State) -> DiagnosticsC:
        self.upload(state)
        d = DiagnosticsC()
        self._check(lib().swdg_gpu_diagnostics(self._h, C.byref(d)))
        return d

    def run_steps(self, nsteps: int, t: float, dt: float, reductions: bool = False) -> bool:
        """Device-resident SSPRK3 steps with fixed dt (no host synchronisation);
        `reductions` adds the per-step StepDiagnostics reductions and the next CFL
        candidate on the device after every step.

        Returns True when every stage of every step kept all element means
        nonnegative.  On False the device state is UNDEFINED (the steps after the
        rejecting one ran on from its output): re-upload before reusing it."""
        self._check(lib().swdg_gpu_run_steps_ex(self._h, nsteps, t, dt, 1 if reductions else 0))
        return bool(self.last_info().accepted)

    def step_device(self, t: float, dt: float, cfl: float):
        """One run_simulation loop body on the device state (driver.hpp:91-127):
        try_step, then, if accepted, the step diagnostics of the new state and its
        compute_dt(cfl), with one host synchronisation in fast mode.  Returns the
        StepReportC (info, diag, next_dt); `info.accepted` False leaves W^n."""
        self._sync_forcing()
        r = StepReportC()
        self._check(lib().swdg_gpu_step_device(self._h, t, dt, cfl, C.byref(r)))
        self._info = r.info
        return r

    # -- track_limiter_entropy (timeloop.hpp:196-199)
    @property
    def track_limiter_entropy(self) -> bool:
        return bool(getattr(self, "_track", False))

    @track_limiter_entropy.setter
    def track_limiter_entropy(self, on: bool):
        self._check(lib().swdg_gpu_set_track_limiter_entropy(self._h, int(bool(on))))
        self._track = bool(on)

    def worst_limiter_entropy_jump(self) -> float:
        v = C.c_double()
        self._check(lib().swdg_gpu_worst_limiter_entropy_jump(self._h, C.byref(v)))
        return v.value

    # -- one stage of the split step (parity tests, partitioned runs)
    def run_stage(self, k: int, wn: State, w_in: State | None, t: float, dt: float) -> State:
        """Run SSPRK3 stage k (0, 1, 2) of a step at time t with W^n = `wn` and stage
        input `w_in` (None: W^n, stage 0) through the fused stage kernels and return
        the kernel-written stage output (update, combine, limiter, dry-node cut)."""
        L = lib()
        self._sync_forcing()
        self.upload(wn)
        if k > 0:
            self._check(L.swdg_gpu_upload_stage_input(self._h, k, *(_ptr(a) for a in w_in.arrays())))
        self._check(L.swdg_gpu_step_begin(self._h))
        self._check(L.swdg_gpu_stage_visc(self._h, k, t, dt))
        self._check(L.swdg_gpu_stage_run(self._h, k, t, dt))
        out = State(*(np.empty(self.mesh.n_nodes) for _ in range(3)))
        self._check(L.swdg_gpu_download_stage_output(self._h, k, *(_ptr(a) for a in out.arrays())))
        return out

    def stage_info(self, k: int) -> StepInfoC:
        info = StepInfoC()
        self._check(lib().swdg_gpu_stage_info(self._h, k, C.byref(info)))
        return info

    def last_info(self) -> StepInfoC:
        info = StepInfoC()
        self._check(lib().swdg_gpu_last_info(self._h, C.byref(info)))
        return info

    def try_step_device(self, t: float, dt: float) -> bool:
        """try_step of the device-resident state (no host copies): on a reject the
        state stays W^n on the device (the stage buffers are discarded)."""
        self._sync_forcing()
        self._check(lib().swdg_gpu_try_step(self._h, t, dt, C.byref(self._info)))
        return bool(self._info.accepted)

    def diagnostics_device(self) -> DiagnosticsC:
        """mass, entropy, min h and the positivity bound of the device-resident state"""
        d = DiagnosticsC()
        self._check(lib().swdg_gpu_diagnostics(self._h, C.byref(d)))
        return d

    def compute_dt_device(self, cfl: float) -> float:
        """compute_dt of the device-resident state (no upload)."""
        dt = C.c_double()
        self._check(lib().swdg_gpu_compute_dt(self._h, cfl, C.byref(dt)))
        return dt.value

    def set_stream(self, stream_handle: int | None):
        """Launch on an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream;
        0 is the legacy default stream)."""
        self._check(lib().swdg_gpu_set_stream(self._h, C.c_void_p(stream_handle or None)))

    def synchronize(self):
        self._check(lib().swdg_gpu_synchronize(self._h))

    def last_eps(self) -> np.ndarray:
        e = np.zeros(self.mesh.n_elem)
        self._check(lib().swdg_gpu_last_eps(self._h, _ptr(e)))
        return e

    def last_limited_count(self) -> int:
        return int(self._info.n_limited)

    def last_max_eps(self) -> float:
        return float(self._info.max_eps)

    def last_min_stage_h(self) -> float:
        return float(self._info.min_stage_h)

    def launch_count(self) -> int:
        return int(lib().swdg_gpu_launch_count(self._h))

    def device_state(self):
        hp, hup, hvp = _dp(), _dp(), _dp()
        self._check(lib().swdg_gpu_device_state(self._h, C.byref(hp), C.byref(hup),
                                                C.byref(hvp)))
        return [C.cast(p, C.c_void_p).value for p in (hp, hup, hvp)]


def set_grid_cap(max_ctas: int):
    """Test hook: cap the persistent stage kernels' grid (0 = resident slots)."""
    if lib().swdg_gpu_set_grid_cap(int(max_ctas)) != SWDG_OK:
        raise SwdgError("grid cap must be >= 0")


# ---------------------------------------------------------------- free functions
def assemble_rhs(state: State, mesh, phys: PhysicsParams, mode: int = MODE_EXACT) -> State:
    """dg_rhs.hpp:267 (entropy-stable, inviscid, no forcing)."""
    integ = TimeIntegrator(mesh, RunConfig(phys=phys, mode=mode))
    try:
        return integ.assemble_rhs(state)
    finally:
        integ.close()


def compute_dt(state: State, mesh, phys: PhysicsParams, cfl: float,
               mode: int = MODE_EXACT) -> float:
    """timeloop.hpp:53"""
    integ = TimeIntegrator(mesh, RunConfig(phys=phys, mode=mode))
    try:
        return integ.compute_dt(state, cfl)
    finally:
        integ.close()
