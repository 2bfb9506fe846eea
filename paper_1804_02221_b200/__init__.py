"""B200-native (sm_100a, FP64) ES-DGSEM shallow-water stage path (arXiv 1804.02221).

Drop-in for the reference `swdg` TimeIntegrator/assemble_rhs/compute_dt seams via the
C ABI in include/swdg_gpu.h; see DESIGN.md.
"""
from .swdg import (MODE_EXACT, MODE_FAST, CudaError, Mesh, NumericalAbort,  # noqa: F401
                   PhysicsParams, RunConfig, State, SwdgError, TimeIntegrator,
                   ViscosityConfig, assemble_rhs, compute_dt, default_sigma_band)

__all__ = ["TimeIntegrator", "Mesh", "State", "RunConfig", "PhysicsParams", "ViscosityConfig",
           "SwdgError", "NumericalAbort", "CudaError", "assemble_rhs", "compute_dt",
           "default_sigma_band", "MODE_EXACT", "MODE_FAST"]
