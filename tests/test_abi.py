"""The drop-in boundary: the C-ABI library loads and exports every declared entry
point (CPU only, no compute calls), and the host mirror reports errors like the
reference without a device."""
import ctypes as C

import numpy as np
import pytest

from paper_1804_02221_b200 import swdg


def test_library_exports_every_declared_symbol():
    L = swdg.lib()
    declared = swdg.exported_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(L, name), f"{name} declared in include/swdg_gpu.h but not exported"


def test_struct_layouts_match_header():
    # swdg_params: 7 doubles + 4 int32; swdg_mesh_view: 4 int32 + 18 pointers
    assert C.sizeof(swdg.ParamsC) == 7 * 8 + 4 * 4
    assert C.sizeof(swdg.MeshViewC) == 4 * 4 + 18 * 8
    assert C.sizeof(swdg.StepInfoC) == 24
    assert C.sizeof(swdg.FaceC) == 24


def test_create_without_device_fails_loudly():
    """No CPU fallback: without a CUDA device, create reports an error."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a device is present")
    except Exception:
        pass
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    m = ref.build_mesh("cartesian", 2, 2, 2)
    with pytest.raises(swdg.CudaError):
        swdg.TimeIntegrator(m, swdg.RunConfig())


def test_input_errors_match_reference():
    """Input validation happens before any device call (timeloop.hpp:149-150)."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    m = ref.build_mesh("cartesian", 1, 2, 2)
    cfg = swdg.RunConfig(visc=swdg.ViscosityConfig(True, 0.1, -6.0, -4.0))
    with pytest.raises(swdg.SwdgError, match="degree >= 2"):
        swdg.TimeIntegrator(m, cfg)
    bad = ref.build_mesh("cartesian", 2, 2, 2)
    bad.arrays["face_nx"] = bad.arrays["face_nx"] * 0.9
    with pytest.raises(swdg.SwdgError, match="unit length"):
        swdg.TimeIntegrator(bad, swdg.RunConfig())
    faces = bad.faces.copy()
    faces[1] = faces[0]
    bad2 = ref.build_mesh("cartesian", 2, 2, 2)
    bad2.faces = faces
    with pytest.raises(swdg.SwdgError, match="listed twice"):
        swdg.TimeIntegrator(bad2, swdg.RunConfig())
