"""Host-built inputs of the product library (no device needed): the LGL operators and
the structured face lists are bitwise the reference's (operators.hpp:148-188,
mesh.hpp:237-290)."""
import numpy as np
import pytest

from oracle import ref
from paper_1804_02221_b200 import swdg

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("degree", list(range(1, 16)))
def test_operators_bitwise(degree):
    a, b = swdg.operators(degree), ref.operators(degree)
    for k in a:
        assert np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64)), k


@pytest.mark.parametrize("kx,ky,px,py", [(3, 4, 0, 0), (5, 2, 1, 0), (1, 1, 1, 1), (4, 4, 1, 1),
                                         (2, 3, 0, 1), (1, 6, 0, 0)])
def test_structured_faces_match(kx, ky, px, py):
    m = ref.build_mesh("cartesian", 2, kx, ky, periodic_x=bool(px), periodic_y=bool(py))
    assert np.array_equal(swdg.structured_faces(kx, ky, px, py), m.faces)


def test_degree_out_of_range():
    with pytest.raises(swdg.SwdgError):
        swdg.operators(16)
