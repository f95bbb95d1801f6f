"""Error paths of the device path, mapped onto the reference's exceptions
(containers.py:79-98 raises FloatingPointError on a non-finite nearfield
entry; dense_block raises ValueError on unknown kinds / touching pairs)."""

import numpy as np
import pytest

from .helpers import sphere

pytestmark = pytest.mark.gpu


def test_non_finite_entry_raises_floating_point_error():
    """Two panels with distinct vertex ids but the same geometry: their
    regular-rule points coincide, 1/r is infinite."""
    from paper_2001_05523_b200.containers import AssemblyContext, dense_block
    from paper_2001_05523_b200.mesh import SurfaceMesh

    m = sphere(1)
    V = np.vstack([m.vertices, m.vertices])
    T = np.vstack([m.triangles, m.triangles + m.n_vertices])
    ctx = AssemblyContext(SurfaceMesh(V, T))
    with pytest.raises(FloatingPointError):
        dense_block(ctx, "slp", [0], [m.n_triangles], 3)


def test_bad_vector_shapes_raise(cfg_small):
    H = cfg_small
    with pytest.raises(ValueError):
        H.matvec(np.zeros(H.shape[1] + 1))
    with pytest.raises(ValueError):
        H.matmat(np.zeros((H.shape[1] + 1, 2)))


@pytest.fixture(scope="module")
def cfg_small():
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import gca, spaces
    from paper_2001_05523_b200.containers import AssemblyContext

    m = sphere(3)
    ctx = AssemblyContext(m)
    t = C.build_cluster_tree(spaces.DofSpace(spaces.P0, m).support_boxes(), 16)
    b = gca.build_basis(ctx, t, gca.P0_SLP, 3, 1e-4, threads=2)
    return gca.assemble_h2(ctx, "slp", C.BlockTree(t, t, 2.0), b, b, 3, q_singular=4)
