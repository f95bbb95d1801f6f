"""P0 / P1 boundary element spaces (host).  API subset of h2bem.spaces
(spaces.py:1-186) that the hot path needs: support boxes (cluster-tree input,
spaces.py:29-41), the mixed mass matrix and the Galerkin load vector of the
config-3 right-hand side.  Post-processing (L2 projection, error norms) is out
of scope."""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import quadrature as quad

P0 = "P0_triangles"
P1 = "P1_vertices"
ERROR_QUAD_ORDER = 4


@dataclass
class DofSpace:
    kind: str
    mesh: object

    @property
    def n_dofs(self):
        return self.mesh.n_triangles if self.kind == P0 else self.mesh.n_vertices

    def support_boxes(self):
        """(n_dofs, 2, 3) [min; max] of each dof support (spaces.py:29-41)."""
        mesh = self.mesh
        c = mesh.corners()
        lo_t, hi_t = c.min(axis=1), c.max(axis=1)
        if self.kind == P0:
            return np.stack([lo_t, hi_t], axis=1)
        if self.kind != P1:
            raise ValueError(f"unknown space kind {self.kind!r}")
        ptr, idx = mesh.vertex_triangle_csr()
        lo = np.minimum.reduceat(lo_t[idx], ptr[:-1], axis=0)
        hi = np.maximum.reduceat(hi_t[idx], ptr[:-1], axis=0)
        return np.stack([lo, hi], axis=1)


def assemble_mass(mesh):
    """Mixed P0 x P1 mass matrix, area/3 per (triangle, corner)."""
    F = mesh.n_triangles
    return sp.csr_matrix(
        (np.repeat(mesh.areas / 3.0, 3), (np.repeat(np.arange(F), 3), mesh.triangles.ravel())),
        shape=(F, mesh.n_vertices),
    )


def load_vector(space, fn):
    """Galerkin load b_i = int phi_i f (P0: per-triangle integral)."""
    mesh = space.mesh
    tris = np.arange(mesh.n_triangles)
    X, W, lam = quad.triangle_points(mesh, tris, ERROR_QUAD_ORDER)
    f = fn(X, tris)
    if space.kind == P0:
        return np.einsum("pq,pq->p", W, f)
    load = np.zeros(mesh.n_vertices)
    for l in range(3):
        np.add.at(load, mesh.triangles[:, l], np.einsum("pq,pq,q->p", W, f, lam[:, l]))
    return load
