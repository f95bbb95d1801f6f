"""P0 / P1 boundary element spaces (host).  API subset of h2bem.spaces
(spaces.py:1-186): support boxes (cluster-tree input), mixed mass matrix,
L2 projection/load vectors and the energy error used by the drivers."""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

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


def l2_project(space, fn):
    """Coefficients of the L2 projection of fn(X, tris) onto the space."""
    mesh = space.mesh
    tris = np.arange(mesh.n_triangles)
    X, W, lam = quad.triangle_points(mesh, tris, ERROR_QUAD_ORDER)
    f = fn(X, tris)
    if space.kind == P0:
        return np.einsum("pq,pq->p", W, f) / mesh.areas
    load = np.zeros(mesh.n_vertices)
    for l in range(3):
        np.add.at(load, mesh.triangles[:, l], np.einsum("pq,pq,q->p", W, f, lam[:, l]))
    ptl = np.einsum("pq,qa,qb->pab", W, lam, lam)
    rows = np.repeat(mesh.triangles, 3, axis=1).ravel()
    cols = np.tile(mesh.triangles, (1, 3)).ravel()
    gram = sp.csr_matrix((ptl.ravel(), (rows, cols)), shape=(mesh.n_vertices,) * 2)
    return spla.spsolve(gram.tocsc(), load)


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


def energy_error(apply_g, d):
    """sqrt(d^T G d) through the (compressed) single-layer action."""
    d = np.asarray(d, dtype=float)
    if not d.any():
        return 0.0
    val = float(d @ apply_g(d))
    if val < -1e-12 * float(d @ d):
        raise ArithmeticError(f"energy product is negative ({val:.3e}): operator lost definiteness")
    return float(np.sqrt(max(val, 0.0)))
