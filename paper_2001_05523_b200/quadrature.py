"""Quadrature rules (host tables, uploaded once per order).  API of
h2bem.quadrature (quadrature.py:1-211).

* Gauss-Legendre on [0, 1] from numpy's leggauss (same nodes/weights bits as
  the reference, quadrature.py:49-55).
* Duffy tensor rule on the reference triangle, s-major point order
  (quadrature.py:58-68).
* Sauter-Schwab relative-coordinate rules for identical / shared-edge /
  shared-vertex panel pairs (quadrature.py:121-190).  The 4-D point set
  (u1, v1, u2, v2) lives in the chart simplex {0 <= v <= u <= 1} of each panel,
  chart(u, v) = P1 + u (P2 - P1) + v (P3 - P2); weights include the Jacobians
  but not the areas (sum = 1/4).  Subdomain blocks are concatenated in the
  order of the classical transform so rule arrays match the reference.
"""

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

IDENTICAL = "identical"
SHARED_EDGE = "shared_edge"
SHARED_VERTEX = "shared_vertex"
DISJOINT = "disjoint"

SUBDOMAINS = {IDENTICAL: 6, SHARED_EDGE: 5, SHARED_VERTEX: 2, DISJOINT: 1}
#: case code = number of shared vertices (what the device classifier emits)
CODE_OF_CASE = {DISJOINT: 0, SHARED_VERTEX: 1, SHARED_EDGE: 2, IDENTICAL: 3}


@dataclass(frozen=True)
class QuadRule1D:
    points: np.ndarray
    weights: np.ndarray


@dataclass(frozen=True)
class PanelPairRule:
    case: str
    points: np.ndarray   # (N, 4): u1, v1, u2, v2
    weights: np.ndarray  # (N,)


def _ro(a):
    a = np.ascontiguousarray(a)
    a.setflags(write=False)
    return a


@lru_cache(maxsize=None)
def gauss_legendre(q):
    """q-point Gauss-Legendre rule on [0, 1] (exact to degree 2q-1)."""
    if q < 1:
        raise ValueError("quadrature order must be >= 1")
    x, w = np.polynomial.legendre.leggauss(q)
    return QuadRule1D(_ro(0.5 * (x + 1.0)), _ro(0.5 * w))


@lru_cache(maxsize=None)
def triangle_rule(q):
    """Duffy rule (x, y) = (s (1 - t), s t), weight w_s w_t s; q^2 points, sum 1/2."""
    g = gauss_legendre(q)
    s = np.repeat(g.points, q)
    t = np.tile(g.points, q)
    ws = np.repeat(g.weights, q)
    wt = np.tile(g.weights, q)
    pts = np.column_stack([s * (1.0 - t), s * t])
    return _ro(pts), _ro(ws * wt * s)


def triangle_points(mesh, tris, q):
    """Physical points X (P, q^2, 3), weights incl. 2*area (P, q^2), barycentrics (q^2, 3).
    Host reference form of the device kernel h2b_panel_points."""
    pts, w = triangle_rule(q)
    c = mesh.vertices[mesh.triangles[tris]]
    x = pts[:, 0][None, :, None]
    y = pts[:, 1][None, :, None]
    X = c[:, None, 0, :] + x * (c[:, 1, :] - c[:, 0, :])[:, None, :] + y * (c[:, 2, :] - c[:, 0, :])[:, None, :]
    W = w[None, :] * (2.0 * mesh.areas[tris])[:, None]
    lam = np.column_stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]])
    return X, W, lam


def classify_panel_pair(tri_a, tri_b):
    """(case, perm_a, perm_b): shared vertices first (ascending global id), then
    the remaining local vertices in their original order."""
    a = [int(v) for v in tri_a]
    b = [int(v) for v in tri_b]
    ident = (0, 1, 2)
    if a == b:
        return IDENTICAL, ident, ident
    shared = sorted(set(a).intersection(b))

    def perm(tri):
        head = tuple(tri.index(s) for s in shared)
        return head + tuple(i for i in range(3) if i not in head)

    if len(shared) == 2:
        return SHARED_EDGE, perm(a), perm(b)
    if len(shared) == 1:
        return SHARED_VERTEX, perm(a), perm(b)
    return DISJOINT, ident, ident


def _grid4(q):
    g = gauss_legendre(q)
    idx = np.indices((q, q, q, q)).reshape(4, -1)
    P = g.points[idx].T
    W = g.weights[idx].T.prod(axis=1)
    return P, W


def _identical_subdomains(e1, e2, e3, xi):
    j = xi**3 * e1**2 * e2
    a = xi * (1 - e1 + e1 * e2)
    b = xi * (1 - e1 * e2 * e3)
    c = xi * (1 - e1)
    d = xi * e1 * (1 - e2 + e2 * e3)
    e = xi * (1 - e1 * e2)
    f = xi * e1 * (1 - e2)
    g = xi * e1 * (1 - e2 * e3)
    return [
        (xi, a, b, c, j),
        (b, c, xi, a, j),
        (xi, d, e, f, j),
        (e, f, xi, d, j),
        (b, g, xi, f, j),
        (xi, f, b, g, j),
    ]


def _edge_subdomains(e1, e2, e3, xi):
    ja = xi**3 * e1**2
    jb = xi**3 * e1**2 * e2
    return [
        (xi, xi * e1 * e3, xi * (1 - e1 * e2), xi * e1 * (1 - e2), ja),
        (xi, xi * e1, xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), jb),
        (xi * (1 - e1 * e2), xi * e1 * (1 - e2), xi, xi * e1 * e2 * e3, jb),
        (xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), xi, xi * e1, jb),
        (xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), xi, xi * e1 * e2, jb),
    ]


def _vertex_subdomains(e1, e2, e3, xi):
    j = xi**3 * e2
    return [
        (xi, xi * e1, xi * e2, xi * e2 * e3, j),
        (xi * e2, xi * e2 * e3, xi, xi * e1, j),
    ]


@lru_cache(maxsize=None)
def sauter_schwab_rule(case, q):
    """4-D panel-pair rule for an adjacency case; SUBDOMAINS[case] * q^4 points."""
    if q < 1:
        raise ValueError("quadrature order must be >= 1")
    if case == DISJOINT:
        P, W = _grid4(q)
        s1, t1, s2, t2 = P.T
        pts = np.column_stack([s1, s1 * t1, s2, s2 * t2])
        return PanelPairRule(case, _ro(pts), _ro(W * s1 * s2))
    maps = {IDENTICAL: _identical_subdomains, SHARED_EDGE: _edge_subdomains, SHARED_VERTEX: _vertex_subdomains}
    if case not in maps:
        raise ValueError(f"unknown panel-pair case {case!r}")
    P, W = _grid4(q)
    parts = maps[case](P[:, 0], P[:, 1], P[:, 2], P[:, 3])
    pts = np.vstack([np.column_stack(p[:4]) for p in parts])
    wts = np.concatenate([W * p[4] for p in parts])
    return PanelPairRule(case, _ro(pts), _ro(wts))


def chart_points(corners, uv):
    u = uv[:, 0][:, None]
    v = uv[:, 1][:, None]
    p1 = corners[..., 0, :][..., None, :]
    p2 = corners[..., 1, :][..., None, :]
    p3 = corners[..., 2, :][..., None, :]
    return p1 + u * (p2 - p1) + v * (p3 - p2)


def chart_bary(uv):
    u, v = uv[:, 0], uv[:, 1]
    return np.column_stack([1.0 - u, u - v, v])
