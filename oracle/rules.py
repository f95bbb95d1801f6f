"""Quadrature rules, restated (oracle; test infrastructure only).

Reference: /root/reference/pkg/src/h2bem/quadrature.py
  gauss_legendre        :49-55   Gauss-Legendre on [0,1]
  triangle_rule         :58-68   Duffy tensor rule, s-major
  _identical/_edge/_vertex_maps  :130-160  Sauter-Schwab subdomain maps
  sauter_schwab_rule    :163-190 concatenated subdomain blocks, weights w/o areas
"""

import numpy as np


def gauss01(q):
    """(x, w) on [0, 1] -- quadrature.py:49-55."""
    x, w = np.polynomial.legendre.leggauss(q)
    return 0.5 * (x + 1.0), 0.5 * w


def duffy(q):
    """(points (q^2, 2), weights) -- quadrature.py:58-68."""
    x, w = gauss01(q)
    s = np.repeat(x, q)
    t = np.tile(x, q)
    return np.column_stack([s * (1.0 - t), s * t]), np.repeat(w, q) * np.tile(w, q) * s


def _tensor4(q):
    x, w = gauss01(q)
    g = np.array(np.meshgrid(x, x, x, x, indexing="ij")).reshape(4, -1)
    wg = np.array(np.meshgrid(w, w, w, w, indexing="ij")).reshape(4, -1)
    return g, wg[0] * wg[1] * wg[2] * wg[3]


def ss_rule(case, q):
    """Sauter-Schwab rule for case in {'identical', 'edge', 'vertex', 'disjoint'}:
    (points (N, 4) = u1, v1, u2, v2, weights) -- quadrature.py:121-190."""
    (e1, e2, e3, xi), W = _tensor4(q)
    if case == "identical":
        # quadrature.py:130-141; Jacobian xi^3 e1^2 e2 on all six subdomains
        J = xi**3 * e1**2 * e2
        A = (xi, xi * (1 - e1 + e1 * e2))
        B = (xi * (1 - e1 * e2 * e3), xi * (1 - e1))
        Cc = (xi, xi * e1 * (1 - e2 + e2 * e3))
        Dd = (xi * (1 - e1 * e2), xi * e1 * (1 - e2))
        Ee = (xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3))
        Ff = (xi, xi * e1 * (1 - e2))
        pairs = [(A, B), (B, A), (Cc, Dd), (Dd, Cc), (Ee, Ff), (Ff, Ee)]
        jac = [J] * 6
    elif case == "edge":
        # quadrature.py:144-153
        ja = xi**3 * e1**2
        jb = xi**3 * e1**2 * e2
        pairs = [
            ((xi, xi * e1 * e3), (xi * (1 - e1 * e2), xi * e1 * (1 - e2))),
            ((xi, xi * e1), (xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3))),
            ((xi * (1 - e1 * e2), xi * e1 * (1 - e2)), (xi, xi * e1 * e2 * e3)),
            ((xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3)), (xi, xi * e1)),
            ((xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3)), (xi, xi * e1 * e2)),
        ]
        jac = [ja, jb, jb, jb, jb]
    elif case == "disjoint":
        # quadrature.py:171-180: the tensor product of two Duffy rules in chart
        # coordinates (u, v) = (s, s t), weight w_s w_t w_s' w_t' s s'
        x, w = gauss01(q)
        G = np.array(np.meshgrid(x, x, x, x, indexing="ij")).reshape(4, -1)
        Wg = np.array(np.meshgrid(w, w, w, w, indexing="ij")).reshape(4, -1)
        P = np.column_stack([G[0], G[0] * G[1], G[2], G[2] * G[3]])
        return P, Wg[0] * Wg[1] * Wg[2] * Wg[3] * G[0] * G[2]
    elif case == "vertex":
        # quadrature.py:156-160
        j = xi**3 * e2
        pairs = [((xi, xi * e1), (xi * e2, xi * e2 * e3)), ((xi * e2, xi * e2 * e3), (xi, xi * e1))]
        jac = [j, j]
    else:
        raise ValueError(case)
    P = np.vstack([np.column_stack([x[0], x[1], y[0], y[1]]) for x, y in pairs])
    w = np.concatenate([W * j for j in jac])
    return P, w
