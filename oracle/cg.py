"""Jacobi-preconditioned CG on numpy vectors (oracle; test infrastructure only).

Restates the iteration of /root/reference/pkg/src/h2bem/solver.py:22-59 (cg):
relative residual ||r|| / ||b|| as the stopping test, a breakdown error when
the Jacobi diagonal is not positive or p^T A p <= 0, and after max_it steps
the true residual ||b - A x|| / ||b|| of the returned iterate.  Used only by
tests/ to check the device CG of paper_2001_05523_b200.solver.
"""

import numpy as np


class Breakdown(Exception):
    pass


def cg(apply_a, b, eps, max_it, precond_diag=None):
    """Returns (x, iterations, converged, residual)."""
    b = np.asarray(b, dtype=float)
    nb = float(np.linalg.norm(b))
    if nb == 0.0:
        return np.zeros_like(b), 0, True, 0.0
    scale = None
    if precond_diag is not None:
        d = np.asarray(precond_diag, dtype=float)
        if np.any(d <= 0.0):
            raise Breakdown("non-positive Jacobi diagonal")
        scale = 1.0 / d
    x = np.zeros_like(b)
    r = b.copy()
    z = r if scale is None else r * scale
    p = z.copy()
    rho = float(r @ z)
    for k in range(max_it):
        q = apply_a(p)
        curv = float(p @ q)
        if curv <= 0.0:
            raise Breakdown("non-positive curvature")
        step = rho / curv
        x += step * p
        r -= step * q
        res = float(np.linalg.norm(r)) / nb
        if res <= eps:
            return x, k + 1, True, res
        z = r if scale is None else r * scale
        rho_next = float(r @ z)
        p = z + (rho_next / rho) * p
        rho = rho_next
    return x, max_it, False, float(np.linalg.norm(b - apply_a(x))) / nb
