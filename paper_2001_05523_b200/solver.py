"""Jacobi-preconditioned conjugate gradients (h2bem.solver.cg, solver.py:22-59).

Same iteration, stopping rule and breakdown checks as the reference; the
operator application is whatever `apply_a` is -- for an H2Matrix the device
matvec.  Vectors may be numpy arrays (host loop, reference semantics) or CUDA
tensors (device-resident loop: no host round trip per iteration except the
scalar residual test)."""

from dataclasses import dataclass

import numpy as np


class SolverBreakdown(Exception):
    """CG met a non-positive curvature direction (operator not SPD)."""


@dataclass
class CGResult:
    x: object
    iterations: int
    converged: bool
    residual: float


def cg(apply_a, b, eps, max_it, precond_diag=None):
    try:
        import torch
        is_t = isinstance(b, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_t = False
    if is_t:
        return _cg_torch(apply_a, b, eps, max_it, precond_diag)
    b = np.asarray(b, dtype=float)
    norm_b = float(np.linalg.norm(b))
    if norm_b == 0.0:
        return CGResult(np.zeros_like(b), 0, True, 0.0)
    inv_d = None
    if precond_diag is not None:
        precond_diag = np.asarray(precond_diag, dtype=float)
        if (precond_diag <= 0.0).any():
            raise SolverBreakdown("Jacobi preconditioner requires a positive diagonal")
        inv_d = 1.0 / precond_diag
    x = np.zeros_like(b)
    r = b.copy()
    z = r * inv_d if inv_d is not None else r
    p = z.copy()
    rz = float(r @ z)
    for it in range(1, max_it + 1):
        Ap = apply_a(p)
        pAp = float(p @ Ap)
        if pAp <= 0.0:
            raise SolverBreakdown(f"non-positive curvature p^T A p = {pAp:.3e} at iteration {it}")
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        res = float(np.linalg.norm(r)) / norm_b
        if res <= eps:
            return CGResult(x, it, True, res)
        z = r * inv_d if inv_d is not None else r
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return CGResult(x, max_it, False, float(np.linalg.norm(b - apply_a(x))) / norm_b)


def _cg_torch(apply_a, b, eps, max_it, precond_diag):
    import torch

    norm_b = float(torch.linalg.vector_norm(b))
    if norm_b == 0.0:
        return CGResult(torch.zeros_like(b), 0, True, 0.0)
    inv_d = None
    if precond_diag is not None:
        d = torch.as_tensor(precond_diag, dtype=b.dtype, device=b.device)
        if bool((d <= 0.0).any()):
            raise SolverBreakdown("Jacobi preconditioner requires a positive diagonal")
        inv_d = 1.0 / d
    x = torch.zeros_like(b)
    r = b.clone()
    z = r * inv_d if inv_d is not None else r
    p = z.clone()
    rz = torch.dot(r, z)
    for it in range(1, max_it + 1):
        Ap = apply_a(p)
        pAp = torch.dot(p, Ap)
        if float(pAp) <= 0.0:
            raise SolverBreakdown(f"non-positive curvature p^T A p = {float(pAp):.3e} at iteration {it}")
        alpha = rz / pAp
        x.add_(alpha * p)
        r.sub_(alpha * Ap)
        res = float(torch.linalg.vector_norm(r)) / norm_b
        if res <= eps:
            return CGResult(x, it, True, res)
        z = r * inv_d if inv_d is not None else r
        rz_new = torch.dot(r, z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return CGResult(x, max_it, False, float(torch.linalg.vector_norm(b - apply_a(x))) / norm_b)
