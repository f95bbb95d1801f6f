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


def _cg_torch(apply_a, b, eps, max_it, precond_diag, allreduce=None):
    """Device-resident CG on CUDA float64 tensors: fused libh2b vector passes
    (h2b_cg_dot / h2b_cg_step / h2b_cg_direction), scalars kept on the device
    and one 4-double read-back per iteration for the breakdown and stopping
    tests.  `allreduce(t)` (row-sharded vectors) sums a small device tensor
    over the ranks in place."""
    import ctypes

    import torch

    from . import _lib

    L = _lib.lib()
    st = _lib.stream_ptr()
    n = b.numel()
    b = b.contiguous()
    ws = ctypes.c_int64()
    _lib.check(L.h2b_cg_workspace_size(ctypes.byref(ws)))
    work = torch.zeros(ws.value, dtype=torch.uint8, device=b.device)
    sc = torch.zeros(4, dtype=torch.float64, device=b.device)  # rz, pAp, rz_new, r.r
    host = torch.zeros(4, dtype=torch.float64).pin_memory()

    def dot(a, c, out):
        _lib.check(L.h2b_cg_dot(a.data_ptr(), c.data_ptr(), n, work.data_ptr(), out.data_ptr(), st))
        if allreduce is not None:
            allreduce(out)

    nb = torch.zeros(1, dtype=torch.float64, device=b.device)
    dot(b, b, nb)
    norm_b = float(nb.sqrt())
    if norm_b == 0.0:
        return CGResult(torch.zeros_like(b), 0, True, 0.0)
    inv_d = None
    if precond_diag is not None:
        d = torch.as_tensor(precond_diag, dtype=b.dtype, device=b.device)
        if bool((d <= 0.0).any()):
            raise SolverBreakdown("Jacobi preconditioner requires a positive diagonal")
        inv_d = (1.0 / d).contiguous()
    x = torch.zeros_like(b)
    r = b.clone()
    z = r * inv_d if inv_d is not None else r
    p = z.clone()
    dot(r, z, sc[0:1])
    z_ptr = z.data_ptr() if inv_d is not None else None
    for it in range(1, max_it + 1):
        Ap = apply_a(p)
        dot(p, Ap, sc[1:2])
        _lib.check(L.h2b_cg_step(n, sc.data_ptr(), x.data_ptr(), r.data_ptr(), p.data_ptr(), Ap.data_ptr(),
                                 inv_d.data_ptr() if inv_d is not None else None, z_ptr, work.data_ptr(),
                                 sc[2:4].data_ptr(), st))
        if allreduce is not None:
            allreduce(sc[2:4])
        host.copy_(sc)
        pAp, rr = float(host[1]), float(host[3])
        if pAp <= 0.0:
            raise SolverBreakdown(f"non-positive curvature p^T A p = {pAp:.3e} at iteration {it}")
        res = float(np.sqrt(rr)) / norm_b
        if res <= eps:
            return CGResult(x, it, True, res)
        _lib.check(L.h2b_cg_direction(n, sc.data_ptr(), (z if inv_d is not None else r).data_ptr(), p.data_ptr(),
                                      st))
        sc[0:1].copy_(sc[2:3])
    res_vec = b - apply_a(x)
    dot(res_vec, res_vec, nb)
    return CGResult(x, max_it, False, float(nb.sqrt()) / norm_b)
