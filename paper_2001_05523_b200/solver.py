"""Jacobi-preconditioned conjugate gradients on the device.

Drop-in for h2bem.solver.cg (reference solver.py:22-59): same arguments
(apply_a, b, eps, max_it, precond_diag), same stopping rule (relative residual
||r|| / ||b|| <= eps), same breakdown conditions (SolverBreakdown for a
non-positive Jacobi diagonal or non-positive curvature) and the same result
fields.  The vectors always live in HBM and every vector pass is a fused
libh2b kernel (h2b_cg_dot / h2b_cg_step / h2b_cg_direction) with
deterministic reductions; the scalars stay on the device and one 32-byte
read-back per iteration feeds the host-side tests.

* b a CUDA float64 tensor: apply_a maps CUDA tensors to CUDA tensors (e.g.
  MatvecPlan.apply_device); x is returned as a tensor.
* b a numpy array (the reference call, e.g. cg(G.matvec, b, ...)): apply_a is
  called with numpy vectors, as in the reference; x is returned as numpy.
* Row-sharded vectors (one process per GPU): pass `allreduce(t)`, an in-place
  sum of a small device tensor over the ranks (distributed.allreduce_sum);
  each rank then holds its own rows of x, r, p and the Jacobi diagonal, and
  the iteration count is the single-GPU one.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import device as D


class SolverBreakdown(Exception):
    """CG met a non-positive curvature direction (operator not SPD)."""


@dataclass
class CGResult:
    x: object
    iterations: int
    converged: bool
    residual: float


def cg(apply_a, b, eps, max_it, precond_diag=None, allreduce=None):
    t = D.require_cuda()
    if isinstance(b, t.Tensor):
        return _cg_device(apply_a, b, eps, max_it, precond_diag, allreduce)
    bh = np.asarray(b, dtype=np.float64)

    def apply_dev(p):
        return D.dev(np.asarray(apply_a(D.host(p)), dtype=np.float64))

    res = _cg_device(apply_dev, D.dev(bh), eps, max_it, precond_diag, allreduce)
    return CGResult(D.host(res.x), res.iterations, res.converged, res.residual)


def _cg_device(apply_a, b, eps, max_it, precond_diag, allreduce=None):
    import torch

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
        bad = (d <= 0.0).any().to(torch.float64).reshape(1)
        if allreduce is not None:
            allreduce(bad)
        if bool(bad.item() > 0):
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
