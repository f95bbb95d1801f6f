"""Device CG (libh2b fused vector passes) vs the oracle's host CG
(oracle/cg.py, restating src/solver.py:22-59) on the config-0 single-layer
operator with the Jacobi preconditioner."""

import numpy as np
import pytest

from .helpers import sphere, trees

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def op0():
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import gca, spaces
    from paper_2001_05523_b200.containers import AssemblyContext

    m = sphere(4)
    t0, _ = trees(m, 32)
    ctx = AssemblyContext(m)
    bt = C.BlockTree(t0, t0, 2.0)
    basis = gca.build_basis(ctx, t0, gca.P0_SLP, 3, 1e-4, threads=4)
    H = gca.assemble_h2(ctx, "slp", bt, basis, basis, 3, q_singular=4)
    b = spaces.load_vector(spaces.DofSpace(spaces.P0, m), lambda X, t: X[..., 0] ** 2 - X[..., 1] ** 2)
    return H, b


def test_device_cg_matches_host_cg(op0):
    import torch

    from paper_2001_05523_b200 import solver

    from oracle import cg as OC

    H, b = op0
    diag = H.diagonal()
    hx, hit, hconv, _ = OC.cg(H.matvec, b, 1e-10, 500, precond_diag=diag)
    dev = solver.cg(H.matvec, torch.from_numpy(b).cuda(), 1e-10, 500, precond_diag=diag)
    assert hconv and dev.converged
    # the reductions round differently on host and device: near 1e-10 the
    # stopping test may trip a couple of iterations apart
    assert abs(hit - dev.iterations) <= 3
    xd = dev.x.cpu().numpy()
    assert np.linalg.norm(xd - hx) <= 1e-8 * np.linalg.norm(hx)
    # the reference call shape (numpy in, numpy out) runs the same device loop
    hn = solver.cg(H.matvec, b, 1e-10, 500, precond_diag=diag)
    assert isinstance(hn.x, np.ndarray) and hn.iterations == dev.iterations
    assert np.linalg.norm(hn.x - xd) <= 1e-12 * np.linalg.norm(xd)
    # the solution solves the system
    assert np.linalg.norm(H.matvec(xd) - b) <= 1.1e-10 * np.linalg.norm(b)


def test_device_cg_deterministic_and_unpreconditioned(op0):
    import torch

    from paper_2001_05523_b200 import solver

    H, b = op0
    bt = torch.from_numpy(b).cuda()
    a = solver.cg(H.matvec, bt, 1e-8, 500)
    c = solver.cg(H.matvec, bt, 1e-8, 500)
    assert a.converged and a.iterations == c.iterations and torch.equal(a.x, c.x)
    from oracle import cg as OC

    _, hit, _, _ = OC.cg(H.matvec, b, 1e-8, 500)
    assert abs(hit - a.iterations) <= 1


def test_device_cg_breakdown_raises(op0):
    import torch

    from paper_2001_05523_b200 import solver

    H, b = op0
    with pytest.raises(solver.SolverBreakdown):
        solver.cg(lambda p: -H.matvec(p), torch.from_numpy(b).cuda(), 1e-8, 50)
