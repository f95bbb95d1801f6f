"""Block product H2Matrix.matmat (libh2b h2b_matmat, FP64 tensor cores) vs the
single-vector matvec, column by column (the reference has no block product;
its matvec is pinned by the other parity tests)."""

import numpy as np
import pytest

from .helpers import sphere, trees

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import gca
    from paper_2001_05523_b200.containers import AssemblyContext

    m = sphere(4)
    t0, t1 = trees(m, 32)
    ctx = AssemblyContext(m)
    b0 = gca.build_basis(ctx, t0, gca.P0_SLP, 3, 1e-4, threads=4)
    b1 = gca.build_basis(ctx, t1, gca.P1_DLP, 3, 1e-4, threads=4)
    slp = gca.assemble_h2(ctx, "slp", C.BlockTree(t0, t0, 2.0), b0, b0, 3, q_singular=4)
    dlp = gca.assemble_h2(ctx, "dlp", C.BlockTree(t0, t1, 2.0), b0, b1, 3, q_singular=5)
    return slp, dlp


@pytest.mark.parametrize("nrhs", [1, 3, 8, 11, 16, 21])
@pytest.mark.parametrize("kind", ["slp", "dlp"])
def test_matmat_columns_equal_matvec(ops, kind, nrhs):
    H = ops[0] if kind == "slp" else ops[1]
    X = np.random.default_rng(nrhs).uniform(-1, 1, (H.shape[1], nrhs))
    Y = H.matmat(X)
    assert Y.shape == (H.shape[0], nrhs)
    for j in range(nrhs):
        y = H.matvec(X[:, j])
        assert np.abs(Y[:, j] - y).max() <= 1e-13 * np.abs(y).max(), j


def test_matmat_device_deterministic(ops):
    import torch

    H = ops[0]
    X = torch.from_numpy(np.random.default_rng(7).standard_normal((H.shape[1], 16))).cuda()
    a, b = H.matmat(X), H.matmat(X)
    assert a.is_cuda and torch.equal(a, b)
