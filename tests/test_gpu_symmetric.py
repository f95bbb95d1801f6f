"""Symmetric storage in the matvec: plans of a bitwise symmetric nearfield
(the single-layer Galerkin matrix on one tree) stream every block pair once
and deliver the transposed product as partial vectors; anything else streams
every block.  Both must give the same operator."""

import os

import numpy as np
import pytest

from .helpers import rel, sphere, trees

pytestmark = pytest.mark.gpu


def _plan(H, near_sym):
    """A plan with the symmetric nearfield allowed or not."""
    from paper_2001_05523_b200.containers import MatvecPlan

    env = {"H2B_NEAR_SYM": "1" if near_sym else "0"}
    os.environ.update(env)
    try:
        return MatvecPlan(H.block_tree, H.row_basis, H.col_basis, H.S_dev, H.D_dev, H.far_layout, H.near_layout)
    finally:
        for k in env:
            del os.environ[k]


def _slp(level, leaf, m=3):
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import gca
    from paper_2001_05523_b200.containers import AssemblyContext

    mesh = sphere(level)
    t0, _ = trees(mesh, leaf)
    ctx = AssemblyContext(mesh)
    b = gca.build_basis(ctx, t0, gca.P0_SLP, m, 1e-4, threads=8)
    return gca.assemble_h2(ctx, "slp", C.BlockTree(t0, t0, 2.0), b, b, 3, q_singular=4)


@pytest.mark.parametrize("level,leaf", [(4, 32), (5, 16), (5, 64)])
def test_symmetric_nearfield_matches_one_sided(level, leaf):
    import torch

    H = _slp(level, leaf)
    info = H.plan().info()
    assert info["near_symmetric"] and not info["coupling_symmetric"]
    ref = _plan(H, False)
    full = ref.info()
    # every block pair once: the upper blocks (diagonal blocks in full)
    assert full["near_bytes"] >= 8 * H.near_layout.entries  # (+ the rows' padding columns)
    assert info["near_bytes"] < 0.6 * full["near_bytes"]
    assert full["coupling_bytes"] >= 8 * H.far_layout.entries
    rng = np.random.default_rng(level * 100 + leaf)
    for _ in range(3):
        x = rng.standard_normal(H.shape[1])
        y = H.matvec(x)
        y1 = ref.apply(x)
        assert rel(y, y1) < 1e-14
        xd = torch.from_numpy(x).cuda()
        yd = H.matvec(xd)
        assert torch.equal(yd, H.matvec(xd))  # bitwise reproducible
        assert np.array_equal(yd.cpu().numpy(), y)  # host and device inputs agree bit for bit


def test_nonsymmetric_nearfield_streams_every_block():
    """One perturbed entry: the bitwise symmetry check fails at plan creation
    and the plan streams every block (and sees the perturbation)."""
    from paper_2001_05523_b200.containers import H2Matrix

    H = _slp(4, 32)
    Dn = H.D_dev.clone()
    nl = H.near_layout
    i = int(np.nonzero(nl.blk_cols > 1)[0][0])
    Dn[int(nl.blk_off[i]) + 1] += 1.0  # entry (0, 1) of a near block
    H2 = H2Matrix.from_device(H.block_tree, H.row_basis, H.col_basis, H.S_dev, Dn)
    info = _plan(H2, True).info()
    assert not info["near_symmetric"]
    x = np.random.default_rng(1).standard_normal(H.shape[1])
    d = H2.matvec(x) - H.matvec(x)
    r = H.row_tree.perm[H.row_tree.start[H.block_tree.near_uids[i, 0]]]
    assert abs(d[r] - x[H.col_tree.perm[H.col_tree.start[H.block_tree.near_uids[i, 1]] + 1]]) < 1e-12
    d[r] = 0.0
    assert np.abs(d).max() < 1e-12


def test_dlp_plan_is_one_sided():
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import gca
    from paper_2001_05523_b200.containers import AssemblyContext

    mesh = sphere(3)
    t0, t1 = trees(mesh, 32)
    ctx = AssemblyContext(mesh)
    rb = gca.build_basis(ctx, t0, gca.P0_SLP, 3, 1e-4, threads=4)
    cb = gca.build_basis(ctx, t1, gca.P1_DLP, 3, 1e-4, threads=4)
    H = gca.assemble_h2(ctx, "dlp", C.BlockTree(t0, t1, 2.0), rb, cb, 3, q_singular=4)
    info = _plan(H, True).info()
    assert not info["near_symmetric"] and not info["coupling_symmetric"]
