"""Parity at configuration-2 size (sphere level 8: 524 288 panels, 262 146
vertices), where the reference's full nearfield takes hours: a seeded sample
of single- and double-layer near blocks (regular order 3, Sauter-Schwab
order 5) and of touching-pair integrals, produced by the reference itself
(tests/golden/make_golden.py gen_sample_l8), against the device assembly."""

import numpy as np
import pytest

from .conftest import golden
from .helpers import rel, sphere, trees

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def world8():
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200.containers import AssemblyContext

    m = sphere(8)
    t0, t1 = trees(m, 64)
    return m, AssemblyContext(m), C.BlockTree(t0, t0, 2.0), C.BlockTree(t0, t1, 2.0)


def _blocks(out, lay, sel):
    """Sampled blocks of a packed device nearfield, row-major, concatenated."""
    import torch

    idx = []
    for i in sel:
        off, ld = int(lay.blk_off[i]), int(lay.blk_ld[i])
        r, c = int(lay.blk_rows[i]), int(lay.blk_cols[i])
        idx.append((off + np.arange(r)[:, None] * ld + np.arange(c)[None, :]).ravel())
    return out[torch.from_numpy(np.concatenate(idx)).cuda()].cpu().numpy()


@pytest.mark.parametrize("kind", ["slp", "dlp"])
def test_level8_near_blocks_vs_reference(world8, kind):
    from paper_2001_05523_b200.containers import assemble_nearfield_device, near_layout

    g = golden("sample_l8.npz")
    m, ctx, bs, bd = world8
    bt = bs if kind == "slp" else bd
    out = assemble_nearfield_device(ctx, kind, bt, 3, 5)
    got = _blocks(out, near_layout(bt), g[f"{kind}_sel"])
    ref = g[f"{kind}_vals"]
    assert got.shape == ref.shape
    assert rel(got, ref) < 1e-10
    if kind == "slp":  # all single-layer entries are positive: entrywise
        assert np.abs(got - ref).max() / np.abs(ref).min() < 1e-10


@pytest.mark.parametrize("kind", ["slp", "dlp"])
def test_level8_touching_pairs_vs_reference(world8, kind):
    g = golden("sample_l8.npz")
    m, ctx, _, _ = world8
    got = ctx.singular_table(kind, 5).lookup(g["pa"], g["pb"])
    assert rel(got, g[f"{kind}_pairs"]) < 1e-10


def test_level8_operator_properties(world8):
    """Size-independent checks of the level-8 single-layer H^2 operator
    (device GCA basis, device assembly): symmetry x.Ay = y.Ax of the
    symmetric Galerkin matrix, linearity, bitwise repeatability, the block
    product against the matvec, and the symmetric-nearfield plan against the
    one-sided one."""
    import torch

    from paper_2001_05523_b200 import gca

    m, ctx, bs, _ = world8
    t0 = bs.row_tree
    b = gca.build_basis(ctx, t0, gca.P0_SLP, 4, 1e-4, device=True)
    H = gca.assemble_h2(ctx, "slp", bs, b, b, 3, q_singular=5)
    n = H.shape[0]
    gen = torch.Generator(device="cuda").manual_seed(8)
    X = torch.randn((n, 3), dtype=torch.float64, device="cuda", generator=gen)
    x, z = X[:, 0].contiguous(), X[:, 1].contiguous()
    ax, az = H.matvec(x), H.matvec(z)
    assert abs(float(z @ ax - x @ az)) <= 1e-12 * abs(float(z @ ax)) + 1e-12 * float(ax.norm() * z.norm())
    lin = H.matvec(0.7 * x - 1.3 * z) - (0.7 * ax - 1.3 * az)
    assert float(lin.norm()) <= 1e-13 * float(ax.norm())
    assert torch.equal(H.matvec(x), ax)
    Y = H.matmat(X)
    for j in range(3):
        yj = H.matvec(X[:, j].contiguous())
        assert float((Y[:, j] - yj).abs().max()) <= 1e-13 * float(yj.abs().max())
    # the symmetric nearfield (streamed once per block pair) against the
    # one-sided plan at full size
    import os

    from paper_2001_05523_b200.containers import MatvecPlan

    assert H.plan().info()["near_symmetric"]
    os.environ["H2B_NEAR_SYM"] = "0"
    try:
        one = MatvecPlan(H.block_tree, H.row_basis, H.col_basis, H.S_dev, H.D_dev, H.far_layout, H.near_layout)
    finally:
        del os.environ["H2B_NEAR_SYM"]
    assert float((one.apply(x) - ax).norm()) <= 1e-14 * float(ax.norm())
