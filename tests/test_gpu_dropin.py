"""The reference's kernel-level and basis entry points, called with the
reference's arguments, on the device: kernels.pair_integrals /
panel_pair_matrix / slp_block / dlp_block / SingularTable (kernels.py:260-468)
and ClusterBasis.forward / backward / expand (containers.py:201-235).  Values
are checked against the reference's own outputs (tests/golden/pairs.npz,
h2_cfg0.npz) and the CPU oracle."""

import numpy as np
import pytest

from oracle import h2 as OH
from oracle import quad as OQ

from .conftest import golden
from .helpers import basis_from_arrays, oracle_tree, rel, sphere, trees

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mesh3():
    return sphere(3)


@pytest.mark.parametrize("q", [2, 3, 4])
@pytest.mark.parametrize("kind", ["slp", "dlp"])
def test_pair_integrals_vs_reference(mesh3, kind, q):
    from paper_2001_05523_b200 import kernels

    g = golden("pairs.npz")
    v = kernels.pair_integrals(mesh3, g["pa"], g["pb"], kind, q)
    ref = g[f"{kind}_q{q}"]
    assert v.shape == ref.shape
    assert rel(v, ref) < 1e-10
    # entrywise on the single layer (every value is a positive integral)
    if kind == "slp":
        assert np.max(np.abs(v - ref) / np.abs(ref)) < 1e-10


@pytest.mark.parametrize("q", [3, 4])
def test_panel_pair_matrix_and_blocks_vs_reference(mesh3, q):
    """No singular table: touching pairs integrated at order q, as the
    reference's panel_pair_matrix(singular=None) does."""
    from paper_2001_05523_b200 import kernels

    g = golden("pairs.npz")
    ra, rb, verts = g["ra"], g["rb"], g["verts"]
    ppm = kernels.panel_pair_matrix(mesh3, ra, rb, "slp", q)
    assert ppm.shape == (len(ra), len(rb)) and rel(ppm, g[f"ppm_slp_q{q}"]) < 1e-10
    ppd = kernels.panel_pair_matrix(mesh3, ra, rb, "dlp", q)
    assert ppd.shape == (len(ra), len(rb), 3) and rel(ppd, g[f"ppm_dlp_q{q}"]) < 1e-10
    assert rel(kernels.slp_block(mesh3, ra, rb, q), g[f"slpb_q{q}"]) < 1e-10
    assert rel(kernels.dlp_block(mesh3, ra, verts, q), g[f"dlpb_q{q}"]) < 1e-10


def test_split_orders_with_table(mesh3):
    """The split-order call of SURVEY section 0: panel_pair_matrix(q_reg=3,
    singular=SingularTable(q_ss=4)) against the oracle with the same split."""
    from paper_2001_05523_b200 import kernels

    m = mesh3
    V, T, N, A = m.vertices, m.triangles, m.normals, m.areas
    rows = np.arange(0, 64)
    cols = np.arange(32, 128)
    for kind in ("slp", "dlp"):
        tab = kernels.SingularTable(m, kind, 4)  # reference signature (host mesh)
        otab = OQ.Table(V, T, N, A, kind, 4)
        got = kernels.panel_pair_matrix(m, rows, cols, kind, 3, singular=tab)
        want = OQ.pair_matrix(V, T, N, A, rows, cols, kind, 3, otab)
        assert rel(got, want) < 1e-10, kind
        # table lookups agree with the oracle table
        keys = tab.keys
        assert np.array_equal(keys, otab.keys)
        F = m.n_triangles
        sel = keys[::7]
        assert rel(tab.lookup(sel // F, sel % F), otab.lookup(sel // F, sel % F)) < 1e-10
        with pytest.raises(KeyError):
            tab.lookup(np.array([0]), np.array([F - 1]))


def test_require_disjoint_raises(mesh3):
    from paper_2001_05523_b200 import kernels

    with pytest.raises(ValueError):
        kernels.slp_block(mesh3, [0, 1], [1, 2], 3, require_disjoint=True)
    with pytest.raises(ValueError):
        kernels.dlp_block(mesh3, [0], [int(mesh3.triangles[0, 0])], 3, require_disjoint=True)
    with pytest.raises(ValueError):
        kernels.pair_integrals(mesh3, [0], [1], "hyp", 3)
    # separated panels pass
    far = np.flatnonzero(~np.isin(mesh3.triangles, mesh3.triangles[0]).any(axis=1))[:5]
    assert kernels.slp_block(mesh3, [0], far, 3, require_disjoint=True).shape == (1, 5)


@pytest.fixture(scope="module")
def cfg0_basis():
    g = golden("h2_cfg0.npz")
    m = sphere(4)
    t0, _ = trees(m, 32)
    b = basis_from_arrays(t0, g["ranks"], g["pivots"], g["V"], g["E"])
    return t0, b


def test_basis_forward_backward_vs_oracle(cfg0_basis):
    """ClusterBasis.forward / backward on the reference's config-0 basis
    against the oracle restatement of containers.py:201-228."""
    import torch

    t0, b = cfg0_basis
    rng = np.random.default_rng(3)
    xp = rng.standard_normal(t0.n_dofs)
    ot = oracle_tree(t0)
    want = OH.forward(ot, b.V, b.E, b.rank, xp)
    got = b.forward(xp)
    assert set(got) == set(want)
    for u in want:
        assert rel(got[u], want[u]) < 1e-13, u
    # device tensors in -> device tensors out, same values
    gd = b.forward(torch.from_numpy(xp).cuda())
    assert all(torch.is_tensor(v) and np.array_equal(v.cpu().numpy(), got[u]) for u, v in gd.items())
    # backward: coefficients on a few clusters at different depths
    picks = [int(u) for u in rng.choice(t0.n_nodes, 12, replace=False)]
    yhat = {u: rng.standard_normal(b.rank[u]) for u in picks}
    yhat_o = {u: v.copy() for u, v in yhat.items()}
    yp = rng.standard_normal(t0.n_dofs)
    yp_o = yp.copy()
    OH.backward(ot, b.V, b.E, yhat_o, yp_o)
    out = b.backward(yhat, yp)
    assert out is yp
    assert rel(yp, yp_o) < 1e-13
    assert set(yhat) == set(yhat_o)
    for u in yhat_o:
        assert rel(yhat[u], yhat_o[u]) < 1e-13


def test_forward_transform_single_leaf(cfg0_basis):
    """Port of the reference's test_forward_transform_single_leaf
    (pkg/tests/test_containers.py:132-147): the transfer recursion equals the
    expanded basis V_t^T x|_t of every cluster."""
    t0, b = cfg0_basis
    rng = np.random.default_rng(4)
    xp = rng.standard_normal(t0.n_dofs)
    xhat = b.forward(xp)
    for c in t0.nodes:
        direct = b.expand(c).T @ xp[c.start : c.end]
        assert np.allclose(xhat[c.uid], direct, rtol=1e-12, atol=1e-12 * np.abs(direct).max())
    # a unit vector supported on one leaf: only that leaf and its ancestors see it
    leaf = t0.leaves()[3]
    e = np.zeros(t0.n_dofs)
    e[leaf.start] = 1.0
    xh = b.forward(e)
    anc = set()
    c = leaf
    while c is not None:
        anc.add(c.uid)
        c = c.parent
    for u, v in xh.items():
        if u not in anc:
            assert not np.any(v)
    assert np.allclose(xh[leaf.uid], b.V[leaf.uid][0], rtol=1e-14, atol=0)
