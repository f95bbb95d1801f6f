"""GPU GCA basis construction (gca.build_basis(device=True)) vs the host path,
which reproduces the reference's pivots bit for bit (tests/test_host.py)."""

import numpy as np
import pytest

from .helpers import sphere, trees

pytestmark = pytest.mark.gpu


def _compare(bh, bd, tree):
    same = {u for u in range(tree.n_nodes)
            if bh.rank[u] == bd.rank[u] and np.array_equal(bh.pivots[u], bd.pivots[u])}
    frac = len(same) / tree.n_nodes
    worst = 0.0

    def rel(a, b):
        return float(np.abs(a - b).max() / max(np.abs(a).max(), 1e-300)) if a.size else 0.0

    for u in same:
        if u in bh.V:
            worst = max(worst, rel(bh.V[u], bd.V[u]))
        # a transfer matrix is a row block of the parent's interpolation matrix
        if u in bh.E and tree.parent_of[u] in same and all(ch.uid in same for ch in
                                                           tree.nodes[tree.parent_of[u]].children):
            worst = max(worst, rel(bh.E[u], bd.E[u]))
    return frac, worst


@pytest.mark.parametrize("flavor", ["p0_slp", "p1_dlp", "p1_curl"])
def test_device_basis_matches_host_cfg0(flavor):
    from paper_2001_05523_b200 import gca
    from paper_2001_05523_b200.containers import AssemblyContext

    m = sphere(4)
    t0, t1 = trees(m, 32)
    tree = t0 if flavor == "p0_slp" else t1
    ctx = AssemblyContext(m)
    bh = gca.build_basis(ctx, tree, flavor, 3, 1e-4, threads=4)
    bd = gca.build_basis(ctx, tree, flavor, 3, 1e-4, device=True)
    frac, worst = _compare(bh, bd, tree)
    assert frac >= 0.97, frac
    assert worst < 1e-9, worst


def test_device_basis_operator_accuracy_cfg0():
    """H^2 operators from both bases are equally accurate against the dense
    Galerkin matrix, and agree with each other to the GCA tolerance."""
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import gca
    from paper_2001_05523_b200.containers import AssemblyContext, assemble_dense

    m = sphere(4)
    t0, _ = trees(m, 32)
    ctx = AssemblyContext(m)
    bt = C.BlockTree(t0, t0, 2.0)
    bh = gca.build_basis(ctx, t0, gca.P0_SLP, 3, 1e-4, threads=4)
    bd = gca.build_basis(ctx, t0, gca.P0_SLP, 3, 1e-4, device=True)
    Hh = gca.assemble_h2(ctx, "slp", bt, bh, bh, 3, q_singular=4)
    Hd = gca.assemble_h2(ctx, "slp", bt, bd, bd, 3, q_singular=4)
    G = assemble_dense(ctx, "slp", 3, q_singular=4)
    x = np.random.default_rng(0).uniform(-1, 1, G.shape[1])
    ref = G @ x
    eh = np.linalg.norm(Hh.matvec(x) - ref) / np.linalg.norm(ref)
    ed = np.linalg.norm(Hd.matvec(x) - ref) / np.linalg.norm(ref)
    assert ed < 1e-3 and ed <= 2.0 * eh + 1e-12, (ed, eh)


def test_device_curl_basis_hyp_operator():
    """P1_CURL basis on the GPU (h2b_gca_columns_curl + h2b_gca_aca with 6k
    columns) -> hypersingular H^2 operator: agrees with the reference's matvec
    on tests/golden/h2_hyp4.npz to the GCA tolerance, like the host basis."""
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import gca
    from paper_2001_05523_b200.containers import AssemblyContext

    from .conftest import golden

    g = golden("h2_hyp4.npz")
    m = sphere(4)
    _, t1 = trees(m, 32)
    ctx = AssemblyContext(m)
    bt = C.BlockTree(t1, t1, 2.0)
    bd = gca.build_basis(ctx, t1, gca.P1_CURL, 3, 1e-4, device=True)
    ranks = np.array([bd.rank[u] for u in range(t1.n_nodes)])
    assert np.abs(ranks - g["ranks"]).max() <= 2
    Hd = gca.assemble_h2(ctx, "hyp", bt, bd, bd, 3, q_singular=4)
    y = Hd.matvec(g["x"])
    assert np.linalg.norm(y - g["y"]) / np.linalg.norm(g["y"]) < 1e-3


def test_problem_setup_with_device_basis():
    """Public API: RunParams(gca_device=True) -> ProblemSetup.operator builds
    the bases on the GPU; the operator matches the dense Galerkin product to
    the GCA tolerance and the host-basis operator closely."""
    from paper_2001_05523_b200.containers import assemble_dense
    from paper_2001_05523_b200.driver import ProblemSetup
    from paper_2001_05523_b200.params import RunParams

    m = sphere(4)
    kw = dict(order=3, q_near=3, q_singular=4, r_leaf=32, eta=2.0, eps_aca=1e-4, threads=4)
    Sd = ProblemSetup(m, RunParams(gca_device=True, **kw).resolved())
    Sh = ProblemSetup(m, RunParams(**kw).resolved())
    x = np.random.default_rng(3).uniform(-1, 1, m.n_triangles)
    yd, yh = Sd.operator("slp").matvec(x), Sh.operator("slp").matvec(x)
    G = assemble_dense(Sd.ctx, "slp", 3, q_singular=4)
    ref = G @ x
    assert np.linalg.norm(yd - ref) / np.linalg.norm(ref) < 1e-3
    assert np.linalg.norm(yd - yh) / np.linalg.norm(yh) < 1e-3


def test_green_points_device_bit_identical():
    from paper_2001_05523_b200 import gca

    rng = np.random.default_rng(5)
    lo = rng.uniform(-1, 1, (64, 3))
    ext = rng.uniform(0, 0.5, (64, 3))
    ext[::7, 2] = 0.0
    boxes = np.stack([lo, lo + ext], axis=1)
    for m in (3, 4, 5):
        assert np.array_equal(gca.green_points_batch_device(boxes, m).cpu().numpy(), gca.green_points_batch(boxes, m))
