"""Pin the CPU oracle against the reference's own outputs (tests/golden/)."""

import numpy as np
import pytest

from oracle import h2 as OH
from oracle import quad as OQ
from oracle import rules as OR

from .conftest import golden
from .helpers import basis_from_arrays, oracle_tree, rel, sphere, trees


def test_rules_bit_exact():
    g = golden("rules.npz")
    for q in range(1, 9):
        x, w = OR.gauss01(q)
        assert np.array_equal(x, g[f"gl{q}_x"]) and np.array_equal(w, g[f"gl{q}_w"])
    for q in (2, 3, 4, 5):
        p, w = OR.duffy(q)
        assert np.array_equal(p, g[f"tri{q}_p"]) and np.array_equal(w, g[f"tri{q}_w"])
    for case, name in (("identical", "identical"), ("edge", "shared_edge"), ("vertex", "shared_vertex")):
        for q in (3, 4, 5):
            p, w = OR.ss_rule(case, q)
            assert np.array_equal(p, g[f"ss_{name}_{q}_p"]), (case, q)
            assert np.array_equal(w, g[f"ss_{name}_{q}_w"]), (case, q)


def test_ss_weight_sum_quarter():
    # tests/test_quadrature.py:85-89 of the reference
    for case in ("identical", "edge", "vertex"):
        _, w = OR.ss_rule(case, 4)
        assert abs(w.sum() - 0.25) < 1e-13


@pytest.mark.parametrize("level", [2, 4])
def test_touching_pairs_and_classification(level):
    g = golden("touch.npz")
    m = sphere(level)
    keys = OQ.touching_pairs(m.triangles, m.n_vertices)
    F = m.n_triangles
    code, pa, pb = OQ.classify(m.triangles[keys // F], m.triangles[keys % F], keys // F == keys % F)
    assert np.array_equal(keys, g[f"l{level}_keys"])
    assert np.array_equal(code, g[f"l{level}_codes"])
    assert np.array_equal(np.hstack([pa, pb]), g[f"l{level}_perms"])


@pytest.mark.parametrize("q", [3, 4, 5])
@pytest.mark.parametrize("kind", ["slp", "dlp"])
def test_singular_integrals(kind, q):
    s = golden("singular.npz")
    m = sphere(4)
    v = OQ.singular_integrals(m.vertices, m.triangles, m.normals, m.areas, s["pa"], s["pb"], kind, q)
    assert rel(v, s[f"{kind}_q{q}"]) < 1e-12


@pytest.mark.parametrize("q", [3, 4])
@pytest.mark.parametrize("kind", ["slp", "dlp"])
def test_regular_pair_matrix(kind, q):
    s = golden("singular.npz")
    m = sphere(4)
    tb = OQ.Table(m.vertices, m.triangles, m.normals, m.areas, kind, q)
    v = OQ.pair_matrix(m.vertices, m.triangles, m.normals, m.areas, s["reg_rows"], s["reg_cols"], kind, q, tb)
    assert rel(v, s[f"reg_{kind}_q{q}"]) < 1e-12


@pytest.fixture(scope="module")
def cfg0_oracle_operator():
    """Config 0 assembled entirely by the oracle on the reference's basis."""
    from paper_2001_05523_b200 import clustering as C

    g = golden("h2_cfg0.npz")
    m = sphere(4)
    t0, _ = trees(m, 32)
    bt = C.BlockTree(t0, t0, 2.0)
    b = basis_from_arrays(t0, g["ranks"], g["pivots"], g["V"], g["E"])
    V, T, N, A = m.vertices, m.triangles, m.normals, m.areas
    tab = OQ.Table(V, T, N, A, "slp", 4)
    near = [OQ.slp_block(V, T, N, A, t0.perm[t0.start[t] : t0.end[t]], t0.perm[t0.start[s] : t0.end[s]], 3, tab)
            for t, s in bt.near_uids]
    far = [OQ.slp_block(V, T, N, A, b.pivots[t], b.pivots[s], 3, None) for t, s in bt.far_uids]
    return g, t0, bt, b, near, far


def test_oracle_nearfield_and_couplings_vs_reference(cfg0_oracle_operator):
    g, t0, bt, b, near, far = cfg0_oracle_operator
    got = np.concatenate([near[i].ravel() for i in g["near_sel"]])
    assert rel(got, g["near_vals"]) < 1e-11
    got = np.concatenate([far[i].ravel() for i in g["far_sel"]])
    assert rel(got, g["far_vals"]) < 1e-11


def test_oracle_matvec_vs_reference(cfg0_oracle_operator):
    g, t0, bt, b, near, far = cfg0_oracle_operator
    ot = oracle_tree(t0)
    y = OH.matvec(ot, ot, b.V, b.E, b.rank, b.V, b.E, b.rank, bt.far_uids, far, bt.near_uids, near, g["x"])
    assert rel(y, g["y"]) < 1e-10
    d = OH.diagonal(ot, ot, bt.near_uids, near)
    assert rel(d, g["diag"]) < 1e-11
    # accuracy of the H^2 approximation itself (reference: 2.5e-4 at eps 1e-4)
    assert np.linalg.norm(y - g["y_dense"]) <= 1e-3 * np.linalg.norm(g["y_dense"])


@pytest.mark.parametrize("q", [2, 3, 4])
@pytest.mark.parametrize("kind", ["slp", "dlp"])
def test_pair_integrals_any_case(kind, q):
    """kernels.pair_integrals on a mixed list (mostly separated panels: the
    disjoint-case tensor rule of quadrature.py:171-180)."""
    g = golden("pairs.npz")
    m = sphere(3)
    assert (g["code"] == 0).sum() > 300
    v = OQ.singular_integrals(m.vertices, m.triangles, m.normals, m.areas, g["pa"], g["pb"], kind, q)
    assert rel(v, g[f"{kind}_q{q}"]) < 1e-12
