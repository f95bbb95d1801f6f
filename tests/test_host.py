"""Host-side product logic: rules, GCA basis construction, ABI surface."""

import ctypes
import re

import numpy as np
import pytest

from paper_2001_05523_b200 import _lib, gca
from paper_2001_05523_b200 import quadrature as quad
from paper_2001_05523_b200 import spaces as S
from paper_2001_05523_b200.containers import AssemblyContext
from paper_2001_05523_b200.lowrank import aca_inverse_core

from .conftest import ROOT, golden
from .helpers import sphere, trees


def test_product_rules_match_reference_bits():
    g = golden("rules.npz")
    for q in range(1, 9):
        r = quad.gauss_legendre(q)
        assert np.array_equal(r.points, g[f"gl{q}_x"]) and np.array_equal(r.weights, g[f"gl{q}_w"])
    for q in (2, 3, 4, 5):
        p, w = quad.triangle_rule(q)
        assert np.array_equal(p, g[f"tri{q}_p"]) and np.array_equal(w, g[f"tri{q}_w"])
    for case in (quad.IDENTICAL, quad.SHARED_EDGE, quad.SHARED_VERTEX, quad.DISJOINT):
        for q in (3, 4, 5):
            r = quad.sauter_schwab_rule(case, q)
            assert np.array_equal(r.points, g[f"ss_{case}_{q}_p"]), (case, q)
            assert np.array_equal(r.weights, g[f"ss_{case}_{q}_w"]), (case, q)
            assert len(r.weights) == quad.SUBDOMAINS[case] * q**4


def test_classify_panel_pair():
    assert quad.classify_panel_pair([0, 1, 2], [0, 1, 2])[0] == quad.IDENTICAL
    case, pa, pb = quad.classify_panel_pair([5, 7, 9], [9, 7, 11])
    assert case == quad.SHARED_EDGE and pa == (1, 2, 0) and pb == (1, 0, 2)
    case, pa, pb = quad.classify_panel_pair([5, 7, 9], [1, 2, 9])
    assert case == quad.SHARED_VERTEX and pa == (2, 0, 1) and pb == (2, 0, 1)
    assert quad.classify_panel_pair([0, 1, 2], [3, 4, 5])[0] == quad.DISJOINT


def test_gca_basis_bit_exact_cfg0():
    g = golden("h2_cfg0.npz")
    m = sphere(4)
    t0, _ = trees(m, 32)
    b = gca.build_basis(AssemblyContext(m), t0, gca.P0_SLP, 3, 1e-4, threads=4)
    ranks = np.array([b.rank[u] for u in range(t0.n_nodes)])
    piv = np.concatenate([b.pivots[u] for u in range(t0.n_nodes)])
    assert np.array_equal(ranks, g["ranks"]) and np.array_equal(piv, g["pivots"])
    V = np.concatenate([b.V[u].ravel() for u in t0.leaf_uids()])
    E = np.concatenate([b.E[u].ravel() for u in range(t0.n_nodes) if u in b.E])
    assert np.array_equal(V, g["V"]) and np.array_equal(E, g["E"])


def test_gca_dlp_bases_bit_exact_level4():
    g = golden("h2_dlp4.npz")
    m = sphere(4)
    t0, t1 = trees(m, 32)
    ctx = AssemblyContext(m)
    for prefix, tree, flavor in (("row_", t0, gca.P0_SLP), ("col_", t1, gca.P1_DLP)):
        b = gca.build_basis(ctx, tree, flavor, 3, 1e-4, threads=4)
        ranks = np.array([b.rank[u] for u in range(tree.n_nodes)])
        piv = np.concatenate([b.pivots[u] for u in range(tree.n_nodes)])
        assert np.array_equal(ranks, g[prefix + "ranks"]) and np.array_equal(piv, g[prefix + "pivots"])
        V = np.concatenate([b.V[u].ravel() for u in tree.leaf_uids()])
        assert np.abs(V - g[prefix + "V"]).max() <= 1e-12 * np.abs(g[prefix + "V"]).max()


@pytest.mark.slow
def test_gca_pivots_cfg1():
    g = golden("h2_cfg1.npz")
    m = sphere(6)
    t0, _ = trees(m, 64)
    b = gca.build_basis(AssemblyContext(m), t0, gca.P0_SLP, 4, 1e-4, threads=8)
    ranks = np.array([b.rank[u] for u in range(t0.n_nodes)])
    piv = np.concatenate([b.pivots[u] for u in range(t0.n_nodes)])
    assert np.array_equal(ranks, g["ranks"]) and np.array_equal(piv, g["pivots"])


def test_aca_inverse_core_properties(rng):
    # reference tests/test_lowrank.py:94-127
    u = rng.standard_normal(8)
    v = rng.standard_normal(6)
    tau, sigma, C, ok = aca_inverse_core(np.outer(u, v), 1e-12)
    assert len(tau) == 1 and ok
    A = rng.standard_normal((20, 5)) @ rng.standard_normal((5, 15))
    tau, sigma, C, ok = aca_inverse_core(A, 1e-10)
    R = A[:, sigma] @ C @ A[tau, :]
    assert np.linalg.norm(R - A) <= 1e-8 * np.linalg.norm(A)
    with pytest.raises(ValueError):
        aca_inverse_core(np.array([[np.nan]]), 1e-3)
    tau, sigma, C, ok = aca_inverse_core(np.zeros((3, 3)), 1e-3)
    assert len(tau) == 0 and ok


def test_green_quadrature_integrates_area():
    gq = gca.green_quadrature(np.array([[0.0, 0, 0], [1.0, 2.0, 3.0]]), 3)
    assert len(gq.weights) == 6 * 9
    assert abs(gq.weights.sum() - 2 * (2 * 3 + 1 * 3 + 1 * 2)) < 1e-12


def test_support_boxes_contain_dofs():
    m = sphere(2)
    b1 = S.DofSpace(S.P1, m).support_boxes()
    assert (b1[:, 0, :] <= m.vertices).all() and (m.vertices <= b1[:, 1, :]).all()


def test_library_exports_every_declared_symbol():
    """libh2b.so loads without a GPU and exports what include/h2b.h declares."""
    header = open(f"{ROOT}/include/h2b.h").read()
    declared = set(re.findall(r"\bint\s+(h2b_\w+)\s*\(", header))
    assert declared == set(_lib.EXPORTS)
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name)
    assert L.h2b_abi_version() == 1
    # error plumbing works without a device
    rc = L.h2b_cluster_tree(None, 0, 1, None, None, None, None, None, None, None, None)
    assert rc == _lib.H2B_ERR_INVALID
    with pytest.raises(ValueError, match="empty index set"):
        _lib.check(rc)
    assert "empty" in _lib.last_error()
    rc = L.h2b_plan_create(None, ctypes.byref(ctypes.c_void_p()))
    assert rc == _lib.H2B_ERR_INVALID


def test_native_dlp_job_builder_matches_restatement():
    """h2b_dlp_jobs_build (C++) == the Python restatement of the column-panel
    tiling, element for element: near blocks of a P0 x P1 block tree plus
    ragged and single-vertex blocks."""
    import numpy as np

    from paper_2001_05523_b200 import clustering as C, kernels, spaces
    from paper_2001_05523_b200.containers import near_layout
    from paper_2001_05523_b200.mesh import sphere_mesh

    m = sphere_mesh(4)
    t_r = C.build_cluster_tree(spaces.DofSpace(spaces.P0, m).support_boxes(), 32)
    t_c = C.build_cluster_tree(spaces.DofSpace(spaces.P1, m).support_boxes(), 32)
    bt = C.BlockTree(t_r, t_c, 2.0)
    nl = near_layout(bt)
    blocks = [(t_r.perm[t_r.start[t] : t_r.end[t]], t_c.perm[t_c.start[s] : t_c.end[s]], int(nl.blk_off[i]),
               int(nl.blk_ld[i])) for i, (t, s) in enumerate(bt.near_uids)]
    rng = np.random.default_rng(0)
    blocks.append((np.arange(70), rng.permutation(m.n_vertices)[:130], 5, 130))  # > one tile both ways
    blocks.append((np.array([3]), np.array([7]), 0, 1))
    a = kernels.build_dlp_jobs(m, blocks)
    b = kernels._build_dlp_jobs_py(m, blocks)
    assert set(a) == set(b)
    for k in a:
        assert a[k].dtype == b[k].dtype and np.array_equal(a[k], b[k]), k
    assert kernels.build_dlp_jobs(m, []) is None


def test_mirror_and_tile_jobs_cover_every_entry_once():
    """Host job logic of the symmetric single-layer assembly: every entry of
    every block is written exactly once (directly or as a mirror), diagonal
    blocks larger than a tile keep their upper-triangle tiles only."""
    from paper_2001_05523_b200 import kernels

    sizes = {0: 100, 1: 40, 2: 70}
    uids = np.array([(0, 0), (0, 1), (1, 0), (1, 1), (2, 0), (0, 2), (1, 2), (2, 2)])
    off, jobs, start = 0, [], {0: 0, 1: 100, 2: 140}
    blocks = {}
    for t, s in uids:
        nr, nc = sizes[t], sizes[s]
        jobs.append((start[t], nr, start[s], nc, off, nc))
        blocks[(t, s)] = (off, nc, nr)
        off += nr * nc
    jobs = kernels.tile_jobs(kernels.mirror_jobs(np.array(jobs), uids[:, ::-1][:, ::-1]))
    hits = np.zeros(off, dtype=np.int64)
    for r0, nr, c0, nc, o, ld, mo, mld in jobs:
        assert nr <= kernels.TILE and nc <= kernels.TILE
        tri = mo == o
        for a in range(nr):
            for b in range(nc):
                if tri and a > b:
                    continue
                hits[o + a * ld + b] += 1
                if mo >= 0 and not (tri and a == b):
                    hits[mo + b * mld + a] += 1
    assert (hits == 1).all()


def test_green_points_batch_matches_per_cluster_bits():
    from paper_2001_05523_b200 import gca

    rng = np.random.default_rng(5)
    lo = rng.uniform(-1, 1, (40, 3))
    ext = rng.uniform(0, 0.5, (40, 3))
    ext[::7, 1] = 0.0  # flat boxes are widened
    boxes = np.stack([lo, lo + ext], axis=1)
    for m in (3, 4, 5):
        got = gca.green_points_batch(boxes, m)
        for i, box in enumerate(boxes):
            gq = gca.green_quadrature(gca.green_box(box), m)
            assert np.array_equal(got[i, :, :3], gq.points)
            assert np.array_equal(got[i, :, 3], np.sqrt(gq.weights))
            assert np.array_equal(got[i, :, 4:7], gq.normals)


def test_gca_pivots_bit_exact_cube_shell():
    """Host GCA basis on the config-4 geometry: ranks and pivots bit-exact."""
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200.mesh import cube_shell_mesh

    g = golden("cube4.npz")
    m = cube_shell_mesh(4)
    t0 = C.build_cluster_tree(S.DofSpace(S.P0, m).support_boxes(), 32)
    b = gca.build_basis(AssemblyContext(m), t0, gca.P0_SLP, 3, 1e-4, threads=4)
    assert np.array_equal(np.array([b.rank[u] for u in range(t0.n_nodes)]), g["slp_ranks"])
    assert np.array_equal(np.concatenate([b.pivots[u] for u in range(t0.n_nodes)]), g["slp_pivots"])


def test_native_block_jobs_match_numpy_restatement():
    """h2b_block_partners / h2b_block_jobs (one native pass) against the numpy
    chain they replace (block partners by sort + search, stacked job columns,
    mirror_jobs), on the sphere level-4 block tree with made-up ranks: far
    blocks (coupling jobs) and near blocks, mirrored and one-sided."""
    from paper_2001_05523_b200 import clustering, kernels, mesh, spaces

    m = mesh.sphere_mesh(4)
    tree = clustering.build_cluster_tree(spaces.DofSpace(spaces.P0, m).support_boxes(), 16)
    bt = clustering.BlockTree(tree, tree, 1.2)
    rng = np.random.default_rng(5)
    rank = rng.integers(3, 20, tree.n_nodes).astype(np.int64)
    off = np.zeros(tree.n_nodes + 1, dtype=np.int64)
    np.cumsum(rank, out=off[1:])
    for uids, r_off, r_cnt in ((bt.far_uids, off[:-1], rank), (bt.near_uids, tree.start, tree.end - tree.start)):
        uids = np.asarray(uids, dtype=np.int64)
        part = kernels.block_partners(uids)
        assert np.array_equal(part, kernels._block_partners_py(uids))
        assert (part >= 0).all()  # one tree on both sides: every block has its transpose
        blk_ld = r_cnt[uids[:, 1]] + 3
        blk_off = np.cumsum(r_cnt[uids[:, 0]] * blk_ld) - r_cnt[uids[:, 0]] * blk_ld
        six = np.stack([r_off[uids[:, 0]], r_cnt[uids[:, 0]], r_off[uids[:, 1]], r_cnt[uids[:, 1]], blk_off, blk_ld],
                       axis=1)
        got = kernels.block_jobs(uids, r_off, r_cnt, r_off, r_cnt, blk_off, blk_ld, part)
        assert np.array_equal(got, kernels.mirror_jobs(six, uids, part))
        assert len(got) < len(uids)
        one = kernels.block_jobs(uids, r_off, r_cnt, r_off, r_cnt, blk_off, blk_ld, None)
        assert np.array_equal(one, kernels._as_job8(six))
    # a list with unpaired blocks and a diagonal block
    uids = np.array([(0, 1), (2, 2), (1, 0), (3, 1), (0, 3)], dtype=np.int64)
    part = kernels.block_partners(uids)
    assert part.tolist() == [2, 1, 0, -1, -1]
    cnt = np.array([4, 5, 6, 7], dtype=np.int64)
    o = np.array([0, 4, 9, 15], dtype=np.int64)
    bo = np.arange(5, dtype=np.int64) * 100
    bl = cnt[uids[:, 1]]
    six = np.stack([o[uids[:, 0]], cnt[uids[:, 0]], o[uids[:, 1]], cnt[uids[:, 1]], bo, bl], axis=1)
    assert np.array_equal(kernels.block_jobs(uids, o, cnt, o, cnt, bo, bl, part), kernels.mirror_jobs(six, uids, part))
    assert len(kernels.block_jobs(uids[:0], o, cnt, o, cnt, bo[:0], bl[:0], part[:0])) == 0
