"""Bit-exact structure layer vs the reference (mesh, cluster trees, block trees)."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2001_05523_b200 import clustering as C
from paper_2001_05523_b200 import mesh as M
from paper_2001_05523_b200 import spaces as S

from .conftest import GOLDEN, golden


def digest(a, dtype=None):
    a = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    return hashlib.sha256(a.tobytes()).hexdigest()


def test_sphere_level2_exact():
    g = golden("mesh.npz")
    m = M.sphere_mesh(2)
    for a, k in ((m.vertices, "l2_vertices"), (m.triangles, "l2_triangles"), (m.normals, "l2_normals"),
                 (m.areas, "l2_areas")):
        assert np.array_equal(a, g[k])


@pytest.mark.parametrize("level", [4, 6, 8])
def test_sphere_digests(level):
    meta = json.load(open(os.path.join(GOLDEN, "mesh_digests.json")))[str(level)]
    m = M.sphere_mesh(level)
    assert m.n_triangles == meta["n_triangles"] == 8 * 4**level
    assert digest(m.vertices) == meta["vertices"]
    assert digest(m.triangles, np.int64) == meta["triangles"]
    assert digest(m.normals) == meta["normals"]
    assert digest(m.areas) == meta["areas"]


@pytest.mark.parametrize("name,level,leaf,eta", [("cfg0", 4, 32, 2.0), ("cfg1", 6, 64, 2.0)])
def test_trees_and_blocks_exact(name, level, leaf, eta):
    st = golden(f"struct_{name}.npz")
    m = M.sphere_mesh(level)
    trees = {}
    for sp, kind in (("p0", S.P0), ("p1", S.P1)):
        boxes = S.DofSpace(kind, m).support_boxes()
        assert np.array_equal(boxes, st[f"{sp}_support"])
        t = C.build_cluster_tree(boxes, leaf)
        for a in ("perm", "start", "end", "left", "right", "boxes"):
            assert np.array_equal(getattr(t, a), st[f"{sp}_{a}"]), a
        assert np.array_equal(t.depth_of, st[f"{sp}_depth"])
        trees[sp] = t
    bt = C.BlockTree(trees["p0"], trees["p0"], eta)
    assert np.array_equal(bt.far_uids, st["slp_far"]) and np.array_equal(bt.near_uids, st["slp_near"])
    assert bt.check_partition()
    bt = C.BlockTree(trees["p0"], trees["p1"], eta)
    assert np.array_equal(bt.far_uids, st["dlp_far"]) and np.array_equal(bt.near_uids, st["dlp_near"])
    assert bt.check_partition()


def _structure_digest(mesh, leaf, eta, col_space):
    rt = C.build_cluster_tree(S.DofSpace(S.P0, mesh).support_boxes(), leaf)
    ct = rt if col_space == S.P0 else C.build_cluster_tree(S.DofSpace(col_space, mesh).support_boxes(), leaf)
    bt = C.BlockTree(rt, ct, eta)
    out = {"n_far": len(bt.far_uids), "n_near": len(bt.near_uids), "far": digest(bt.far_uids),
           "near": digest(bt.near_uids)}
    for name, t in (("row", rt), ("col", ct)):
        out[f"{name}_nodes"] = t.n_nodes
        out[f"{name}_perm"] = digest(t.perm)
        out[f"{name}_ranges"] = digest(np.stack([t.start, t.end, t.depth_of, t.left, t.right]))
        out[f"{name}_boxes"] = digest(t.boxes)
    return out


@pytest.mark.parametrize("key,level,eta,col", [("cfg2_slp", 8, 2.0, S.P0), ("cfg2_dlp", 8, 2.0, S.P1),
                                               ("cfg3_slp", 9, 1.5, S.P0)])
def test_large_structure_digests(key, level, eta, col):
    meta = json.load(open(os.path.join(GOLDEN, "struct_large.json")))[key]
    got = _structure_digest(M.sphere_mesh(level), 64, eta, col)
    assert got == meta


def test_admissibility_examples():
    a = np.array([[0.0, 0, 0], [1, 1, 1]])
    b = np.array([[3.0, 0, 0], [4, 1, 1]])
    assert C.admissible(a, b, 1.0)
    assert not C.admissible(a, b, 0.4)
    with pytest.raises(ValueError):
        C.admissible(a, b, 0.0)


def test_tiny_eta_is_all_nearfield():
    m = M.sphere_mesh(2)
    t = C.build_cluster_tree(S.DofSpace(S.P0, m).support_boxes(), 8)
    bt = C.BlockTree(t, t, 1e-9)
    assert len(bt.far_uids) == 0 and bt.check_partition()


def test_degenerate_inputs():
    with pytest.raises(ValueError):
        C.build_cluster_tree(np.zeros((0, 2, 3)), 4)
    with pytest.raises(ValueError):
        C.build_cluster_tree(np.zeros((3, 2, 3)), 0)
    # identical boxes: median fallback splits the index set in halves
    t = C.build_cluster_tree(np.zeros((10, 2, 3)), 2)
    assert sorted(t.perm.tolist()) == list(range(10))
    assert all(n.size <= 2 for n in t.leaves())


def test_mesh_validation_and_io(tmp_path):
    m = M.sphere_mesh(1)
    p = tmp_path / "s.txt"
    M.write_mesh(m, p)
    r = M.read_mesh(p)
    assert np.array_equal(r.vertices, m.vertices) and np.array_equal(r.triangles, m.triangles)
    bad = M.SurfaceMesh(m.vertices, m.triangles[:-1])
    with pytest.raises(M.MeshError):
        bad.validate()
    flipped = m.triangles.copy()
    flipped[0] = flipped[0, ::-1]
    with pytest.raises(M.MeshError):
        M.SurfaceMesh(m.vertices, flipped).validate()


def test_cube_shell_mesh():
    m = M.cube_shell_mesh(2)
    assert m.n_triangles == 60 * 2 * 4
    # outer volume 27 minus the cavity 1
    assert abs(m.signed_volume() - 26.0) < 1e-12


def test_cube_shell_structure_exact():
    """Config-4 geometry (grid-aligned flat panels: split coordinates tie
    exactly) -- trees and block trees bit-exact vs the reference run on the
    same mesh arrays (tests/golden/make_golden.py gen_cube)."""
    g = golden("cube4.npz")
    m = M.cube_shell_mesh(4)
    assert np.array_equal(m.vertices, g["vertices"]) and np.array_equal(m.triangles, g["triangles"])
    trees = {}
    for sp, kind in (("p0", S.P0), ("p1", S.P1)):
        t = C.build_cluster_tree(S.DofSpace(kind, m).support_boxes(), 32)
        for a in ("perm", "start", "end", "left", "right", "boxes"):
            assert np.array_equal(getattr(t, a), g[f"{sp}_{a}"]), (sp, a)
        assert np.array_equal(t.depth_of, g[f"{sp}_depth"])
        trees[sp] = t
    bt = C.BlockTree(trees["p0"], trees["p0"], 2.0)
    assert np.array_equal(bt.far_uids, g["slp_far"]) and np.array_equal(bt.near_uids, g["slp_near"])
    bt = C.BlockTree(trees["p0"], trees["p1"], 2.0)
    assert np.array_equal(bt.far_uids, g["dlp_far"]) and np.array_equal(bt.near_uids, g["dlp_near"])
