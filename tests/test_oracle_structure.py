"""Pin the oracle's structure restatement (oracle/structure.py) against the
reference's own meshes, trees and block lists (tests/golden/, produced by
running the reference).  bench.py's reference arm builds its structure with
this restatement, so that arm never imports the product."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import structure as OS

from .conftest import GOLDEN, golden


def _digest(a, dtype=None):
    a = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    return hashlib.sha256(a.tobytes()).hexdigest()


def test_sphere_level2_arrays():
    g = golden("mesh.npz")
    V, T, N, A = OS.sphere(2)
    assert np.array_equal(V, g["l2_vertices"]) and np.array_equal(T, g["l2_triangles"])
    assert np.array_equal(N, g["l2_normals"]) and np.array_equal(A, g["l2_areas"])


@pytest.mark.parametrize("level", [4, 6, 8])
def test_sphere_digests(level):
    meta = json.load(open(os.path.join(GOLDEN, "mesh_digests.json")))[str(level)]
    V, T, N, A = OS.sphere(level)
    assert _digest(V) == meta["vertices"] and _digest(T, np.int64) == meta["triangles"]
    assert _digest(N) == meta["normals"] and _digest(A) == meta["areas"]


@pytest.mark.parametrize("name,level,leaf,eta", [("cfg0", 4, 32, 2.0), ("cfg1", 6, 64, 2.0)])
def test_cluster_and_block_tree(name, level, leaf, eta):
    g = golden(f"struct_{name}.npz")
    V, T, _, _ = OS.sphere(level)
    boxes = OS.p0_boxes(V, T)
    assert np.array_equal(boxes, g["p0_support"])
    t = OS.cluster_tree(boxes, leaf)
    for k, v in (("perm", t.perm), ("start", t.start), ("end", t.end), ("depth", t.depth), ("left", t.left),
                 ("right", t.right), ("boxes", t.boxes)):
        assert np.array_equal(v, g[f"p0_{k}"]), k
    far, near = OS.block_tree(t, t, eta)
    assert np.array_equal(far, g["slp_far"]) and np.array_equal(near, g["slp_near"])
    # a row slice: the same lists filtered to the slice's rows and ancestors
    keep = np.zeros(t.n_nodes, dtype=bool)
    u = int(t.left[t.left[0]])
    keep[(t.start >= t.start[u]) & (t.end <= t.end[u])] = True
    p = u
    while p >= 0:
        keep[p] = True
        p = int(t.parent[p])
    f2, n2 = OS.block_tree(t, t, eta, row_keep=keep)
    assert np.array_equal(f2, far[keep[far[:, 0]]]) and np.array_equal(n2, near[keep[near[:, 0]]])


def test_config3_structure_digests():
    """Config 3 (sphere level 9, leaf 64, eta 1.5) in full: the tree and the
    970 336 far / 480 864 near blocks in the reference's order (digests)."""
    meta = json.load(open(os.path.join(GOLDEN, "struct_large.json")))["cfg3_slp"]
    V, T, _, _ = OS.sphere(9)
    t = OS.cluster_tree(OS.p0_boxes(V, T), 64)
    assert t.n_nodes == meta["row_nodes"] and _digest(t.perm) == meta["row_perm"]
    assert _digest(t.boxes) == meta["row_boxes"]
    far, near = OS.block_tree(t, t, 1.5)
    assert len(far) == meta["n_far"] and len(near) == meta["n_near"]
    assert _digest(far) == meta["far"] and _digest(near) == meta["near"]
