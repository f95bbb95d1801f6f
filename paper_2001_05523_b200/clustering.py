"""Cluster trees and block trees (host, native).  API of h2bem.clustering
(clustering.py:1-171); the recursion runs in libh2b (h2b_cluster_tree,
h2b_block_tree: C++ with exact IEEE evaluation) and is bit-exact with the
reference: same perm, node ranges, uid (preorder) order, far/near lists and
their order.  A level-9 sphere block tree takes well under a second instead of
~30 s of Python recursion."""

import ctypes

import numpy as np

from . import _lib


def box_diameter(box):
    return float(np.linalg.norm(box[1] - box[0]))


def box_distance(box_a, box_b):
    gaps = np.maximum(0.0, np.maximum(box_a[0] - box_b[1], box_b[0] - box_a[1]))
    return float(np.linalg.norm(gaps))


def admissible(box_t, box_s, eta):
    """max(diam B_t, diam B_s) <= 2 eta dist(B_t, B_s)."""
    if eta <= 0.0:
        raise ValueError("eta must be positive")
    return max(box_diameter(box_t), box_diameter(box_s)) <= 2.0 * eta * box_distance(box_t, box_s)


class Cluster:
    """Contiguous index range [start, end) of the permuted ordering."""

    __slots__ = ("start", "end", "box", "depth", "children", "uid", "parent")

    def __init__(self, start, end, box, depth, uid):
        self.start = start
        self.end = end
        self.box = box
        self.depth = depth
        self.children = []
        self.uid = uid
        self.parent = None

    @property
    def size(self):
        return self.end - self.start

    @property
    def is_leaf(self):
        return not self.children

    def __repr__(self):
        return f"Cluster([{self.start}:{self.end}), depth={self.depth})"


class ClusterTree:
    """Binary cluster tree; perm[p] = original dof at permuted position p.

    Besides the reference's object view (`nodes` in preorder, `root`), the
    tree keeps flat uid-indexed arrays (start, end, depth, left, right, boxes)
    that the device layout is packed from."""

    def __init__(self, perm, start, end, depth, left, right, boxes):
        self.perm = perm
        self.iperm = np.empty_like(perm)
        self.iperm[perm] = np.arange(len(perm))
        self.start, self.end, self.depth_of = start, end, depth
        self.left, self.right, self.boxes = left, right, boxes
        n = len(start)
        self.parent_of = np.full(n, -1, dtype=np.int64)
        inner = np.flatnonzero(left >= 0)
        self.parent_of[left[inner]] = inner
        self.parent_of[right[inner]] = inner
        nodes = [Cluster(int(start[u]), int(end[u]), boxes[u], int(depth[u]), u) for u in range(n)]
        for u in inner:
            nodes[u].children = [nodes[left[u]], nodes[right[u]]]
            nodes[left[u]].parent = nodes[u]
            nodes[right[u]].parent = nodes[u]
        self.nodes = nodes
        self.root = nodes[0]

    @property
    def n_dofs(self):
        return len(self.perm)

    @property
    def n_nodes(self):
        return len(self.nodes)

    def dofs(self, cluster):
        return self.perm[cluster.start : cluster.end]

    def leaves(self):
        return [c for c in self.nodes if c.is_leaf]

    def leaf_uids(self):
        return np.flatnonzero(self.left < 0)

    def bottom_up(self):
        """Children before parents (stable sort by decreasing depth)."""
        order = np.argsort(-self.depth_of, kind="stable")
        return [self.nodes[u] for u in order]

    def depth(self):
        return int(self.depth_of.max())

    def c_tree(self):
        """ctypes view for h2b_block_tree (keeps arrays alive on self)."""
        self._ct_keep = (np.ascontiguousarray(self.left), np.ascontiguousarray(self.right),
                         np.ascontiguousarray(self.boxes))
        return _lib.Tree(self.n_nodes, _lib.ptr(self._ct_keep[0]), _lib.ptr(self._ct_keep[1]),
                         _lib.ptr(self._ct_keep[2]))


def build_cluster_tree(boxes, r_leaf, device=False):
    """Geometric bisection of support boxes (clustering.py:78-121).
    device=True builds it on the GPU (h2b_cluster_tree_device, bit-exact with
    the host builder)."""
    boxes = np.ascontiguousarray(boxes, dtype=np.float64)
    n = len(boxes)
    if n == 0:
        raise ValueError("cannot build a cluster tree over an empty index set")
    if r_leaf < 1:
        raise ValueError("r_leaf must be >= 1")
    cap = 2 * n - 1
    perm = np.empty(n, dtype=np.int64)
    nn = np.zeros(1, dtype=np.int64)
    start, end, depth, left, right = (np.empty(cap, dtype=np.int64) for _ in range(5))
    nb = np.empty((cap, 2, 3))
    L = _lib.lib()
    fn = L.h2b_cluster_tree_device if device else L.h2b_cluster_tree
    rc = fn(_lib.ptr(boxes), n, int(r_leaf), _lib.ptr(perm), _lib.ptr(nn), _lib.ptr(start), _lib.ptr(end),
            _lib.ptr(depth), _lib.ptr(left), _lib.ptr(right), _lib.ptr(nb))
    _lib.check(rc)
    m = int(nn[0])
    return ClusterTree(perm, start[:m].copy(), end[:m].copy(), depth[:m].copy(), left[:m].copy(),
                       right[:m].copy(), nb[:m].copy())


class Block:
    __slots__ = ("row", "col", "admissible")

    def __init__(self, row, col, adm):
        self.row = row
        self.col = col
        self.admissible = adm

    def __repr__(self):
        return f"Block({self.row!r}, {self.col!r}, {'far' if self.admissible else 'near'})"


class BlockTree:
    """Leaf partition into admissible (far) and leaf-leaf (near) blocks, in
    the reference's depth-first order (clustering.py:137-160).  `far_uids` /
    `near_uids` are the (n, 2) [row uid, col uid] arrays; `.far` / `.near` the
    reference's Block lists (built lazily)."""

    def __init__(self, row_tree, col_tree, eta, device=False):
        """device=True runs the recursion on the GPU (h2b_block_tree_device,
        same lists in the same order)."""
        if eta <= 0.0:
            raise ValueError("eta must be positive")
        self.row_tree = row_tree
        self.col_tree = col_tree
        self.eta = eta
        L = _lib.lib()
        rt, ct = row_tree.c_tree(), col_tree.c_tree()
        nf = np.zeros(1, dtype=np.int64)
        nn = np.zeros(1, dtype=np.int64)
        cap = 1024
        while True:
            far = np.empty((cap, 2), dtype=np.int64)
            near = np.empty((cap, 2), dtype=np.int64)
            fn = L.h2b_block_tree_device if device else L.h2b_block_tree
            rc = fn(ctypes.byref(rt), ctypes.byref(ct), float(eta), _lib.ptr(far), cap, _lib.ptr(near), cap,
                    _lib.ptr(nf), _lib.ptr(nn))
            if rc == _lib.H2B_ERR_CAPACITY:
                cap = int(max(nf[0], nn[0])) + 1
                continue
            _lib.check(rc)
            break
        self.far_uids = far[: int(nf[0])].copy()
        self.near_uids = near[: int(nn[0])].copy()
        self._far = None
        self._near = None

    def _blocks(self, uids, adm):
        rn, cn = self.row_tree.nodes, self.col_tree.nodes
        return [Block(rn[t], cn[s], adm) for t, s in uids]

    @property
    def far(self):
        if self._far is None:
            self._far = self._blocks(self.far_uids, True)
        return self._far

    @property
    def near(self):
        if self._near is None:
            self._near = self._blocks(self.near_uids, False)
        return self._near

    def leaves(self):
        return self.far + self.near

    def check_partition(self):
        """Every (i, j) covered exactly once (vectorised difference-array count)."""
        nr, nc = self.row_tree.n_dofs, self.col_tree.n_dofs
        cover = np.zeros((nr + 1, nc + 1), dtype=np.int32)
        rt, ct = self.row_tree, self.col_tree
        for uids in (self.far_uids, self.near_uids):
            if len(uids) == 0:
                continue
            r0, r1 = rt.start[uids[:, 0]], rt.end[uids[:, 0]]
            c0, c1 = ct.start[uids[:, 1]], ct.end[uids[:, 1]]
            np.add.at(cover, (r0, c0), 1)
            np.add.at(cover, (r0, c1), -1)
            np.add.at(cover, (r1, c0), -1)
            np.add.at(cover, (r1, c1), 1)
        cover = cover.cumsum(0).cumsum(1)[:nr, :nc]
        return bool((cover == 1).all())
