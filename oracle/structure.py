"""Mesh, support boxes, cluster tree and block tree, restated in numpy (oracle;
test infrastructure only -- and the structure of bench.py's reference arm,
which must not import the product).

Reference: /root/reference/pkg/src/h2bem/
  mesh.build_octahedron / refine_red / project_unit_sphere / sphere_mesh  mesh.py:90-154
  SurfaceMesh normals and areas                                           mesh.py:19-37
  spaces.DofSpace.support_boxes (P0)                                      spaces.py:29-41
  clustering.build_cluster_tree                                           clustering.py:78-121
  clustering.box_diameter / box_distance / admissible                     clustering.py:7-21
  clustering.BlockTree._descend                                           clustering.py:149-160

Bit-exact by construction where the reference is: refinement numbers new
vertices in first-use order over (triangle, edge ij/jk/ki) and forms
midpoints as 0.5 (v_a + v_b); projection and normals use np.linalg.norm
along axis 1 (sqrt((a a + b b) + c c)); admissibility calls np.linalg.norm
on the 3-vectors exactly as the reference does (the host BLAS ddot).
Pinned by tests/test_oracle_structure.py against the reference's own trees,
block lists and mesh digests (tests/golden/struct_*.npz, mesh*.json/npz).
"""

import numpy as np

OCTA_V = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, -1.0, 0.0], [0.0, 0.0, 1.0],
                   [0.0, 0.0, -1.0]])
OCTA_T = np.array([[0, 2, 4], [2, 1, 4], [1, 3, 4], [3, 0, 4], [2, 0, 5], [1, 2, 5], [3, 1, 5], [0, 3, 5]],
                  dtype=np.int64)


def normals_areas(V, T):
    """mesh.py:31-37: cross product of the edge vectors, its norm -> unit
    normal and half the norm as the area."""
    cross = np.cross(V[T[:, 1]] - V[T[:, 0]], V[T[:, 2]] - V[T[:, 0]])
    nrm = np.linalg.norm(cross, axis=1)
    return cross / nrm[:, None], 0.5 * nrm


def refine(V, T):
    """mesh.py:117-135: red refinement with first-use midpoint numbering."""
    nV = len(V)
    a = T[:, [0, 1, 2]].reshape(-1)       # edge (i, j), (j, k), (k, i) per triangle, in order
    b = T[:, [1, 2, 0]].reshape(-1)
    key = np.minimum(a, b) * nV + np.maximum(a, b)
    uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")            # unique edges by first use
    new_id = np.empty(len(uniq), dtype=np.int64)
    new_id[order] = nV + np.arange(len(uniq))
    mid = new_id[inv].reshape(-1, 3)                     # ij, jk, ki per triangle
    fa, fb = a[first[order]], b[first[order]]            # endpoints as first used
    Vn = np.vstack([V, 0.5 * (V[fa] + V[fb])])
    i, j, k = T[:, 0], T[:, 1], T[:, 2]
    ij, jk, ki = mid[:, 0], mid[:, 1], mid[:, 2]
    Tn = np.stack([np.stack([i, ij, ki], 1), np.stack([ij, j, jk], 1), np.stack([ki, jk, k], 1),
                   np.stack([ij, jk, ki], 1)], axis=1).reshape(-1, 3)
    return Vn, Tn


def sphere(level):
    """mesh.py:146-154: (vertices, triangles, normals, areas)."""
    V, T = OCTA_V.copy(), OCTA_T.copy()
    for _ in range(level):
        V, T = refine(V, T)
        V = V / np.linalg.norm(V, axis=1)[:, None]
    N, A = normals_areas(V, T)
    return V, T, N, A


def p0_boxes(V, T):
    """spaces.py:29-41 (P0): per-triangle [min; max] of its corners."""
    c = V[T]
    return np.stack([c.min(axis=1), c.max(axis=1)], axis=1)


class Tree:
    """Flat cluster tree (uid = preorder creation index)."""

    def __init__(self, perm, start, end, depth, left, right, boxes):
        self.perm, self.start, self.end, self.depth = perm, start, end, depth
        self.left, self.right, self.boxes = left, right, boxes
        n = len(start)
        self.parent = np.full(n, -1, dtype=np.int64)
        inner = np.flatnonzero(left >= 0)
        self.parent[left[inner]] = inner
        self.parent[right[inner]] = inner

    @property
    def n_nodes(self):
        return len(self.start)

    def bottom_up(self):
        return np.argsort(-self.depth, kind="stable")


def cluster_tree(boxes, r_leaf):
    """clustering.py:78-121: longest box axis, split at the midpoint of the
    dof centres (c <= mid goes left, input order kept), stable-argsort median
    fallback when one side would be empty, leaves of <= r_leaf dofs; perm
    filled at the leaves left to right."""
    boxes = np.asarray(boxes, dtype=float)
    n = len(boxes)
    centers = 0.5 * (boxes[:, 0, :] + boxes[:, 1, :])
    perm = np.empty(n, dtype=np.int64)
    start, end, depth, left, right, nb = [], [], [], [], [], []
    stack = [(np.arange(n, dtype=np.int64), 0, 0, -1, 0)]  # ids, start, depth, parent, which child
    while stack:
        ids, st, dp, par, side = stack.pop()
        u = len(start)
        box = np.stack([boxes[ids, 0, :].min(axis=0), boxes[ids, 1, :].max(axis=0)])
        start.append(st)
        end.append(st + len(ids))
        depth.append(dp)
        left.append(-1)
        right.append(-1)
        nb.append(box)
        if par >= 0:
            (left if side == 0 else right)[par] = u
        if len(ids) <= r_leaf:
            perm[st : st + len(ids)] = ids
            continue
        axis = int(np.argmax(box[1] - box[0]))
        c = centers[ids, axis]
        mid = 0.5 * (c.min() + c.max())
        mask = c <= mid
        if mask.all() or not mask.any():
            order = np.argsort(c, kind="stable")
            mask = np.zeros(len(ids), dtype=bool)
            mask[order[: len(ids) // 2]] = True
        lft, rgt = ids[mask], ids[~mask]
        # preorder: the left subtree is created before the right one
        stack.append((rgt, st + len(lft), dp + 1, u, 1))
        stack.append((lft, st, dp + 1, u, 0))
    a = lambda x: np.asarray(x, dtype=np.int64)  # noqa: E731
    return Tree(perm, a(start), a(end), a(depth), a(left), a(right), np.asarray(nb))


def block_tree(row, col, eta, row_keep=None):
    """clustering.py:149-160 in the reference's depth-first order: admissible
    pairs are far blocks, leaf x leaf pairs near blocks, otherwise the
    children product (a leaf side kept as itself).  row_keep (bool per row
    uid, optional): descend only into pairs whose row cluster is kept (a row
    slice and its ancestors); the lists are then the reference's lists
    filtered to those rows, in the same order.  Returns (far, near) arrays
    (n, 2) of [row uid, col uid]."""
    if eta <= 0.0:
        raise ValueError("eta must be positive")
    diam_r = [float(np.linalg.norm(b[1] - b[0])) for b in row.boxes]
    diam_c = diam_r if col is row else [float(np.linalg.norm(b[1] - b[0])) for b in col.boxes]
    far, near = [], []
    stack = [(0, 0)]
    while stack:
        t, s = stack.pop()
        if row_keep is not None and not row_keep[t]:
            continue
        bt, bs = row.boxes[t], col.boxes[s]
        gaps = np.maximum(0.0, np.maximum(bt[0] - bs[1], bs[0] - bt[1]))
        if max(diam_r[t], diam_c[s]) <= 2.0 * eta * float(np.linalg.norm(gaps)):
            far.append((t, s))
            continue
        tl, sl = row.left[t] < 0, col.left[s] < 0
        if tl and sl:
            near.append((t, s))
            continue
        ts = [t] if tl else [int(row.left[t]), int(row.right[t])]
        ss = [s] if sl else [int(col.left[s]), int(col.right[s])]
        for tc in reversed(ts):
            for sc in reversed(ss):
                stack.append((tc, sc))
    f = np.array(far, dtype=np.int64).reshape(-1, 2)
    nr = np.array(near, dtype=np.int64).reshape(-1, 2)
    return f, nr
