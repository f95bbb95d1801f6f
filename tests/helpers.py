"""Shared builders for the test-suite (configs of BASELINE.json at test sizes)."""

import numpy as np

from paper_2001_05523_b200 import clustering as C
from paper_2001_05523_b200 import mesh as M
from paper_2001_05523_b200 import spaces as S
from paper_2001_05523_b200.containers import ClusterBasis

from oracle import h2 as OH

# name: (sphere level, leaf, eta, m, q_reg, q_ss)
CONFIGS = {
    "cfg0": (4, 32, 2.0, 3, 3, 4),
    "cfg1": (6, 64, 2.0, 4, 3, 4),
    "dlp4": (4, 32, 2.0, 3, 3, 5),
}


def trees(mesh, leaf):
    t0 = C.build_cluster_tree(S.DofSpace(S.P0, mesh).support_boxes(), leaf)
    t1 = C.build_cluster_tree(S.DofSpace(S.P1, mesh).support_boxes(), leaf)
    return t0, t1


def basis_from_arrays(tree, ranks, pivots, V, E):
    """ClusterBasis from the flat golden arrays (uid order; V over leaves in
    uid order, E over non-root nodes in uid order)."""
    b = ClusterBasis(tree)
    off = np.concatenate([[0], np.cumsum(ranks)])
    vo = eo = 0
    for u in range(tree.n_nodes):
        k = int(ranks[u])
        b.rank[u] = k
        b.pivots[u] = pivots[off[u] : off[u + 1]]
        if tree.left[u] < 0:
            n = int(tree.end[u] - tree.start[u])
            b.V[u] = V[vo : vo + n * k].reshape(n, k)
            vo += n * k
    for u in range(tree.n_nodes):
        p = tree.parent_of[u]
        if p >= 0:
            k, kp = int(ranks[u]), int(ranks[p])
            b.E[u] = E[eo : eo + k * kp].reshape(k, kp)
            eo += k * kp
    assert vo == len(V) and eo == len(E)
    return b


def oracle_tree(t):
    return OH.Tree(t.perm, t.start, t.end, t.depth_of, t.left, t.right)


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))


def sphere(level):
    return M.sphere_mesh(level)
