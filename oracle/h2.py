"""H^2 matvec over explicit operator data, restated (oracle; test infra only).

Reference: /root/reference/pkg/src/h2bem/containers.py
  ClusterBasis.forward   :201-212  leaves V^T x, parents sum_ch E_ch^T xhat_ch
  ClusterBasis.backward  :214-228  top-down yhat_ch += E_ch yhat_t, leaves y += V yhat
  H2Matrix.matvec        :254-270  permute, forward, couplings, backward, nearfield, un-permute
  H2Matrix.rmatvec       :272-288  the same with the roles of the trees/bases swapped, S^T, D^T
  H2Matrix.diagonal      :290-301
"""

import numpy as np


class Tree:
    """Flat cluster tree: perm, start, end, depth, left, right (uid-indexed)."""

    def __init__(self, perm, start, end, depth, left, right):
        self.perm, self.start, self.end, self.depth, self.left, self.right = perm, start, end, depth, left, right

    def bottom_up(self):
        return np.argsort(-np.asarray(self.depth), kind="stable")


def forward(tree, V, E, rank, xp):
    """containers.py:201-212."""
    xhat = {}
    for u in tree.bottom_up():
        u = int(u)
        if tree.left[u] < 0:
            xhat[u] = V[u].T @ xp[tree.start[u] : tree.end[u]]
        else:
            acc = np.zeros(rank[u])
            for ch in (int(tree.left[u]), int(tree.right[u])):
                acc += E[ch].T @ xhat[ch]
            xhat[u] = acc
    return xhat


def backward(tree, V, E, yhat, yp):
    """containers.py:214-228."""
    for u in tree.bottom_up()[::-1]:
        u = int(u)
        v = yhat.get(u)
        if v is None:
            continue
        if tree.left[u] < 0:
            yp[tree.start[u] : tree.end[u]] += V[u] @ v
        else:
            for ch in (int(tree.left[u]), int(tree.right[u])):
                c = E[ch] @ v
                yhat[ch] = yhat[ch] + c if ch in yhat else c


def matvec(row_tree, col_tree, rV, rE, rrank, cV, cE, crank, far, S, near, Dn, x):
    """y = A x in natural order.  far/near: (n, 2) [row uid, col uid] lists in
    block-tree order; S / Dn: matching lists of dense payloads."""
    xp = np.asarray(x, dtype=float)[col_tree.perm]
    yp = np.zeros(len(row_tree.perm))
    xhat = forward(col_tree, cV, cE, crank, xp)
    yhat = {}
    for (t, s), Sb in zip(far, S):
        c = Sb @ xhat[int(s)]
        yhat[int(t)] = yhat[int(t)] + c if int(t) in yhat else c
    backward(row_tree, rV, rE, yhat, yp)
    for (t, s), Db in zip(near, Dn):
        yp[row_tree.start[t] : row_tree.end[t]] += Db @ xp[col_tree.start[s] : col_tree.end[s]]
    y = np.empty_like(yp)
    y[row_tree.perm] = yp
    return y


def rmatvec(row_tree, col_tree, rV, rE, rrank, cV, cE, crank, far, S, near, Dn, x):
    """y = A^T x (containers.py:272-288): forward over the ROW basis, S_b^T
    into the column clusters, backward over the COLUMN basis, D_b^T."""
    xp = np.asarray(x, dtype=float)[row_tree.perm]
    yp = np.zeros(len(col_tree.perm))
    xhat = forward(row_tree, rV, rE, rrank, xp)
    yhat = {}
    for (t, s), Sb in zip(far, S):
        c = Sb.T @ xhat[int(t)]
        yhat[int(s)] = yhat[int(s)] + c if int(s) in yhat else c
    backward(col_tree, cV, cE, yhat, yp)
    for (t, s), Db in zip(near, Dn):
        yp[col_tree.start[s] : col_tree.end[s]] += Db.T @ xp[row_tree.start[t] : row_tree.end[t]]
    y = np.empty_like(yp)
    y[col_tree.perm] = yp
    return y


def diagonal(row_tree, col_tree, near, Dn):
    """containers.py:290-301."""
    dp = np.zeros(len(row_tree.perm))
    for (t, s), Db in zip(near, Dn):
        lo = max(row_tree.start[t], col_tree.start[s])
        hi = min(row_tree.end[t], col_tree.end[s])
        if hi > lo:
            idx = np.arange(lo, hi)
            dp[idx] += Db[idx - row_tree.start[t], idx - col_tree.start[s]]
    out = np.empty_like(dp)
    out[row_tree.perm] = dp
    return out


class RowSlice:
    """The H^2 matvec (containers.py:254-270) restricted to the rows of one
    cluster subtree (`root`), over explicit operator data: bench.py's
    reference arm times the reference algorithm on bounded row slices of the
    full configuration.  The slice holds every block a full matvec applies to
    its rows: the far blocks of its clusters and of their ancestors (their
    coefficients reach the slice through the downward pass), the near blocks
    of its leaves, and the forward transform of every column cluster those
    far blocks read (the subtree closure).  The per-block work is the
    reference's: one numpy product per block, clusters bottom-up / top-down.

    far / near: (n, 2) [row uid, col uid] block lists of the whole operator;
    values: callables giving the dense payloads (shape-exact)."""

    def __init__(self, tree, root, far, near, rank, V, E, S, Dn):
        n = tree.n_nodes if hasattr(tree, "n_nodes") else len(tree.start)
        start, end = np.asarray(tree.start), np.asarray(tree.end)
        left, right = np.asarray(tree.left), np.asarray(tree.right)
        self.tree, self.root = tree, root
        sub = (start >= start[root]) & (end <= end[root])
        anc = np.zeros(n, dtype=bool)
        parent = np.full(n, -1, dtype=np.int64)
        inner = np.flatnonzero(left >= 0)
        parent[left[inner]] = inner
        parent[right[inner]] = inner
        p = int(parent[root])
        while p >= 0:
            anc[p] = True
            p = int(parent[p])
        rows = sub | anc
        fsel = np.flatnonzero(rows[far[:, 0]])
        nsel = np.flatnonzero(sub[near[:, 0]] & (left[near[:, 0]] < 0))
        self.far = far[fsel]
        self.near = near[nsel]
        self.S = [S(i) for i in fsel]
        self.D = [Dn(i) for i in nsel]
        # forward closure: the column clusters read by the far blocks and their subtrees
        need = np.zeros(n, dtype=bool)
        need[self.far[:, 1]] = True
        for u in np.argsort(np.asarray(tree.depth), kind="stable"):
            if parent[u] >= 0 and need[parent[u]]:
                need[u] = True
        self.fwd = [int(u) for u in np.argsort(-np.asarray(tree.depth), kind="stable") if need[u]]
        self.down = [int(u) for u in np.argsort(np.asarray(tree.depth), kind="stable") if rows[u]]
        self.rows = rows
        self.rank = rank
        used = need | rows
        self.V = {u: V(u) for u in np.flatnonzero(used & (left < 0))}
        self.E = {u: E(u) for u in np.flatnonzero(used & (parent >= 0))}
        self.n_rows = int(end[root] - start[root])

    def matvec(self, x):
        """The slice's rows of y = A x (permuted order)."""
        t = self.tree
        xp = np.asarray(x, dtype=float)[t.perm]
        xhat = {}
        for u in self.fwd:
            if t.left[u] < 0:
                xhat[u] = self.V[u].T @ xp[t.start[u] : t.end[u]]
            else:
                acc = np.zeros(self.rank[u])
                for ch in (int(t.left[u]), int(t.right[u])):
                    acc += self.E[ch].T @ xhat[ch]
                xhat[u] = acc
        yhat = {}
        for (a, b), Sb in zip(self.far, self.S):
            c = Sb @ xhat[int(b)]
            yhat[int(a)] = yhat[int(a)] + c if int(a) in yhat else c
        r0 = t.start[self.root]
        yp = np.zeros(self.n_rows)
        for u in self.down:
            v = yhat.get(u)
            if v is None:
                continue
            if t.left[u] < 0:
                yp[t.start[u] - r0 : t.end[u] - r0] += self.V[u] @ v
            else:
                for ch in (int(t.left[u]), int(t.right[u])):
                    if self.rows[ch]:
                        c = self.E[ch] @ v
                        yhat[ch] = yhat[ch] + c if ch in yhat else c
        for (a, b), Db in zip(self.near, self.D):
            yp[t.start[a] - r0 : t.end[a] - r0] += Db @ xp[t.start[b] : t.end[b]]
        return yp
