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
