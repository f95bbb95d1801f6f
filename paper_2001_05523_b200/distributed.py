"""Row-sharded multi-GPU H^2 matvec (one process per GPU, torch.distributed).

Partition: the row leaves, in permuted (tree) order, are cut
into `world` contiguous ranges balanced by streamed bytes (nearfield rows x
C_t + leaf basis + coupling rows of the leaf).  Rank r owns permuted rows
[lo_r, hi_r) and every row cluster whose index range intersects it; clusters
above the cut are evaluated redundantly by each rank that shares them, and
each rank's backward pass only descends into its own subtrees.  No value is
reduced across ranks: each rank writes its own rows of y.

Per matvec the only exchange is one all-gather of x (permuted order, padded
to equal chunks) over NCCL; every rank then runs the full forward transform
(the column tree is needed by all coupling blocks) and its share of the
backward/nearfield work.  Row accumulation order does not depend on the rank
count, so 1- and N-GPU results are bitwise identical.
"""

import numpy as np

from . import _lib


def leaf_costs(rt, near_C, far_K, ranks):
    """Bytes streamed per row leaf (nearfield rows + leaf basis + the leaf's
    couplings); an inner cluster's coupling work is charged to its first leaf."""
    size = rt.end - rt.start
    cost = size * near_C + size * ranks + ranks * far_K
    leaves = rt.leaf_uids()
    order = leaves[np.argsort(rt.start[leaves], kind="stable")]
    # charge each internal node's coupling to the leaf at its start
    first_leaf = {}
    for u in order:
        first_leaf[int(rt.start[u])] = int(u)
    lc = {int(u): float(cost[u]) for u in order}
    for u in np.flatnonzero(rt.left >= 0):
        lc[first_leaf[int(rt.start[u])]] += float(cost[u])
    return order, np.array([lc[int(u)] for u in order])


def partition_rows(rt, near_C, far_K, ranks, world):
    """Contiguous permuted row ranges [(lo, hi)] per rank, balanced by cost
    (rt: row ClusterTree; near_C / far_K: per-node nearfield / coupling
    matrix widths; ranks: per-node row-basis ranks)."""
    order, cost = leaf_costs(rt, near_C, far_K, ranks)
    cum = np.cumsum(cost)
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        i = int(np.searchsorted(cum, target))
        i = min(max(i, bounds[-1] + 1), len(order) - (world - r))
        bounds.append(i)
    bounds.append(len(order))
    ranges = []
    for r in range(world):
        a, b = bounds[r], bounds[r + 1]
        lo = int(rt.start[order[a]]) if a < len(order) else int(rt.n_dofs)
        hi = int(rt.end[order[b - 1]]) if b > a else lo
        ranges.append((lo, hi))
    return ranges


def owned_nodes(tree, lo, hi):
    """Row clusters whose range intersects [lo, hi), parents first (by depth)."""
    hit = np.flatnonzero((tree.start < hi) & (tree.end > lo))
    return hit[np.argsort(tree.depth_of[hit], kind="stable")]


def gather_layout(ranges, n):
    """Equal-size all-gather chunks: (chunk, pad_index) with pad_index[p] the
    position of permuted dof p in the gathered buffer of world * chunk."""
    chunk = max(max(h - l for l, h in ranges), 1)
    pad_index = np.empty(n, dtype=np.int64)
    for r, (a, b) in enumerate(ranges):
        pad_index[a:b] = r * chunk + np.arange(b - a)
    return chunk, pad_index


def operator_partition(H, world):
    ranks = np.array([H.row_basis.rank[u] for u in range(H.row_tree.n_nodes)], dtype=np.int64)
    return partition_rows(H.row_tree, H.near_layout.C, H.far_layout.K, ranks, world)


class LocalMatvec:
    """Single-GPU matvec on device tensors (natural order)."""

    def __init__(self, H):
        self.H = H
        self.plan = H.plan()

    def apply(self, x, y):
        self.plan.apply_device(x, y)
        return y



class ShardedMatvec:
    """Row-sharded matvec: apply(x, y) takes the full natural-order x on every
    rank (the bench's input) or, via apply_local, this rank's permuted slice."""

    def __init__(self, H, rank, world, dist):
        import torch

        from .containers import MatvecPlan

        if H.shape[0] != H.shape[1]:
            raise ValueError("row sharding with the x all-gather needs a square operator")
        self.H, self.rank, self.world, self.dist = H, rank, world, dist
        rt = H.row_tree
        self.ranges = operator_partition(H, world)
        lo, hi = self.ranges[rank]
        self.lo, self.hi = lo, hi
        # padded gather layout: permuted position p of rank r -> r*chunk + (p - lo_r)
        self.chunk, pad_index = gather_layout(self.ranges, rt.n_dofs)
        row_local = np.arange(rt.n_dofs, dtype=np.int64) - lo  # only owned rows are written
        owned = owned_nodes(rt, lo, hi)
        self.plan = MatvecPlan(H.block_tree, H.row_basis, H.col_basis, H.S_dev, H.D_dev, H.far_layout,
                               H.near_layout, owned=owned, col_perm=pad_index, row_perm=row_local)
        self.xbuf = torch.zeros(world * self.chunk, dtype=torch.float64, device="cuda")
        self.xloc = torch.zeros(self.chunk, dtype=torch.float64, device="cuda")
        self.yloc = torch.zeros(max(hi - lo, 1), dtype=torch.float64, device="cuda")
        self.perm_dev = torch.from_numpy(rt.perm[lo:hi].copy()).cuda()

    def apply_local(self, x_local_perm, y_local_perm):
        """x_local_perm: this rank's permuted slice of x (hi-lo); returns its rows of y."""
        n = self.hi - self.lo
        self.xloc[:n].copy_(x_local_perm)
        self.dist.all_gather_into_tensor(self.xbuf, self.xloc)
        _lib.check(_lib.lib().h2b_matvec(self.plan.handle, self.xbuf.data_ptr(), y_local_perm.data_ptr(),
                                         _lib.stream_ptr()))
        return y_local_perm

    def apply(self, x, y):
        """Bench entry: full natural-order x -> this rank's rows written into y[perm]."""
        n = self.hi - self.lo
        self.xloc[:n].copy_(x[self.perm_dev])
        self.dist.all_gather_into_tensor(self.xbuf, self.xloc)
        _lib.check(_lib.lib().h2b_matvec(self.plan.handle, self.xbuf.data_ptr(), self.yloc.data_ptr(),
                                         _lib.stream_ptr()))
        y[self.perm_dev] = self.yloc[:n]
        return y
