"""Row-sharded multi-GPU H^2 operator (one process per GPU, torch.distributed).

Partition: the row leaves, in permuted (tree) order, are cut
into `world` contiguous ranges balanced by streamed bytes (nearfield rows x
C_t + leaf basis + coupling rows of the leaf).  Rank r owns permuted rows
[lo_r, hi_r), every row leaf inside that range and every row cluster whose
index range intersects it; clusters above the cut (spanning several ranks)
are processed redundantly by each rank that shares them, and each rank's
backward pass only descends into its own subtrees.

Assembly is sharded too (reference work split: containers.py:79-98 nearfield,
gca.py:194-205 couplings): a rank integrates and stores only the near blocks
of its row leaves, the far blocks of its row clusters and the touching pairs
those blocks look up (RowShard.assemble).  Single-layer block pairs are
integrated in the orientation the single-GPU job list uses, so the stored
entries are the same bits as a single-GPU assembly.

Per matvec the only exchange is one all-gather of x (permuted order, padded
to equal chunks) over NCCL; every rank then runs its own task list of the
fused matvec kernel and writes its own rows of y.  No value is reduced across
ranks.  Within a rank the bitwise-symmetric single-layer nearfield is
streamed once per block pair whose two row leaves it owns (the cross-rank
blocks one-sided), so per-rank nearfield bytes are ~1/N of the single-GPU
symmetric stream.  Row results agree with the single-GPU operator to
rounding (the per-row association of the nearfield partials differs); with
the symmetric pairing switched off (H2B_NEAR_SYM=0) sharded and single-GPU
one-sided plans are bitwise identical.

CG on row-sharded vectors: solver.cg(..., allreduce=allreduce_sum(dist)).
"""

import ctypes

import numpy as np

from . import _lib


def leaf_costs(rt, near_C, far_K, ranks):
    """Bytes streamed per row leaf: its nearfield rows and basis V_t, plus an
    even share of the couplings and transfer matrix E of every cluster above it
    (an inner cluster has no V_t and no nearfield; charging its work -- or a
    |t| x k_t basis it does not have -- to its first leaf loaded rank 0 with the
    top of the tree: measured 0.6 vs 1.35 GB per rank at config 3, 8 ranks)."""
    size = rt.end - rt.start
    ranks = np.asarray(ranks, dtype=np.float64)
    leaf = rt.left < 0
    parent = rt.parent_of
    kp = np.where(parent >= 0, ranks[np.maximum(parent, 0)], 0.0)
    own = np.where(leaf, size * np.asarray(near_C, dtype=np.float64) + size * ranks, 0.0)
    shared = ranks * np.asarray(far_K, dtype=np.float64) + ranks * kp
    leaves = rt.leaf_uids()
    order = leaves[np.argsort(rt.start[leaves], kind="stable")]
    # leaves below each node (preorder uids: parents before children)
    nleaf = leaf.astype(np.float64)
    for u in np.argsort(-rt.depth_of, kind="stable"):
        if parent[u] >= 0:
            nleaf[parent[u]] += nleaf[u]
    # top-down: the per-leaf share of every ancestor's (and own) shared cost
    share = shared / np.maximum(nleaf, 1.0)
    acc = np.zeros(rt.n_nodes)
    for u in np.argsort(rt.depth_of, kind="stable"):
        acc[u] = share[u] + (acc[parent[u]] if parent[u] >= 0 else 0.0)
    return order, own[order] + acc[order]


def partition_rows(rt, near_C, far_K, ranks, world):
    """Contiguous permuted row ranges [(lo, hi)] per rank, cut at leaf
    boundaries and balanced by cost (rt: row ClusterTree; near_C / far_K:
    per-node nearfield / coupling matrix widths; ranks: per-node row ranks)."""
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


def block_tree_partition(bt, row_basis, col_basis, world):
    """partition_rows from the block tree and the bases (before assembly)."""
    from .containers import _basis_ranks, far_layout, near_layout

    rr = _basis_ranks(row_basis, bt.row_tree.n_nodes)
    return partition_rows(bt.row_tree, near_layout(bt).C, far_layout(bt, row_basis, col_basis).K, rr, world)


def operator_partition(H, world):
    ranks = np.array([H.row_basis.rank[u] for u in range(H.row_tree.n_nodes)], dtype=np.int64)
    return partition_rows(H.row_tree, H.near_layout.C, H.far_layout.K, ranks, world)


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


class BlockTreeView:
    """The block tree restricted to one rank's rows: the near blocks of its row
    leaves and the far blocks of the row clusters intersecting its range, in
    the full lists' order (near_index / far_index: positions in the full
    lists).  Same trees as the full block tree; usable wherever a BlockTree is
    (layouts, assembly, matvec plans)."""

    def __init__(self, bt, lo, hi):
        rt = bt.row_tree
        self.full = bt
        self.row_tree, self.col_tree, self.eta = bt.row_tree, bt.col_tree, bt.eta
        self.lo, self.hi = lo, hi
        nu, fu = bt.near_uids, bt.far_uids
        leaf_in = (rt.start >= lo) & (rt.end <= hi)
        touches = (rt.start < hi) & (rt.end > lo)
        self.near_index = np.flatnonzero(leaf_in[nu[:, 0]]) if len(nu) else np.zeros(0, dtype=np.int64)
        self.far_index = np.flatnonzero(touches[fu[:, 0]]) if len(fu) else np.zeros(0, dtype=np.int64)
        self.near_uids = nu[self.near_index]
        self.far_uids = fu[self.far_index]
        self._far = self._near = None
        self._near_layout = None

    @property
    def far(self):
        if self._far is None:
            full = self.full.far
            self._far = [full[i] for i in self.far_index]
        return self._far

    @property
    def near(self):
        if self._near is None:
            full = self.full.near
            self._near = [full[i] for i in self.near_index]
        return self._near


class RowShard:
    """One rank's share of a row-sharded H^2 operator: partition, view of the
    block tree, sharded assembly and the rank's matvec plan."""

    def __init__(self, bt, row_basis, col_basis, rank, world, ranges=None):
        if bt.row_tree.n_dofs != bt.col_tree.n_dofs:
            raise ValueError("row sharding with the x all-gather needs a square operator")
        self.bt, self.rb, self.cb = bt, row_basis, col_basis
        self.rank, self.world = rank, world
        self.ranges = ranges if ranges is not None else block_tree_partition(bt, row_basis, col_basis, world)
        self.lo, self.hi = self.ranges[rank]
        self.view = BlockTreeView(bt, self.lo, self.hi)
        rt = bt.row_tree
        self.owned = owned_nodes(rt, self.lo, self.hi)
        self.own_panels = np.zeros(rt.n_dofs, dtype=bool)
        self.own_panels[rt.perm[self.lo : self.hi]] = True
        self.chunk, self.pad_index = gather_layout(self.ranges, rt.n_dofs)
        self.S = self.D = None

    def assemble(self, ctx, kind, q, q_singular=None):
        """Integrate this rank's couplings and nearfield (device)."""
        from .containers import assemble_couplings, assemble_nearfield_sharded

        self.S = assemble_couplings(ctx, kind, self.view, self.rb, self.cb, q)
        self.D = assemble_nearfield_sharded(ctx, kind, self.view, q, q_singular, self.own_panels)
        return self.S, self.D

    def near_entries(self):
        from .containers import near_layout

        return near_layout(self.view).entries

    def plan(self, xhat_mask=None):
        from .containers import MatvecPlan, far_layout, near_layout

        rt = self.bt.row_tree
        row_local = np.arange(rt.n_dofs, dtype=np.int64) - self.lo  # only owned rows are written
        return MatvecPlan(self.view, self.rb, self.cb, self.S, self.D, far_layout(self.view, self.rb, self.cb),
                          near_layout(self.view), owned=self.owned, col_perm=self.pad_index, row_perm=row_local,
                          xhat_mask=xhat_mask)


class LocalMatvec:
    """Single-GPU matvec on device tensors (natural order)."""

    def __init__(self, H):
        self.H = H
        self.plan = H.plan()

    def apply(self, x, y):
        self.plan.apply_device(x, y)
        return y


def xhat_exchange_layout(tree, ranks, ranges):
    """The x_hat exchange of SURVEY 8(e)'s better variant: rank r owns the
    column clusters inside its permuted range [lo_r, hi_r) and computes their
    coefficients; every rank's owned coefficients (uid order) fill one chunk
    of the gathered buffer.  Returns (masks (world, n_nodes) int8, chunk,
    src (n_nodes,) offset of each cluster in the gathered buffer, -1 for the
    clusters spanning several ranks)."""
    world = len(ranges)
    n = tree.n_nodes
    masks = np.zeros((world, n), dtype=np.int8)
    src = np.full(n, -1, dtype=np.int64)
    sizes = []
    for r, (lo, hi) in enumerate(ranges):
        m = (tree.start >= lo) & (tree.end <= hi) & (tree.end > tree.start)
        masks[r] = m
        sizes.append(int(np.asarray(ranks, dtype=np.int64)[m].sum()))
    chunk = max(max(sizes), 1)
    for r in range(world):
        u = np.flatnonzero(masks[r])
        k = np.asarray(ranks, dtype=np.int64)[u]
        src[u] = r * chunk + np.cumsum(k) - k
    return masks, chunk, src


class NativeComm:
    """An NCCL communicator owned by libh2b (h2b_comm_init): a sharded plan
    with it attached runs its x all-gather inside h2b_matvec_sharded, so the
    whole sharded matvec is one C-ABI call.  Rank 0 draws the unique id;
    `dist` (torch.distributed, any backend) broadcasts it when world > 1."""

    def __init__(self, rank, world, device=0, dist=None):
        L = _lib.lib()
        uid = (ctypes.c_char * 128)()
        if rank == 0:
            _lib.check(L.h2b_comm_unique_id(uid))
        if world > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0)
            ctypes.memmove(uid, box[0], 128)
        self.handle = ctypes.c_void_p()
        _lib.check(L.h2b_comm_init(ctypes.byref(self.handle), world, uid, rank, device))
        self.rank, self.world = rank, world

    def close(self):
        if self.handle:
            _lib.check(_lib.lib().h2b_comm_destroy(self.handle))
            self.handle = ctypes.c_void_p()


class ShardedMatvec:
    """Row-sharded matvec of one rank.  apply_local(x_loc, y_loc) takes this
    rank's permuted slice of x and returns its permuted rows of y (the CG
    path); apply(x, y) takes a full natural-order x and scatters the rank's
    rows into y (bench / tests).  `dist` provides all_gather_into_tensor.

    Built either from a RowShard (sharded assembly: the rank holds only its
    share of the operator) or, for tests, from a full single-GPU H2Matrix."""

    def __init__(self, src, rank, world, dist, comm=None, xhat=False):
        """xhat=True: the x_hat exchange variant: the rank's
        forward transform covers only its own column subtrees, the
        coefficients are all-gathered (second collective) and the clusters
        spanning several ranks are climbed on every rank."""
        import torch

        if isinstance(src, RowShard):
            shard = src
            if shard.S is None:
                raise ValueError("RowShard.assemble() first")
        else:
            H = src
            shard = RowShard(H.block_tree, H.row_basis, H.col_basis, rank, world,
                             ranges=operator_partition(H, world))
            shard.view = H.block_tree  # full operator arrays: every block present
            shard.S, shard.D = H.S_dev, H.D_dev
        self.shard, self.rank, self.world, self.dist = shard, rank, world, dist
        self.lo, self.hi, self.chunk = shard.lo, shard.hi, shard.chunk
        self.xhat = xhat
        xmask = None
        if xhat:
            from .containers import _basis_ranks

            ct = shard.bt.col_tree
            masks, self.xchunk, xsrc = xhat_exchange_layout(ct, _basis_ranks(shard.cb, ct.n_nodes), shard.ranges)
            xmask = masks[rank]
        if shard.view is shard.bt:
            from .containers import MatvecPlan

            rt = shard.bt.row_tree
            H = src
            self.plan = MatvecPlan(H.block_tree, H.row_basis, H.col_basis, H.S_dev, H.D_dev, H.far_layout,
                                   H.near_layout, owned=shard.owned, col_perm=shard.pad_index,
                                   row_perm=np.arange(rt.n_dofs, dtype=np.int64) - shard.lo, xhat_mask=xmask)
        else:
            self.plan = shard.plan(xhat_mask=xmask)
        if xhat:
            _lib.check(_lib.lib().h2b_xhat_set_import(self.plan.handle, _lib.ptr(np.ascontiguousarray(xsrc))))
            self.xsend = torch.zeros(self.xchunk, dtype=torch.float64, device="cuda")
            self.xrecv = torch.zeros(world * self.xchunk, dtype=torch.float64, device="cuda")
        rt = shard.bt.row_tree
        self.xbuf = torch.zeros(world * self.chunk, dtype=torch.float64, device="cuda")
        self.xloc = torch.zeros(self.chunk, dtype=torch.float64, device="cuda")
        self.yloc = torch.zeros(max(self.hi - self.lo, 1), dtype=torch.float64, device="cuda")
        self.perm_dev = torch.from_numpy(rt.perm[self.lo : self.hi].copy()).cuda()
        self.comm = comm
        if comm is not None:
            _lib.check(_lib.lib().h2b_plan_set_comm(self.plan.handle, comm.handle, rank, world, self.chunk))

    def info(self):
        return self.plan.info()

    def apply_local(self, x_local_perm, y_local_perm=None):
        """x_local_perm: this rank's permuted slice of x (hi - lo); returns its rows of y."""
        n = self.hi - self.lo
        if y_local_perm is None:
            y_local_perm = self.yloc[:n].clone()
        self.xloc[:n].copy_(x_local_perm)
        self._gather_apply(y_local_perm)
        return y_local_perm

    def _gather_apply(self, y):
        if self.xhat:
            L, st = _lib.lib(), _lib.stream_ptr()
            self.dist.all_gather_into_tensor(self.xbuf, self.xloc)
            _lib.check(L.h2b_xhat_forward(self.plan.handle, self.xbuf.data_ptr(), self.xsend.data_ptr(), st))
            self.dist.all_gather_into_tensor(self.xrecv, self.xsend)
            _lib.check(L.h2b_xhat_main(self.plan.handle, self.xbuf.data_ptr(), self.xrecv.data_ptr(), y.data_ptr(),
                                       st))
            return
        if self.comm is not None:
            # all-gather (NCCL) + fused matvec in one C-ABI call
            _lib.check(_lib.lib().h2b_matvec_sharded(self.plan.handle, self.xloc.data_ptr(), y.data_ptr(),
                                                     _lib.stream_ptr()))
        else:
            self.dist.all_gather_into_tensor(self.xbuf, self.xloc)
            _lib.check(_lib.lib().h2b_matvec(self.plan.handle, self.xbuf.data_ptr(), y.data_ptr(),
                                             _lib.stream_ptr()))

    def apply(self, x, y):
        """Full natural-order x -> this rank's rows written into y[perm]."""
        n = self.hi - self.lo
        self.xloc[:n].copy_(x[self.perm_dev])
        self._gather_apply(self.yloc)
        y[self.perm_dev] = self.yloc[:n]
        return y

    def diagonal_local(self):
        """This rank's rows of the operator diagonal (permuted order)."""
        import torch

        d = torch.zeros(max(self.hi - self.lo, 1), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().h2b_diagonal(self.plan.handle, d.data_ptr(), _lib.stream_ptr()))
        return d[: self.hi - self.lo]


class ShardedOperator:
    """The reference's operator interface (matvec / diagonal on full
    natural-order vectors, containers.py:254-301) over a row-sharded operator:
    what ProblemSetup.operator returns when RunParams.devices > 1.  Every rank
    passes the same x and receives the full y (its own rows computed here, the
    others summed in by one all-reduce); solvers that keep their vectors
    sharded use `.sharded` (ShardedMatvec.apply_local) directly."""

    def __init__(self, sharded):
        self.sharded = sharded
        n = sharded.shard.bt.row_tree.n_dofs
        self.shape = (n, n)

    def _full(self, fill):
        import torch

        mv = self.sharded
        y = torch.zeros(self.shape[0], dtype=torch.float64, device="cuda")
        fill(y)
        if mv.world > 1:
            mv.dist.all_reduce(y, op=mv.dist.ReduceOp.SUM)
        return y

    def matvec(self, x):
        import torch

        from . import device as D

        dev_in = isinstance(x, torch.Tensor)
        xd = x if dev_in else D.dev(np.ascontiguousarray(x, dtype=np.float64))
        if xd.dtype != torch.float64 or xd.ndim != 1 or xd.numel() != self.shape[1]:
            raise ValueError(f"expected a float64 vector of length {self.shape[1]}")
        y = self._full(lambda y: self.sharded.apply(xd, y))
        return y if dev_in else D.host(y)

    def diagonal(self):
        from . import device as D

        mv = self.sharded

        def fill(y):
            y[mv.perm_dev] = mv.diagonal_local()

        return D.host(self._full(fill))


def allreduce_sum(dist, group=None):
    """In-place sum of a small device tensor over the ranks (CG scalars)."""

    def f(t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)

    return f
