"""Operators and containers.  API of h2bem.containers (containers.py:1-328).

Device layout (HBM) of an H^2 operator, built once from the block tree and
the bases:

  D  nearfield, one row-major |t| x C_t matrix per row leaf t whose columns are
     its near blocks side by side (near-list order), C_t padded to a multiple of 4
     so rows start 32-byte aligned (256-bit loads);
  S  couplings, one row-major k_t x K_t matrix per row cluster t, far blocks
     side by side (far-list order), K_t padded to a multiple of 4;
  V  leaf bases |t| x k_t, E transfer matrices k_child x k_parent (row-major).

The matvec streams D and S row by row (libh2b k_backward) and V/E once each
way; per-block numpy views for the reference API (`.near`, `.far`) are cut
from host copies on demand.
"""

import ctypes

import numpy as np

from . import _lib
from . import device as D
from . import kernels
from . import quadrature as quad

ORACLE_CAP = 4096


class AssemblyContext:
    """Per-mesh caches: device mesh, regular panel points per order, touching
    table and singular integrals per (kind, order) (containers.py:14-45)."""

    def __init__(self, mesh):
        self.mesh = mesh
        self._dmesh = None
        self._host_pq = {}
        self._singular = {}

    @property
    def dmesh(self):
        if self._dmesh is None:
            self._dmesh = kernels.device_mesh(self.mesh)
        return self._dmesh

    @property
    def vertex_tris(self):
        return self.mesh.vertex_triangles()

    @property
    def curls(self):
        """Per-panel surface curls of the P1 hats (kernels.triangle_curls)."""
        if getattr(self, "_curls", None) is None:
            self._curls = kernels.triangle_curls(self.mesh)
        return self._curls

    def host_panel_quad(self, q):
        """Host panel points (GCA Green columns); reference: panel_quad(q)."""
        if q not in self._host_pq:
            self._host_pq[q] = quad.triangle_points(self.mesh, np.arange(self.mesh.n_triangles), q)
        return self._host_pq[q]

    panel_quad = host_panel_quad

    def singular_table(self, kind, q):
        kind = kernels.SLP if kind == kernels.HYP else kind
        key = (kind, q)
        if key not in self._singular:
            self._singular[key] = kernels.SingularTable(self.dmesh, kind, q)
        return self._singular[key]

    def incident_panels(self, verts):
        ptr, idx = self.mesh.vertex_triangle_csr()
        verts = np.asarray(verts, dtype=np.int64)
        if len(verts) == 0:
            return np.empty(0, dtype=np.int64)
        return np.unique(np.concatenate([idx[ptr[v] : ptr[v + 1]] for v in verts]))


def _blocks_to_device(ctx, kind, blocks, q, q_singular, require_disjoint, out, table=None):
    """Run (row dofs, col dofs, out_off, ld) dense blocks through the kernels."""
    if table is None and not require_disjoint:
        table = ctx.singular_table(kind, q_singular)
    if kind == kernels.SLP:
        ri = np.concatenate([np.asarray(b[0], dtype=np.int64) for b in blocks]) if blocks else np.zeros(0)
        ci = np.concatenate([np.asarray(b[1], dtype=np.int64) for b in blocks]) if blocks else np.zeros(0)
        jobs = []
        r0 = c0 = 0
        for rows, cols, off, ld in blocks:
            jobs.append((r0, len(rows), c0, len(cols), off, ld))
            r0 += len(rows)
            c0 += len(cols)
        kernels.run_slp_jobs(ctx.dmesh, q, np.array(jobs, dtype=np.int64).reshape(-1, 6), ri.astype(np.int32),
                             ci.astype(np.int32), table, out)
    elif kind == kernels.DLP:
        kernels.run_dlp_jobs(ctx.dmesh, q, kernels.build_dlp_jobs(ctx.mesh, blocks), table, out)
    elif kind == kernels.HYP:
        kernels.run_hyp_blocks(ctx.dmesh, q, blocks, table, out)
    else:
        raise ValueError(f"unknown operator kind {kind!r}")


def dense_block(ctx, kind, row_dofs, col_dofs, q, require_disjoint=False, q_singular=None):
    """Dense Galerkin block over original dof lists (containers.py:48-66)."""
    if kind not in (kernels.SLP, kernels.DLP, kernels.HYP):
        raise ValueError(f"unknown operator kind {kind!r}")
    rows = np.asarray(row_dofs, dtype=np.int64)
    cols = np.asarray(col_dofs, dtype=np.int64)
    out = D.zeros((max(len(rows) * len(cols), 1),))
    if len(rows) and len(cols):
        _blocks_to_device(ctx, kind, [(rows, cols, 0, len(cols))], q, q if q_singular is None else q_singular,
                          require_disjoint, out)
    return D.host(out)[: len(rows) * len(cols)].reshape(len(rows), len(cols))


def assemble_dense(ctx, kind, q, cap=ORACLE_CAP, q_singular=None):
    mesh = ctx.mesh
    nr = mesh.n_vertices if kind == kernels.HYP else mesh.n_triangles
    nc = mesh.n_triangles if kind == kernels.SLP else mesh.n_vertices
    if max(nr, nc) > cap:
        raise ValueError(f"dense oracle dimension {max(nr, nc)} exceeds cap {cap}")
    return dense_block(ctx, kind, np.arange(nr), np.arange(nc), q, q_singular=q_singular)


# ---------------------------------------------------------------------------
# packed layouts

def _pad4(a):
    """Round row lengths up to a multiple of 4 doubles (32-byte rows for the
    256-bit streaming loads of the matvec)."""
    return (a + 3) & ~3


class NearLayout:
    """Per-row-leaf packing of the nearfield blocks."""

    def __init__(self, bt):
        rt, ct = bt.row_tree, bt.col_tree
        nu = bt.near_uids
        self.n_blocks = len(nu)
        order = np.argsort(nu[:, 0], kind="stable")
        su = nu[order]
        rows, cols = su[:, 0], su[:, 1]
        width = ct.end[cols] - ct.start[cols]
        nr_nodes = rt.n_nodes
        cnt = np.bincount(rows, minlength=nr_nodes)
        ptr = np.zeros(nr_nodes + 1, dtype=np.int64)
        np.cumsum(cnt, out=ptr[1:])
        wsum = np.zeros(nr_nodes + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, weights=width, minlength=nr_nodes).astype(np.int64), out=wsum[1:])
        C = _pad4(np.diff(wsum))
        # column offset of each block inside its row's matrix
        coloff = np.cumsum(width) - width - wsum[rows]
        height = rt.end - rt.start
        size = height * C
        off = np.zeros(nr_nodes + 1, dtype=np.int64)
        np.cumsum(size, out=off[1:])
        self.total = int(off[-1])
        self.C, self.off, self.ptr, self.col = C, off[:-1], ptr, cols
        self.s_rows, self.s_width, self.s_coloff = rows, width, coloff
        # per block in reference near order
        inv = np.empty_like(order)
        inv[order] = np.arange(len(order))
        self.blk_off = (off[:-1][rows] + coloff)[inv]
        self.blk_ld = C[rows][inv]
        self.blk_rows = (rt.end - rt.start)[nu[:, 0]]
        self.blk_cols = (ct.end - ct.start)[nu[:, 1]]
        self.entries = int((self.blk_rows * self.blk_cols).sum())


class FarLayout:
    """Per-row-cluster packing of the coupling matrices (needs ranks)."""

    def __init__(self, bt, rank_r, rank_c):
        fu = bt.far_uids
        self.n_blocks = len(fu)
        nr_nodes = bt.row_tree.n_nodes
        order = np.argsort(fu[:, 0], kind="stable") if len(fu) else np.zeros(0, dtype=np.int64)
        su = fu[order]
        rows, cols = su[:, 0], su[:, 1]
        width = rank_c[cols]
        cnt = np.bincount(rows, minlength=nr_nodes)
        ptr = np.zeros(nr_nodes + 1, dtype=np.int64)
        np.cumsum(cnt, out=ptr[1:])
        wsum = np.zeros(nr_nodes + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, weights=width, minlength=nr_nodes).astype(np.int64), out=wsum[1:])
        K = _pad4(np.diff(wsum))
        coloff = np.cumsum(width) - width - wsum[rows]
        size = rank_r * K
        off = np.zeros(nr_nodes + 1, dtype=np.int64)
        np.cumsum(size, out=off[1:])
        self.total = int(off[-1])
        self.K, self.off, self.ptr, self.col = K, off[:-1], ptr, cols
        self.s_rows, self.s_width, self.s_coloff = rows, width, coloff
        inv = np.empty_like(order)
        inv[order] = np.arange(len(order))
        self.blk_off = (off[:-1][rows] + coloff)[inv] if len(fu) else np.zeros(0, dtype=np.int64)
        self.blk_ld = K[rows][inv] if len(fu) else np.zeros(0, dtype=np.int64)
        self.blk_rows = rank_r[fu[:, 0]] if len(fu) else np.zeros(0, dtype=np.int64)
        self.blk_cols = rank_c[fu[:, 1]] if len(fu) else np.zeros(0, dtype=np.int64)
        self.entries = int((self.blk_rows * self.blk_cols).sum())


def near_layout(bt):
    if getattr(bt, "_near_layout", None) is None:
        bt._near_layout = NearLayout(bt)
    return bt._near_layout


def _near_blocks(bt, lay):
    rt, ct = bt.row_tree, bt.col_tree
    return [
        (rt.perm[rt.start[t] : rt.end[t]], ct.perm[ct.start[s] : ct.end[s]], int(lay.blk_off[i]), int(lay.blk_ld[i]))
        for i, (t, s) in enumerate(bt.near_uids)
    ]


def _symmetric_trees(bt):
    rt, ct = bt.row_tree, bt.col_tree
    return rt is ct or (np.array_equal(rt.perm, ct.perm) and np.array_equal(rt.start, ct.start)
                        and np.array_equal(rt.end, ct.end))


def _partners(bt, which):
    """kernels.block_partners of the block tree's far or near list, cached."""
    attr = "_h2b_partners_" + which
    hit = getattr(bt, attr, None)
    if hit is None:
        hit = kernels.block_partners(bt.far_uids if which == "far" else bt.near_uids)
        try:
            setattr(bt, attr, hit)
        except AttributeError:
            pass
    return hit


def near_slp_jobs(bt):
    """Pair-block jobs of the single-layer nearfield.  With one tree on both
    sides the matrix is symmetric (G(a,b) = G(b,a) for P0 x P0, and the
    Sauter-Schwab values are symmetrised, kernels.py:303-309): block (s, t) is
    written as the mirror of block (t, s) and diagonal blocks integrate their
    upper triangle only."""
    lay = near_layout(bt)
    rt, ct = bt.row_tree, bt.col_tree
    nu = bt.near_uids
    return kernels.block_jobs(nu, rt.start, rt.end - rt.start, ct.start, ct.end - ct.start, lay.blk_off, lay.blk_ld,
                              _partners(bt, "near") if _symmetric_trees(bt) else None)


def assemble_nearfield_device(ctx, kind, bt, q, q_singular=None, cache=None):
    """Packed device nearfield D (see module docstring)."""
    qs = q if q_singular is None else q_singular
    key = ("packed", kind, q, qs, id(bt))
    if cache is not None and key in cache:
        return cache[key]
    lay = near_layout(bt)
    out = D.zeros((max(lay.total, 1),))
    if kind == kernels.SLP:
        rt, ct = bt.row_tree, bt.col_tree
        jobs = near_slp_jobs(bt)
        kernels.run_slp_jobs(ctx.dmesh, q, jobs, rt.perm.astype(np.int32), ct.perm.astype(np.int32),
                             ctx.singular_table(kind, qs), out)
    else:
        _blocks_to_device(ctx, kind, _near_blocks(bt, lay), q, qs, False, out)
    if cache is not None:
        cache[key] = out
    return out


def _sharded_table(ctx, kind, q, own_panels):
    """The singular table of one rank: only the touching pairs its blocks look
    up are integrated (SingularTable.compute(own_panels))."""
    key = ("sharded", kind, q)
    tab = ctx._singular.get(key)
    if tab is None:
        tab = kernels.SingularTable(ctx.dmesh, kind, q, compute=False)
        ctx._singular[key] = tab
    tab.compute(own_panels)
    return tab


def _dst_map(n_full, index, off, ld):
    """(n_full,) destination offset / leading dimension of every block of the
    full list in a rank's packed layout (-1: stored by another rank)."""
    d_off = np.full(n_full, -1, dtype=np.int64)
    d_ld = np.zeros(n_full, dtype=np.int64)
    d_off[index] = off
    d_ld[index] = ld
    return d_off, d_ld


def near_slp_jobs_sharded(view):
    """Single-layer near jobs of one rank (view: BlockTreeView): the
    single-GPU job list (near_slp_jobs) restricted to the blocks the rank
    stores, every block pair in the single-GPU orientation."""
    full = view.full
    rt, ct = full.row_tree, full.col_tree
    lay = near_layout(view)
    nu = full.near_uids
    geom = np.stack([rt.start[nu[:, 0]], rt.end[nu[:, 0]] - rt.start[nu[:, 0]], ct.start[nu[:, 1]],
                     ct.end[nu[:, 1]] - ct.start[nu[:, 1]], np.zeros(len(nu), dtype=np.int64),
                     np.zeros(len(nu), dtype=np.int64)], axis=1)
    d_off, d_ld = _dst_map(len(nu), view.near_index, lay.blk_off, lay.blk_ld)
    return kernels.mirror_jobs_owned(geom, nu, d_off, d_ld, _partners(full, "near"))


def assemble_nearfield_sharded(ctx, kind, view, q, q_singular=None, own_panels=None):
    """Packed nearfield of one rank of a row-sharded operator (`view`: the
    rank's BlockTreeView, distributed.py): only the rank's near blocks are
    integrated and stored, and only the touching pairs they need.  For the
    single layer the block pairs are integrated in the orientation of the
    single-GPU job list (mirror_jobs_owned), so every stored entry has the
    same bits as the single-GPU assembly."""
    qs = q if q_singular is None else q_singular
    lay = near_layout(view)
    out = D.zeros((max(lay.total, 1),))
    if lay.n_blocks == 0:
        return out
    full = view.full
    rt, ct = full.row_tree, full.col_tree
    table = _sharded_table(ctx, kind, qs, own_panels)
    if kind == kernels.SLP and _symmetric_trees(full):
        kernels.run_slp_jobs(ctx.dmesh, q, near_slp_jobs_sharded(view), rt.perm.astype(np.int32),
                             ct.perm.astype(np.int32), table, out)
    else:
        _blocks_to_device(ctx, kind, _near_blocks(view, lay), q, qs, False, out, table=table)
    return out


def assemble_nearfield(ctx, kind, block_tree, q, cache=None, threads=1, q_singular=None):
    """Dense nearfield payloads in block order (containers.py:79-98); computed
    on the device, returned as host arrays.  Raises FloatingPointError on a
    non-finite entry."""
    out = assemble_nearfield_device(ctx, kind, block_tree, q, q_singular, cache)
    lay = near_layout(block_tree)
    h = D.host(out)
    return [_view(h, lay.blk_off[i], lay.blk_rows[i], lay.blk_cols[i], lay.blk_ld[i]) for i in range(lay.n_blocks)]


def _view(flat, off, nr, nc, ld):
    off, nr, nc, ld = int(off), int(nr), int(nc), int(ld)
    if nr == 0 or nc == 0:
        return np.zeros((nr, nc))
    return np.lib.stride_tricks.as_strided(flat[off:], shape=(nr, nc), strides=(8 * ld, 8)).copy()


def _basis_ranks(basis, n_nodes):
    """Per-node ranks as an array (cached on the basis with its pivot lists)."""
    return _pivots_concat(basis, n_nodes)[0]


def _pivots_concat(basis, n_nodes):
    """(ranks, offsets, concatenated pivots) of a basis in uid order, cached on
    the basis object (keyed by the node count and the identity of its dicts)."""
    key = (n_nodes, id(basis.rank), id(basis.pivots), len(basis.rank))
    hit = getattr(basis, "_h2b_concat", None)
    if hit is not None and hit[0] == key:
        return hit[1]
    ranks = np.array([basis.rank[u] for u in range(n_nodes)], dtype=np.int64)
    off = np.zeros(n_nodes + 1, dtype=np.int64)
    np.cumsum(ranks, out=off[1:])
    piv = np.concatenate([np.asarray(basis.pivots[u], dtype=np.int64) for u in range(n_nodes)]) if n_nodes else []
    res = (ranks, off, np.asarray(piv, dtype=np.int64))
    try:
        basis._h2b_concat = (key, res)
    except AttributeError:
        pass
    return res


def far_layout(bt, row_basis, col_basis):
    """FarLayout of a block tree (or view) for two bases, cached on the block
    tree per (row basis, column basis) pair."""
    rr = _basis_ranks(row_basis, bt.row_tree.n_nodes)
    cr = _basis_ranks(col_basis, bt.col_tree.n_nodes)
    cache = getattr(bt, "_h2b_far_layouts", None)
    if cache is None:
        cache = []
        try:
            bt._h2b_far_layouts = cache
        except AttributeError:
            return FarLayout(bt, rr, cr)
    for r0, c0, lay in cache:
        if r0 is rr and c0 is cr:
            return lay
    lay = FarLayout(bt, rr, cr)
    cache.append((rr, cr, lay))
    return lay


def coupling_slp_jobs(bt, row_basis, col_basis):
    """Single-layer coupling jobs S_b = G[pivots_t, pivots_s] over the
    concatenated pivot lists: (jobs, row pivots, col pivots, layout).  With
    one basis on both sides one job per block pair {(t, s), (s, t)}; `bt` may
    be a rank's BlockTreeView (only its blocks, single-GPU orientation)."""
    rr, roff, rpiv = _pivots_concat(row_basis, bt.row_tree.n_nodes)
    cr, coff, cpiv = _pivots_concat(col_basis, bt.col_tree.n_nodes)
    lay = far_layout(bt, row_basis, col_basis)
    fu = bt.far_uids
    full = getattr(bt, "full", None)
    sym = row_basis is col_basis and _symmetric_trees(bt)
    if full is not None and sym:
        ff = full.far_uids
        geom = np.stack([roff[ff[:, 0]], rr[ff[:, 0]], coff[ff[:, 1]], cr[ff[:, 1]],
                         np.zeros(len(ff), dtype=np.int64), np.zeros(len(ff), dtype=np.int64)], axis=1)
        d_off, d_ld = _dst_map(len(ff), bt.far_index, lay.blk_off, lay.blk_ld)
        jobs = kernels.mirror_jobs_owned(geom, ff, d_off, d_ld, _partners(full, "far"))
    else:
        # symmetric: S_(s,t) = G[piv_s, piv_t] = S_(t,s)^T, one job per block pair
        jobs = kernels.block_jobs(fu, roff[:-1], rr, coff[:-1], cr, lay.blk_off, lay.blk_ld,
                                  _partners(bt, "far") if sym else None)
    return jobs, rpiv.astype(np.int32), cpiv.astype(np.int32), lay


def assemble_couplings(ctx, kind, bt, row_basis, col_basis, q):
    """Packed device couplings S_b = G[pivots_t, pivots_s] (gca.py:198-203).
    `bt` may be a rank's BlockTreeView (row sharding): then only the rank's
    far blocks are integrated and stored, the symmetric pairs in the
    single-GPU orientation (same bits)."""
    rr, roff, rpiv = _pivots_concat(row_basis, bt.row_tree.n_nodes)
    cr, coff, cpiv = _pivots_concat(col_basis, bt.col_tree.n_nodes)
    lay = far_layout(bt, row_basis, col_basis)
    out = D.zeros((max(lay.total, 1),))
    fu = bt.far_uids
    if len(fu):
        if kind == kernels.SLP:
            jobs, rp, cp, _ = coupling_slp_jobs(bt, row_basis, col_basis)
            kernels.run_slp_jobs(ctx.dmesh, q, jobs, rp, cp, None, out)
        else:
            blocks = [(rpiv[roff[t] : roff[t + 1]], cpiv[coff[s] : coff[s + 1]], int(lay.blk_off[i]),
                       int(lay.blk_ld[i])) for i, (t, s) in enumerate(fu)]
            _blocks_to_device(ctx, kind, blocks, q, q, True, out)
    return out


# ---------------------------------------------------------------------------

class DenseOperator:
    def __init__(self, matrix):
        self.matrix = matrix
        self.shape = matrix.shape

    def matvec(self, x):
        return self.matrix @ x

    def rmatvec(self, x):
        return self.matrix.T @ x

    def diagonal(self):
        return np.diag(self.matrix).copy()

    def to_dense(self):
        return self.matrix

    def storage_report(self):
        return {"basis": 0, "coupling": 0, "lowrank": 0, "nearfield": 8 * self.matrix.size}


class ClusterBasis:
    """Nested cluster basis: V[leaf uid] (|t| x k_t), E[child uid]
    (k_child x k_parent), rank and pivots per uid (containers.py:189-238)."""

    def __init__(self, tree):
        self.tree = tree
        self.V = {}
        self.E = {}
        self.rank = {}
        self.pivots = {}

    def expand(self, cluster):
        """Dense V_t through the transfer matrices (testing aid)."""
        if cluster.is_leaf:
            return self.V[cluster.uid]
        return np.vstack([self.expand(ch) @ self.E[ch.uid] for ch in cluster.children])

    def storage_floats(self):
        return sum(v.size for v in self.V.values()) + sum(e.size for e in self.E.values())

    def forward(self, xp):
        """x_hat_t for every cluster from the permuted vector xp
        (containers.py:201-212): leaves V_t^T xp|_t, parents the sum over
        their children of E_ch^T x_hat_ch.  Runs on the device
        (h2b_basis_forward); returns {uid: (k_t,) array} like the reference
        (CUDA tensors in -> CUDA tensor values out)."""
        t = D.require_cuda()
        dev_in = isinstance(xp, t.Tensor)
        n = self.tree.n_dofs
        x = xp.contiguous() if dev_in else D.dev(np.asarray(xp, dtype=np.float64))
        if x.dtype != t.float64 or x.ndim != 1 or x.numel() != n:
            raise ValueError(f"expected a float64 vector of length {n}")
        db = self._device()
        xhat = t.empty(max(int(db.hat[-1]), 1), dtype=t.float64, device="cuda")
        _lib.check(_lib.lib().h2b_basis_forward(ctypes.byref(db.c), x.data_ptr(), xhat.data_ptr(), D.stream()))
        out = xhat if dev_in else D.host(xhat)
        return {u: out[db.hat[u] : db.hat[u + 1]] for u in range(self.tree.n_nodes)}

    def backward(self, yhat, yp):
        """Accumulate sum_t V_t y_hat_t into the permuted vector yp
        (containers.py:214-228): top down y_hat_ch += E_ch y_hat_t, then the
        leaves.  Clusters without an entry in yhat contribute nothing; yhat
        receives the propagated coefficients of every cluster below an entry,
        as in the reference.  Runs on the device (h2b_basis_backward); yp is
        updated in place (numpy array or CUDA tensor)."""
        t = D.require_cuda()
        db = self._device()
        n = self.tree.n_dofs
        dense = np.zeros(max(int(db.hat[-1]), 1))
        for u, v in yhat.items():
            v = D.host(v) if isinstance(v, t.Tensor) else np.asarray(v, dtype=np.float64)
            dense[db.hat[u] : db.hat[u + 1]] = v
        yd = D.dev(dense)
        dev_out = isinstance(yp, t.Tensor)
        if dev_out:
            if yp.dtype != t.float64 or yp.numel() != n or not yp.is_contiguous():
                raise ValueError(f"expected a contiguous float64 vector of length {n}")
            y = yp
        else:
            if np.shape(yp) != (n,):
                raise ValueError(f"expected a vector of length {n}")
            y = D.dev(np.asarray(yp, dtype=np.float64))
        _lib.check(_lib.lib().h2b_basis_backward(ctypes.byref(db.c), yd.data_ptr(), y.data_ptr(), D.stream()))
        if not dev_out:
            yp[...] = D.host(y)
        # the reference leaves the propagated coefficients in yhat
        reached = np.zeros(self.tree.n_nodes, dtype=bool)
        reached[list(yhat.keys())] = True
        for u in np.argsort(self.tree.depth_of, kind="stable"):
            p = self.tree.parent_of[u]
            if p >= 0 and reached[p]:
                reached[u] = True
        h = D.host(yd)
        for u in np.flatnonzero(reached):
            v = h[db.hat[u] : db.hat[u + 1]].copy()
            yhat[int(u)] = D.dev(v) if dev_out else v
        return yp

    def _device(self):
        """Device copy of the packed basis + the h2b_basis descriptor (cached)."""
        if getattr(self, "_dev", None) is None:
            self._dev = _BasisTransforms(self)
        return self._dev

    def packed(self):
        """(ranks, V flat, v_off, E flat, e_off, hat_off) in uid order; cached.
        Every block starts 16-byte aligned and is padded to an even number of
        doubles, so the matvec can stage it with one TMA bulk copy."""
        if getattr(self, "_packed", None) is None:
            t = self.tree
            n = t.n_nodes
            ranks = np.array([self.rank[u] for u in range(n)], dtype=np.int64)
            v_off = np.full(n, -1, dtype=np.int64)
            e_off = np.full(n, -1, dtype=np.int64)
            vs, es = [], []
            pad = np.zeros(1)
            pos = 0
            for u in t.leaf_uids():
                v_off[u] = pos
                vs.append(np.ascontiguousarray(self.V[u]).ravel())
                pos += vs[-1].size
                if pos & 1:
                    vs.append(pad)
                    pos += 1
            pos = 0
            for u in range(n):
                if t.parent_of[u] >= 0:
                    e_off[u] = pos
                    es.append(np.ascontiguousarray(self.E[u]).ravel())
                    pos += es[-1].size
                    if pos & 1:
                        es.append(pad)
                        pos += 1
            hat = np.zeros(n + 1, dtype=np.int64)
            np.cumsum(ranks, out=hat[1:])
            self._packed = (ranks, np.concatenate(vs) if vs else np.zeros(1), v_off,
                            np.concatenate(es) if es else np.zeros(1), e_off, hat)
        return self._packed


class _BasisTransforms:
    """h2b_basis descriptor of a ClusterBasis: packed V / E on the device and
    the clusters listed level by level (root first)."""

    def __init__(self, basis):
        t = basis.tree
        ranks, V, v_off, E, e_off, hat = basis.packed()
        order = np.argsort(t.depth_of, kind="stable")
        depth = t.depth_of[order]
        level_off = np.searchsorted(depth, np.arange(int(depth.max()) + 2)).astype(np.int64)
        self.hat = hat
        self._keep = [D.dev(a, dt) for a, dt in (
            (t.left, np.int32), (t.right, np.int32), (t.start, np.int32), (t.end - t.start, np.int32),
            (ranks, np.int32), (np.maximum(v_off, 0), np.int64), (np.maximum(e_off, 0), np.int64),
            (hat[:-1], np.int64), (V, np.float64), (E, np.float64), (order, np.int32))]
        k = self._keep
        self._level_off = level_off
        self.c = _lib.Basis(t.n_nodes, *(a.data_ptr() for a in k[:10]), len(level_off) - 1, _lib.ptr(level_off),
                            k[10].data_ptr())


class _DeviceBasis:
    def __init__(self, basis):
        ranks, V, v_off, E, e_off, hat = basis.packed()
        self.ranks = ranks
        self.V = D.dev(V)
        self.E = D.dev(E)
        self.v_off = v_off
        self.e_off = e_off
        self.hat = hat


class H2Matrix:
    """Device-resident H^2 operator (containers.py:241-324).  matvec accepts a
    numpy array (copied in/out) or a CUDA tensor (zero-copy) in natural dof
    order and returns the same type."""

    def __init__(self, block_tree, row_basis, col_basis, couplings, near_payloads):
        """Reference constructor from host payload lists (block-tree order)."""
        rr = np.array([row_basis.rank[u] for u in range(block_tree.row_tree.n_nodes)], dtype=np.int64)
        cr = np.array([col_basis.rank[u] for u in range(block_tree.col_tree.n_nodes)], dtype=np.int64)
        fl = FarLayout(block_tree, rr, cr)
        nl = near_layout(block_tree)
        S = np.zeros(max(fl.total, 1))
        Dn = np.zeros(max(nl.total, 1))
        for i, s in enumerate(couplings):
            _scatter(S, fl.blk_off[i], fl.blk_ld[i], np.asarray(s, dtype=float))
        for i, d in enumerate(near_payloads):
            _scatter(Dn, nl.blk_off[i], nl.blk_ld[i], np.asarray(d, dtype=float))
        self._init(block_tree, row_basis, col_basis, D.dev(S), D.dev(Dn), fl)

    @classmethod
    def from_device(cls, block_tree, row_basis, col_basis, S, Dn):
        self = cls.__new__(cls)
        self._init(block_tree, row_basis, col_basis, S, Dn, far_layout(block_tree, row_basis, col_basis))
        return self

    def _init(self, bt, rb, cb, S, Dn, far_layout):
        self.block_tree = bt
        self.row_tree = bt.row_tree
        self.col_tree = bt.col_tree
        self.row_basis = rb
        self.col_basis = cb
        self.shape = (self.row_tree.n_dofs, self.col_tree.n_dofs)
        self.S_dev = S
        self.D_dev = Dn
        self.far_layout = far_layout
        self.near_layout = near_layout(bt)
        self._plan = None
        self._tplan = None
        self._far = None
        self._near = None

    # -- reference attribute views ------------------------------------------------
    @property
    def far(self):
        if self._far is None:
            h = D.host(self.S_dev)
            fl = self.far_layout
            self._far = [(b, _view(h, fl.blk_off[i], fl.blk_rows[i], fl.blk_cols[i], fl.blk_ld[i]))
                         for i, b in enumerate(self.block_tree.far)]
        return self._far

    @property
    def near(self):
        if self._near is None:
            h = D.host(self.D_dev)
            nl = self.near_layout
            self._near = [(b, _view(h, nl.blk_off[i], nl.blk_rows[i], nl.blk_cols[i], nl.blk_ld[i]))
                          for i, b in enumerate(self.block_tree.near)]
        return self._near

    # -- device plan ----------------------------------------------------------------
    def plan(self):
        if self._plan is None:
            self._plan = MatvecPlan(self.block_tree, self.row_basis, self.col_basis, self.S_dev, self.D_dev,
                                    self.far_layout, self.near_layout)
        return self._plan

    def matvec(self, x):
        return self.plan().apply(x)

    def rmatvec(self, x):
        """x^T A (containers.py:272-288).  A single-layer operator assembled
        with one basis on both sides is symmetric entry by entry (mirrored
        couplings and nearfield), so its transpose is the operator itself and
        the matvec plan is reused; otherwise the couplings and nearfield are
        transposed on the device (h2b_transpose_blocks) into a plan for A^T."""
        if getattr(self, "symmetric", False):
            return self.matvec(x)
        if self._tplan is None:
            self._tplan = _transposed_plan(self)
        return self._tplan.apply(x)

    def matmat(self, X):
        """Y = A X for a block of right-hand sides X (n_cols x nrhs): numpy in ->
        numpy out, CUDA tensor -> tensor.  Not in the reference (its matvec is
        single-vector); column j equals matvec(X[:, j]) to rounding."""
        if getattr(self, "_mmplan", None) is None:
            self._mmplan = MatmatPlan(self.plan())
        return self._mmplan.apply(X)

    def diagonal(self):
        assert self.shape[0] == self.shape[1], "diagonal extraction requires a square operator"
        return self.plan().diagonal()

    def to_dense(self):
        n = self.shape[1]
        out = np.empty((self.shape[0], n))
        eye = np.zeros(n)
        for j in range(n):
            eye[j] = 1.0
            out[:, j] = self.matvec(eye)
            eye[j] = 0.0
        return out

    def rank_stats(self):
        if self.far_layout.n_blocks == 0:
            return {"max": 0, "mean": 0.0}
        flat = np.concatenate([self.far_layout.blk_rows, self.far_layout.blk_cols])
        return {"max": int(flat.max()), "mean": float(flat.mean())}

    def storage_report(self):
        basis = self.row_basis.storage_floats()
        if self.col_basis is not self.row_basis:
            basis += self.col_basis.storage_floats()
        return {"basis": 8 * basis, "coupling": 8 * self.far_layout.entries, "lowrank": 0,
                "nearfield": 8 * self.near_layout.entries}

    def matvec_bytes(self):
        """Algorithmic HBM bytes of one matvec: every operator
        entry once, each basis in both roles, plus x and y."""
        basis_r = self.row_basis.storage_floats()
        basis_c = self.col_basis.storage_floats()
        return 8 * (self.near_layout.entries + self.far_layout.entries + basis_r + basis_c + self.shape[0]
                    + self.shape[1])

    def streamed_bytes(self):
        """Bytes the single-GPU plan actually streams per matvec: a symmetric
        nearfield (or coupling set) is stored once per block pair
        (MatvecPlan.info), i.e. below matvec_bytes()."""
        info = self.plan().info()
        near = info["near_bytes"] if info["near_symmetric"] else 8 * self.near_layout.entries
        cpl = info["coupling_bytes"] if info["coupling_symmetric"] else 8 * self.far_layout.entries
        return self.matvec_bytes() - 8 * (self.near_layout.entries + self.far_layout.entries) + near + cpl


def _scatter(flat, off, ld, block):
    nr, nc = block.shape
    if nr == 0 or nc == 0:
        return
    view = np.lib.stride_tricks.as_strided(flat[int(off):], shape=(nr, nc), strides=(8 * int(ld), 8))
    view[...] = block


def _gather_index(n_nodes, row_len, rows, width, coloff, first):
    """Per-row-node gather lists: for every block (row node, width, column
    offset inside the row's matrix) the `width` source indices first[b] + j.
    Returns (offsets per node, flat int32 indices).  Padding columns (zero
    matrix columns) repeat the row's first index: a gather never touches a
    value nobody produces (the matvec skips x_hat of clusters without far
    blocks above them)."""
    goff = np.zeros(n_nodes + 1, dtype=np.int64)
    np.cumsum(row_len, out=goff[1:])
    gidx = np.zeros(max(int(goff[-1]), 1), dtype=np.int64)
    total = int(width.sum())
    if total:
        blk = np.repeat(np.arange(len(width)), width)
        j = np.arange(total) - np.repeat(np.cumsum(width) - width, width)
        gidx[goff[rows][blk] + coloff[blk] + j] = first[blk] + j
        real = np.bincount(rows, weights=width, minlength=n_nodes).astype(np.int64)
        pad = np.asarray(row_len, dtype=np.int64) - real
        has = np.nonzero((pad > 0) & (real > 0))[0]
        if len(has):
            pos = np.repeat(goff[has] + real[has], pad[has]) + (np.arange(int(pad[has].sum())) -
                                                                 np.repeat(np.cumsum(pad[has]) - pad[has], pad[has]))
            gidx[pos] = np.repeat(gidx[goff[has]], pad[has])
    return goff[:-1], gidx


class MatvecPlan:
    """Device layout + libh2b plan for y = A x."""

    def __init__(self, bt, rb, cb, S, Dn, fl, nl, owned=None, col_perm=None, row_perm=None, xhat_mask=None):
        t = D.require_cuda()
        rt, ct = bt.row_tree, bt.col_tree
        self.n_rows, self.n_cols = rt.n_dofs, ct.n_dofs
        self._rb = _DeviceBasis(rb)
        self._cb = self._rb if cb is rb else _DeviceBasis(cb)
        i32 = np.int32
        keep = {}

        def put(name, arr, dtype):
            keep[name] = D.dev(arr, dtype)
            return keep[name].data_ptr()

        cbd, rbd = self._cb, self._rb
        c_child = np.stack([ct.left, ct.right], axis=1)
        c_leaves = ct.leaf_uids()
        r_order = np.argsort(rt.depth_of, kind="stable")
        r_vo = rbd.v_off.copy()
        lay = _lib.Layout()
        lay.n_rows, lay.n_cols = self.n_rows, self.n_cols
        lay.col_perm = put("col_perm", ct.perm if col_perm is None else col_perm, np.int64)
        lay.row_perm = put("row_perm", rt.perm if row_perm is None else row_perm, np.int64)
        lay.c_nodes, lay.c_leaves = ct.n_nodes, len(c_leaves)
        lay.c_parent = put("c_parent", ct.parent_of, i32)
        lay.c_child = put("c_child", c_child, i32)
        lay.c_start = put("c_start", ct.start, i32)
        lay.c_size = put("c_size", ct.end - ct.start, i32)
        lay.c_rank = put("c_rank", cbd.ranks, i32)
        lay.c_v_off = put("c_v_off", cbd.v_off, np.int64)
        lay.c_e_off = put("c_e_off", cbd.e_off, np.int64)
        lay.c_xhat_off = put("c_xhat_off", cbd.hat[:-1], np.int64)
        lay.c_leaf_list = put("c_leaf_list", c_leaves, i32)
        lay.c_V, lay.c_E = cbd.V.data_ptr(), cbd.E.data_ptr()
        lay.xhat_len = int(cbd.hat[-1])
        lay.r_nodes, lay.r_leaves = rt.n_nodes, len(rt.leaf_uids())
        lay.r_parent = put("r_parent", rt.parent_of, i32)
        lay.r_start = put("r_start", rt.start, i32)
        lay.r_size = put("r_size", rt.end - rt.start, i32)
        lay.r_rank = put("r_rank", rbd.ranks, i32)
        lay.r_v_off = put("r_v_off", r_vo, np.int64)
        lay.r_e_off = put("r_e_off", rbd.e_off, np.int64)
        lay.r_yhat_off = put("r_yhat_off", rbd.hat[:-1], np.int64)
        lay.r_order = put("r_order", r_order, i32)
        lay.r_V, lay.r_E = rbd.V.data_ptr(), rbd.E.data_ptr()
        lay.yhat_len = int(rbd.hat[-1])
        lay.s_off = put("s_off", fl.off, np.int64)
        lay.s_cols = put("s_cols", fl.K, i32)
        lay.far_ptr = put("far_ptr", fl.ptr, i32)
        lay.far_col = put("far_col", fl.col if len(fl.col) else np.zeros(1), i32)
        lay.S = S.data_ptr()
        lay.d_off = put("d_off", nl.off, np.int64)
        lay.d_cols = put("d_cols", nl.C, i32)
        lay.near_ptr = put("near_ptr", nl.ptr, i32)
        lay.near_col = put("near_col", nl.col if len(nl.col) else np.zeros(1), i32)
        lay.D = Dn.data_ptr()
        # right-hand-side gather lists (x for the nearfield, x_hat for couplings)
        cperm = ct.perm if col_perm is None else np.asarray(col_perm)
        nrow_len = np.where(rt.left < 0, nl.C, 0)
        goff, gidx = _gather_index(rt.n_nodes, nrow_len, nl.s_rows, nl.s_width, nl.s_coloff, ct.start[nl.col])
        gidx = cperm[gidx] if len(cperm) else gidx
        if nl.total == 0:
            gidx = np.zeros(1, dtype=np.int64)
        lay.d_goff = put("d_goff", goff, np.int64)
        lay.d_gidx = put("d_gidx", gidx, np.int32)
        soff, sidx = _gather_index(rt.n_nodes, fl.K, fl.s_rows, fl.s_width, fl.s_coloff, cbd.hat[:-1][fl.col])
        lay.s_goff = put("s_goff", soff, np.int64)
        lay.s_gidx = put("s_gidx", sidx, np.int32)
        if owned is not None:
            lay.n_owned = len(owned)
            lay.owned = put("owned", owned, i32)
        else:
            lay.n_owned = 0
            lay.owned = None
        self._keep = keep
        self._S, self._D = S, Dn
        self.layout = lay
        h = ctypes.c_void_p()
        if xhat_mask is None:
            _lib.check(_lib.lib().h2b_plan_create(ctypes.byref(lay), ctypes.byref(h)))
        else:
            # x_hat exchange (distributed.ShardedMatvec(xhat=True)): forward
            # tasks over this rank's column clusters only
            self._xmask = np.ascontiguousarray(xhat_mask, dtype=np.int8)
            _lib.check(_lib.lib().h2b_plan_create_xhat(ctypes.byref(lay), _lib.ptr(self._xmask), ctypes.byref(h)))
        self.handle = h
        self._torch = t
        self._host_fn = _lib.lib().h2b_matvec_host

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.lib().h2b_plan_destroy(h)
            except Exception:
                pass

    def apply_device(self, x, y=None, stream=None):
        """y = A x for CUDA float64 tensors (natural order), stream-ordered."""
        t = self._torch
        if y is None:
            y = t.empty(self.n_rows, dtype=t.float64, device=x.device)
        _lib.check(_lib.lib().h2b_matvec(self.handle, x.data_ptr(), y.data_ptr(), _lib.stream_ptr(stream)))
        return y

    def apply(self, x):
        t = self._torch
        if type(x) is np.ndarray and x.dtype == np.float64 and x.ndim == 1 and x.flags.c_contiguous:
            # fast path of the common host call (numpy in, numpy out)
            if len(x) != self.n_cols:
                raise ValueError(f"expected a vector of length {self.n_cols}")
            y = t.empty(self.n_rows, dtype=t.float64, pin_memory=True).numpy()
            rc = self._host_fn(self.handle, x.__array_interface__["data"][0], y.__array_interface__["data"][0],
                               t.cuda.current_stream().cuda_stream)
            if rc:
                _lib.check(rc)
            return y
        if isinstance(x, t.Tensor):
            if x.dtype != t.float64 or not x.is_cuda:
                raise ValueError("expected a CUDA float64 tensor")
            return self.apply_device(x.contiguous())
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.ndim != 1 or len(x) != self.n_cols:
            raise ValueError(f"expected a vector of length {self.n_cols}")
        # the result lands in page-locked host memory (torch's caching host
        # allocator: cheap after the first call), so its copy back is one DMA;
        # x is copied by DMA when page-locked, by the driver's staged copy otherwise
        y = t.empty(self.n_rows, dtype=t.float64, pin_memory=True).numpy()
        _lib.check(_lib.lib().h2b_matvec_host(self.handle, _lib.ptr(x), _lib.ptr(y), _lib.stream_ptr()))
        return y

    def diagonal(self):
        d = D.zeros((self.n_rows,))
        _lib.check(_lib.lib().h2b_diagonal(self.handle, d.data_ptr(), _lib.stream_ptr()))
        return D.host(d)

    def info(self):
        """Plan facts (h2b_plan_info): whether the nearfield is streamed once
        per block pair (single-GPU plans of a bitwise symmetric nearfield), the
        nearfield bytes one matvec streams, task counts."""
        out = (ctypes.c_int64 * 9)()
        _lib.check(_lib.lib().h2b_plan_info(self.handle, out))
        return {"near_symmetric": bool(out[0]), "near_bytes": int(out[1]), "near_tasks": int(out[2]),
                "coupling_tasks": int(out[3]), "partial_bytes": int(out[4]), "coupling_symmetric": bool(out[5]),
                "coupling_bytes": int(out[6]), "stage_bytes": int(out[7]), "smem_per_cta": int(out[8])}


class MatmatPlan:
    """libh2b block product (h2b_matmat) over a matvec plan's device layout."""

    MAX_RHS = 16

    def __init__(self, mv_plan):
        self._mv = mv_plan  # owns the layout arrays the block plan points into
        self.n_rows, self.n_cols = mv_plan.n_rows, mv_plan.n_cols
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().h2b_matmat_create(ctypes.byref(mv_plan.layout), ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.lib().h2b_matmat_destroy(h)
            except Exception:
                pass

    def apply_device(self, X, Y=None, stream=None):
        """Y (n_rows x nrhs) = A X for a CUDA float64 tensor X (n_cols x nrhs),
        in slices of at most 16 columns (stream-ordered)."""
        t = D.torch()
        if X.ndim != 2 or X.shape[0] != self.n_cols:
            raise ValueError(f"expected a ({self.n_cols}, nrhs) block")
        nrhs = X.shape[1]
        if Y is None:
            Y = t.empty((self.n_rows, nrhs), dtype=t.float64, device=X.device)
        L = _lib.lib()
        for j0 in range(0, nrhs, self.MAX_RHS):
            j1 = min(nrhs, j0 + self.MAX_RHS)
            xs = X[:, j0:j1].contiguous() if (j0 > 0 or j1 < nrhs or not X.is_contiguous()) else X
            ys = Y if (j0 == 0 and j1 == nrhs and Y.is_contiguous()) else t.empty((self.n_rows, j1 - j0),
                                                                                   dtype=t.float64, device=X.device)
            _lib.check(L.h2b_matmat(self.handle, xs.data_ptr(), ys.data_ptr(), j1 - j0, _lib.stream_ptr(stream)))
            if ys is not Y:
                Y[:, j0:j1] = ys
        return Y

    def apply(self, X):
        t = D.torch()
        if isinstance(X, t.Tensor):
            if X.dtype != t.float64 or not X.is_cuda:
                raise ValueError("expected a CUDA float64 tensor")
            return self.apply_device(X)
        X = np.asarray(X, dtype=np.float64)
        if X.ndim == 1:
            return D.host(self.apply_device(D.dev(X[:, None])))[:, 0]
        return D.host(self.apply_device(D.dev(np.ascontiguousarray(X))))


def _transposed_plan(H):
    """Plan for A^T: swapped trees/bases, S_b^T and D_b^T repacked on the device."""
    from .clustering import BlockTree

    bt = H.block_tree
    tb = BlockTree.__new__(BlockTree)
    tb.row_tree, tb.col_tree, tb.eta = bt.col_tree, bt.row_tree, bt.eta
    tb.far_uids = bt.far_uids[:, ::-1].copy()
    tb.near_uids = bt.near_uids[:, ::-1].copy()
    tb._far = tb._near = None
    rr = np.array([H.col_basis.rank[u] for u in range(tb.row_tree.n_nodes)], dtype=np.int64)
    cr = np.array([H.row_basis.rank[u] for u in range(tb.col_tree.n_nodes)], dtype=np.int64)
    fl = FarLayout(tb, rr, cr)
    nl = NearLayout(tb)
    St = _transpose_packed(H.S_dev, H.far_layout, fl, max(fl.total, 1))
    Dt = _transpose_packed(H.D_dev, H.near_layout, nl, max(nl.total, 1))
    return MatvecPlan(tb, H.col_basis, H.row_basis, St, Dt, fl, nl)


def _transpose_packed(src, la, lb, total):
    """Repack on the device (h2b_transpose_blocks): entry (i, j) of block b in
    layout `la` -> (j, i) of block b in layout `lb`; padding stays zero."""
    out = D.zeros((total,))
    n = len(la.blk_off)
    if n:
        desc = np.stack([la.blk_off, la.blk_ld, la.blk_rows, la.blk_cols, lb.blk_off, lb.blk_ld],
                        axis=1).astype(np.int64)
        keep = (desc[:, 2] > 0) & (desc[:, 3] > 0)
        desc = np.ascontiguousarray(desc[keep])
        dd = D.dev(desc, np.int64)
        _lib.check(_lib.lib().h2b_transpose_blocks(len(desc), dd.data_ptr(), src.data_ptr(), out.data_ptr(),
                                                   D.stream()))
    return out
