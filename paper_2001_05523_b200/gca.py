"""Green cross approximation (GCA) H^2 construction.  API of h2bem.gca
(gca.py:1-205).

* Basis construction (`build_basis`) runs on the host, level-synchronously
  with a thread pool, and is numerically identical to the reference: the pivot
  sets are integers and decide the whole H^2 operator, so the Green-quadrature
  columns (single-panel potentials, kernels.py:97-196) and the pivoted cross
  approximation are evaluated with the same numpy/BLAS operations in the same
  order (Gram-form squared distances, same chunking, same einsum paths).
  BLAS is pinned to one thread inside the pool (the reference's OpenBLAS race,
  SURVEY.md section 0).  Moving this to the GPU is the next step.
* `assemble_h2` fills the coupling matrices S_b = G[pivots_t, pivots_s] and
  the nearfield on the GPU (libh2b pair-block kernels) and returns the
  device-resident H2Matrix.
"""

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import kernels
from .lowrank import aca_inverse_core
from .quadrature import gauss_legendre

P0_SLP = "p0_slp"
P1_DLP = "p1_dlp"
P1_CURL = "p1_curl"

DEGENERATE_WIDTH = 1e-12
FOUR_PI = 4.0 * np.pi
_TINY = 1e-100


@dataclass(frozen=True)
class GreenBox:
    box: np.ndarray
    points: np.ndarray
    weights: np.ndarray
    normals: np.ndarray


def widen_degenerate(box):
    """Give flat box extents a tiny width (hca.py:28-37)."""
    box = np.asarray(box, dtype=float).copy()
    ext = box[1] - box[0]
    pad = DEGENERATE_WIDTH * max(ext.max(), 1.0)
    for d in range(3):
        if ext[d] < pad:
            mid = 0.5 * (box[0, d] + box[1, d])
            box[0, d] = mid - 0.5 * pad
            box[1, d] = mid + 0.5 * pad
    return box


def green_box(box_t):
    """Cluster box inflated by its longest edge on every side."""
    box_t = widen_degenerate(box_t)
    delta = float((box_t[1] - box_t[0]).max())
    return np.stack([box_t[0] - delta, box_t[1] + delta])


def green_quadrature(box, m):
    """m x m Gauss rule on each of the 6 box faces (k = 6 m^2 points): faces
    ordered axis 0..2, lower side before upper side."""
    if m < 1:
        raise ValueError("quadrature order must be >= 1")
    box = np.asarray(box, dtype=float)
    g = gauss_legendre(m)
    P, Wt, Nn = [], [], []
    for axis in range(3):
        u, v = (axis + 1) % 3, (axis + 2) % 3
        lu, lv = box[1, u] - box[0, u], box[1, v] - box[0, v]
        cu = box[0, u] + lu * g.points
        cv = box[0, v] + lv * g.points
        wface = np.outer(lu * g.weights, lv * g.weights).ravel()
        for side in (0, 1):
            pts = np.empty((m * m, 3))
            pts[:, axis] = box[side, axis]
            pts[:, u] = np.repeat(cu, m)
            pts[:, v] = np.tile(cv, m)
            nrm = np.zeros((m * m, 3))
            nrm[:, axis] = 1.0 if side else -1.0
            P.append(pts)
            Wt.append(wface)
            Nn.append(nrm)
    return GreenBox(box, np.vstack(P), np.concatenate(Wt), np.vstack(Nn))


# ---------------------------------------------------------------------------
# single-panel potentials at external points (host, reference-identical numerics)

def _gram_r2(X, Z):
    r2 = X @ Z.T
    r2 *= -2.0
    r2 += np.einsum("ij,ij->i", X, X)[:, None]
    r2 += np.einsum("ij,ij->i", Z, Z)[None, :]
    return np.maximum(r2, _TINY, out=r2)


def panel_potentials(mesh, tris, Z, kind, q, z_normals=None, bary=False, pq=None, chunk=4_000_000):
    """Integrals of (basis x kernel) over panels `tris` at points Z:
    (P, N), or (P, N, 3) weighted by the local barycentrics when bary=True.
    kind in {value, dn_z, dn_x, dn_x_dn_z} (kernels.K_*)."""
    from . import quadrature as quad

    tris = np.asarray(tris, dtype=np.int64)
    Z = np.atleast_2d(np.asarray(Z, dtype=float))
    if pq is None:
        X, W, lam = quad.triangle_points(mesh, tris, q)
    else:
        X, W, lam = pq[0][tris], pq[1][tris], pq[2]
    P, Q = W.shape
    N = len(Z)
    nz = None if z_normals is None else np.asarray(z_normals, dtype=float)
    if kind in (kernels.K_DN_Z, kernels.K_DN_X_DN_Z) and nz is None:
        raise ValueError(f"kind {kind!r} requires z_normals")
    z_dot_n = np.einsum("nj,nj->n", Z, nz) if kind in (kernels.K_DN_Z, kernels.K_DN_X_DN_Z) else None
    na = mesh.normals[tris] if kind in (kernels.K_DN_X, kernels.K_DN_X_DN_Z) else None
    out = np.empty((P, N, 3)) if bary else np.empty((P, N))
    step = max(1, chunk // max(1, Q * N))
    for lo in range(0, P, step):
        sl = slice(lo, min(lo + step, P))
        Xf = X[sl].reshape(-1, 3)
        r2 = _gram_r2(Xf, Z)
        r = np.sqrt(r2)
        if kind == kernels.K_VALUE:
            k = 1.0 / (FOUR_PI * r)
        elif kind == kernels.K_DN_Z:
            k = ((Xf @ nz.T) - z_dot_n[None, :]) / (FOUR_PI * r2 * r)
        elif kind in (kernels.K_DN_X, kernels.K_DN_X_DN_Z):
            xa = np.einsum("pqj,pj->pq", X[sl], na[sl]).reshape(-1)
            za = na[sl] @ Z.T
            dna = xa[:, None] - np.repeat(za, Q, axis=0)
            if kind == kernels.K_DN_X:
                k = -dna / (FOUR_PI * r2 * r)
            else:
                dnz = (Xf @ nz.T) - z_dot_n[None, :]
                nanz = np.repeat(na[sl] @ nz.T, Q, axis=0)
                k = (nanz - 3.0 * dna * dnz / r2) / (FOUR_PI * r2 * r)
        else:
            raise ValueError(f"unknown kernel tag {kind!r}")
        k = k.reshape(-1, Q, N)
        if bary:
            out[sl] = np.einsum("pqn,pq,ql->pnl", k, W[sl], lam, optimize=True)
        else:
            out[sl] = np.einsum("pqn,pq->pn", k, W[sl], optimize=True)
    return out


def _incident_panels(ctx, verts):
    ptr, idx = ctx.mesh.vertex_triangle_csr()
    verts = np.asarray(verts, dtype=np.int64)
    if len(verts) == 0:
        return np.empty(0, dtype=np.int64)
    return np.unique(np.concatenate([idx[ptr[v] : ptr[v + 1]] for v in verts]))


def p1_potentials(ctx, verts, Z, kind, q, z_normals=None, pq=None):
    """Hat-function potentials out[r, n] = int phi_{verts[r]} kernel(., Z[n])."""
    mesh = ctx.mesh
    verts = np.asarray(verts, dtype=np.int64)
    Z = np.atleast_2d(Z)
    panels = _incident_panels(ctx, verts)
    vals = panel_potentials(mesh, panels, Z, kind, q, z_normals=z_normals, bary=True, pq=pq)
    pos = -np.ones(mesh.n_vertices, dtype=np.int64)
    pos[verts] = np.arange(len(verts))
    out = np.zeros((len(verts), len(Z)))
    ri = pos[mesh.triangles[panels]]
    for l in range(3):
        keep = np.flatnonzero(ri[:, l] >= 0)
        if len(keep):
            np.add.at(out, ri[keep, l], vals[keep, :, l])
    return out


def curl_potentials(ctx, verts, Z, kind, q, z_normals=None, pq=None):
    """Surface-curl-weighted hat potentials, one component per direction:
    out[r, n, d] = int (curl phi_{verts[r]})_d kernel(., Z[n]) (kernels.py:
    172-196): P0 panel potentials scattered with the per-panel curls."""
    mesh = ctx.mesh
    verts = np.asarray(verts, dtype=np.int64)
    Z = np.atleast_2d(Z)
    curls = ctx.curls
    panels = _incident_panels(ctx, verts)
    vals = panel_potentials(mesh, panels, Z, kind, q, z_normals=z_normals, pq=pq)
    pos = -np.ones(mesh.n_vertices, dtype=np.int64)
    pos[verts] = np.arange(len(verts))
    out = np.zeros((len(verts), len(Z), 3))
    ri = pos[mesh.triangles[panels]]
    for l in range(3):
        keep = np.flatnonzero(ri[:, l] >= 0)
        if len(keep):
            np.add.at(out, ri[keep, l], vals[keep, :, None] * curls[panels[keep], l, None, :])
    return out


def green_columns(ctx, flavor, dofs, gq, q_single):
    """L whose rows span the cluster's farfield interaction space: sqrt(w)-scaled
    potentials against the Green kernels, [value | normal derivative] (2k cols)."""
    mesh = ctx.mesh
    sw = np.sqrt(gq.weights)
    pq = ctx.host_panel_quad(q_single)
    if flavor == P0_SLP:
        a = panel_potentials(mesh, dofs, gq.points, kernels.K_VALUE, q_single, pq=pq)
        c = panel_potentials(mesh, dofs, gq.points, kernels.K_DN_Z, q_single, z_normals=gq.normals, pq=pq)
    elif flavor == P1_DLP:
        a = p1_potentials(ctx, dofs, gq.points, kernels.K_DN_X, q_single, pq=pq)
        c = p1_potentials(ctx, dofs, gq.points, kernels.K_DN_X_DN_Z, q_single, z_normals=gq.normals, pq=pq)
    elif flavor == P1_CURL:
        # 6k columns: the three curl components of the value and of the
        # normal-derivative potentials
        a = curl_potentials(ctx, dofs, gq.points, kernels.K_VALUE, q_single, pq=pq)
        c = curl_potentials(ctx, dofs, gq.points, kernels.K_DN_Z, q_single, z_normals=gq.normals, pq=pq)
        return np.hstack([a[:, :, d] * sw for d in range(3)] + [c[:, :, d] * sw for d in range(3)])
    else:
        raise ValueError(f"unknown basis flavor {flavor!r}")
    return np.hstack([a * sw, c * sw])


def cross_interpolate(L, eps):
    """Row pivots tau and V = L[:, sigma] inv(L[tau, sigma])."""
    tau, sigma, C, _ = aca_inverse_core(L, eps)
    if len(tau) == 0:
        return np.empty(0, dtype=np.int64), np.zeros((L.shape[0], 0))
    return tau, L[:, sigma] @ C


def gca_leaf(ctx, flavor, dofs, box, m, eps_aca, q_single):
    L = green_columns(ctx, flavor, dofs, green_quadrature(green_box(box), m), q_single)
    tau, V = cross_interpolate(L, eps_aca)
    return np.asarray(dofs)[tau], V


def gca_nested(ctx, flavor, child_pivots, box, m, eps_aca, q_single):
    rows = np.concatenate(child_pivots)
    L = green_columns(ctx, flavor, rows, green_quadrature(green_box(box), m), q_single)
    tau, Vhat = cross_interpolate(L, eps_aca)
    return rows[tau], Vhat


def green_points_batch(boxes, m):
    """Green points of many clusters at once: (n, 6 m^2, 8) = x, y, z,
    sqrt(w), nx, ny, nz, 0 -- the same floating-point operations as
    green_quadrature(green_box(box), m) per cluster, vectorised."""
    boxes = np.asarray(boxes, dtype=float).reshape(-1, 2, 3).copy()
    n = len(boxes)
    ext = boxes[:, 1] - boxes[:, 0]
    pad = DEGENERATE_WIDTH * np.maximum(ext.max(axis=1), 1.0)
    for d in range(3):
        flat = ext[:, d] < pad
        mid = 0.5 * (boxes[:, 0, d] + boxes[:, 1, d])
        boxes[:, 0, d] = np.where(flat, mid - 0.5 * pad, boxes[:, 0, d])
        boxes[:, 1, d] = np.where(flat, mid + 0.5 * pad, boxes[:, 1, d])
    delta = (boxes[:, 1] - boxes[:, 0]).max(axis=1)
    gb = np.stack([boxes[:, 0] - delta[:, None], boxes[:, 1] + delta[:, None]], axis=1)
    g = gauss_legendre(m)
    mm = m * m
    out = np.zeros((n, 6 * mm, 8))
    f = 0
    for axis in range(3):
        u, v = (axis + 1) % 3, (axis + 2) % 3
        lu = gb[:, 1, u] - gb[:, 0, u]
        lv = gb[:, 1, v] - gb[:, 0, v]
        cu = gb[:, 0, u][:, None] + lu[:, None] * g.points[None, :]
        cv = gb[:, 0, v][:, None] + lv[:, None] * g.points[None, :]
        wface = ((lu[:, None] * g.weights[None, :])[:, :, None] * (lv[:, None] * g.weights[None, :])[:, None, :])
        wface = wface.reshape(n, mm)
        for side in (0, 1):
            blk = out[:, f * mm : (f + 1) * mm]
            blk[:, :, axis] = gb[:, side, axis][:, None]
            blk[:, :, u] = np.repeat(cu, m, axis=1)
            blk[:, :, v] = np.tile(cv, (1, m))
            blk[:, :, 3] = np.sqrt(wface)
            blk[:, :, 4 + axis] = 1.0 if side else -1.0
            f += 1
    return out


def green_points_batch_device(boxes, m):
    """green_points_batch with torch on the GPU: the same elementwise IEEE
    operations in the same order (no contractions), so the same bits."""
    t = __import__("torch")
    b = t.as_tensor(np.asarray(boxes, dtype=float).reshape(-1, 2, 3), device="cuda").clone()
    n = b.shape[0]
    ext = b[:, 1] - b[:, 0]
    pad = DEGENERATE_WIDTH * t.clamp(ext.max(dim=1).values, min=1.0)
    for d in range(3):
        flat = ext[:, d] < pad
        mid = 0.5 * (b[:, 0, d] + b[:, 1, d])
        lo = t.where(flat, mid - 0.5 * pad, b[:, 0, d])
        hi = t.where(flat, mid + 0.5 * pad, b[:, 1, d])
        b[:, 0, d], b[:, 1, d] = lo, hi
    delta = (b[:, 1] - b[:, 0]).max(dim=1).values
    gb = t.stack([b[:, 0] - delta[:, None], b[:, 1] + delta[:, None]], dim=1)
    g = gauss_legendre(m)
    gp = t.as_tensor(np.array(g.points), device="cuda")
    gw = t.as_tensor(np.array(g.weights), device="cuda")
    mm = m * m
    out = t.zeros((n, 6 * mm, 8), dtype=t.float64, device="cuda")
    f = 0
    for axis in range(3):
        u, v = (axis + 1) % 3, (axis + 2) % 3
        lu = gb[:, 1, u] - gb[:, 0, u]
        lv = gb[:, 1, v] - gb[:, 0, v]
        cu = gb[:, 0, u][:, None] + lu[:, None] * gp[None, :]
        cv = gb[:, 0, v][:, None] + lv[:, None] * gp[None, :]
        wface = ((lu[:, None] * gw[None, :])[:, :, None] * (lv[:, None] * gw[None, :])[:, None, :]).reshape(n, mm)
        for side in (0, 1):
            blk = out[:, f * mm : (f + 1) * mm]
            blk[:, :, axis] = gb[:, side, axis][:, None]
            blk[:, :, u] = cu.repeat_interleave(m, dim=1)
            blk[:, :, v] = cv.repeat(1, m)
            blk[:, :, 3] = t.sqrt(wface)
            blk[:, :, 4 + axis] = 1.0 if side else -1.0
            f += 1
    return out


_GCA_FLAVOR_CODE = {P0_SLP: 0, P1_DLP: 1, P1_CURL: 2}


def build_basis_device(ctx, tree, flavor, m, eps_aca, q_single=None):
    """GCA basis on the GPU (libh2b h2b_gca_columns + h2b_gca_aca), one tree
    level per call, leaves first.  Same algorithm as build_basis; the Green
    columns are evaluated with device arithmetic, so a pivot can differ from
    the host path where two residual entries tie to rounding (tests measure
    the agreement)."""
    import ctypes

    from . import _lib
    from . import device as D
    from .containers import ClusterBasis

    if flavor not in _GCA_FLAVOR_CODE:
        raise ValueError(f"unknown basis flavor {flavor!r}")
    if q_single is None:
        q_single = max(2, m)
    L_ = _lib.lib()
    pp, Q, lam = ctx.dmesh.panel_points(q_single)
    basis = ClusterBasis(tree)
    depth = tree.depth_of
    k = 6 * m * m
    ncol = 6 * k if flavor == P1_CURL else 2 * k  # curl: three components of both potentials
    for d in range(int(depth.max()), -1, -1):
        level = np.flatnonzero(depth == d)
        rows, boxes = [], []
        for u in level:
            c = tree.nodes[int(u)]
            rows.append(np.asarray(tree.dofs(c), dtype=np.int64) if c.is_leaf
                        else np.concatenate([basis.pivots[ch.uid] for ch in c.children]))
            boxes.append(c.box)
        nr = np.array([len(r) for r in rows], dtype=np.int64)
        ptr = np.zeros(len(level) + 1, dtype=np.int64)
        np.cumsum(nr, out=ptr[1:])
        l_off = ptr[:-1] * ncol
        total = int(ptr[-1]) * ncol
        d_ptr, d_rows = D.dev(ptr), D.dev(np.concatenate(rows), np.int32)
        d_green, d_loff = green_points_batch_device(np.stack(boxes), m), D.dev(l_off)
        b = _lib.GcaBatch(len(level), d_ptr.data_ptr(), d_rows.data_ptr(), k, int(nr.max()), d_green.data_ptr(),
                          d_loff.data_ptr(), ncol)
        Lm, scratch, Vm = D.empty((total,)), D.empty((total,)), D.empty((total,))
        rank = D.empty((len(level),), "int32")
        tau = D.empty((len(level) * ncol,), "int32")
        if flavor == P1_CURL:
            _lib.check(L_.h2b_gca_columns_curl(ctypes.byref(ctx.dmesh.c), pp.data_ptr(), Q, ctx.dmesh.curls().data_ptr(),
                                               ctypes.byref(b), Lm.data_ptr(), D.stream()))
        else:
            _lib.check(L_.h2b_gca_columns(ctypes.byref(ctx.dmesh.c), pp.data_ptr(), Q, lam.data_ptr(),
                                          _GCA_FLAVOR_CODE[flavor], ctypes.byref(b), Lm.data_ptr(), D.stream()))
        _lib.check(L_.h2b_gca_aca(ctypes.byref(b), float(eps_aca), Lm.data_ptr(), scratch.data_ptr(),
                                  rank.data_ptr(), tau.data_ptr(), ncol, Vm.data_ptr(), D.stream()))
        # download only the used part of every V slot (rows x rank of rows x 2k):
        # compact on the device first
        rk = D.host(rank).astype(np.int64)
        tu = D.host(tau).reshape(-1, ncol)
        sizes = nr * rk
        coff = np.zeros(len(level) + 1, dtype=np.int64)
        np.cumsum(sizes, out=coff[1:])
        t = D.torch()
        if coff[-1] > 0:
            sz = t.from_numpy(sizes).cuda()
            starts = t.from_numpy(l_off - coff[:-1]).cuda()
            src = t.arange(int(coff[-1]), device="cuda", dtype=t.int64) + t.repeat_interleave(starts, sz)
            Vh = D.host(Vm[src])
            del src, sz, starts
        else:
            Vh = np.zeros(0)
        del Lm, scratch, Vm
        for i, u in enumerate(level):
            u = int(u)
            c = tree.nodes[u]
            kk = int(rk[i])
            V = Vh[coff[i] : coff[i + 1]].reshape(nr[i], kk)
            piv = rows[i][tu[i, :kk].astype(np.int64)]
            if c.is_leaf:
                basis.V[u] = V
            else:
                off = 0
                for ch in c.children:
                    kc = basis.rank[ch.uid]
                    basis.E[ch.uid] = V[off : off + kc, :]
                    off += kc
            basis.pivots[u] = piv
            basis.rank[u] = kk
    return basis


def build_basis(ctx, tree, flavor, m, eps_aca, q_single=None, threads=1, device=False):
    """Nested cluster basis from the leaves up (gca.py:149-179): at each depth
    all clusters are independent; transfer matrices are the row blocks of the
    parent's interpolation matrix in child order.  device=True builds it on
    the GPU (build_basis_device); the default host path reproduces the
    reference's pivots bit for bit."""
    from threadpoolctl import threadpool_limits

    from .containers import ClusterBasis

    if device:
        return build_basis_device(ctx, tree, flavor, m, eps_aca, q_single)
    if q_single is None:
        q_single = max(2, m)
    basis = ClusterBasis(tree)
    depth = tree.depth_of
    ctx.host_panel_quad(q_single)  # build the shared cache before the pool starts

    def one(u):
        c = tree.nodes[u]
        if c.is_leaf:
            piv, V = gca_leaf(ctx, flavor, tree.dofs(c), c.box, m, eps_aca, q_single)
        else:
            kids = [basis.pivots[ch.uid] for ch in c.children]
            piv, V = gca_nested(ctx, flavor, kids, c.box, m, eps_aca, q_single)
        return u, piv, V

    with threadpool_limits(limits=1, user_api="blas"):
        pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None
        try:
            for d in range(int(depth.max()), -1, -1):
                level = [int(u) for u in np.flatnonzero(depth == d)]
                results = pool.map(one, level) if pool else map(one, level)
                for u, piv, V in results:
                    c = tree.nodes[u]
                    if c.is_leaf:
                        basis.V[u] = V
                    else:
                        off = 0
                        for ch in c.children:
                            k = basis.rank[ch.uid]
                            basis.E[ch.uid] = V[off : off + k, :]
                            off += k
                    basis.pivots[u] = piv
                    basis.rank[u] = len(piv)
        finally:
            if pool:
                pool.shutdown()
    return basis


_FLAVORS = {kernels.SLP: (P0_SLP, P0_SLP), kernels.DLP: (P0_SLP, P1_DLP), kernels.HYP: (P1_CURL, P1_CURL)}


def basis_flavors(kind):
    return _FLAVORS[kind]


def assemble_h2(ctx, kind, block_tree, row_basis, col_basis, q_near, nearfield_cache=None, threads=1,
                q_singular=None):
    """H^2 operator with S_b = G[pivots_t, pivots_s] (regular quadrature at
    q_near, touching pairs rejected) and the dense nearfield (regular order
    q_near, Sauter-Schwab order q_singular, default q_near), all on the GPU."""
    from .containers import H2Matrix, _symmetric_trees, assemble_couplings, assemble_nearfield_device

    qs = q_near if q_singular is None else q_singular
    S = assemble_couplings(ctx, kind, block_tree, row_basis, col_basis, q_near)
    D = assemble_nearfield_device(ctx, kind, block_tree, q_near, qs, cache=nearfield_cache)
    H = H2Matrix.from_device(block_tree, row_basis, col_basis, S, D)
    # single layer, one basis, one tree: couplings and nearfield are assembled
    # as mirrors of each other, so A = A^T entry by entry
    H.symmetric = kind == kernels.SLP and row_basis is col_basis and _symmetric_trees(block_tree)
    return H
