"""Galerkin pair quadrature, restated in numpy (oracle; test infrastructure only).

Reference: /root/reference/pkg/src/h2bem/
  quadrature.triangle_points      quadrature.py:71-87
  quadrature.classify_panel_pair  quadrature.py:90-118
  kernels._classify_pairs         kernels.py:246-254
  kernels.pair_integrals          kernels.py:260-319
  kernels.touching_pairs          kernels.py:333-343
  kernels.panel_pair_matrix       kernels.py:365-434
  kernels.slp_block / dlp_block   kernels.py:437-468
  kernels.triangle_curls          kernels.py:229-239
  kernels.hyp_block               kernels.py:471-511

Distances are direct differences (not the reference's Gram identity); the two
agree to ~1e-12 relative, far inside the 1e-10 bar.
"""

import numpy as np

from .rules import duffy, ss_rule

INV4PI = 1.0 / (4.0 * np.pi)


def panel_points(V, T, A, tris, q):
    """X (P, Q, 3), W (P, Q) incl. 2*area, lam (Q, 3) -- quadrature.py:71-87."""
    pts, w = duffy(q)
    c = V[T[tris]]
    X = c[:, None, 0, :] + pts[None, :, 0, None] * (c[:, None, 1, :] - c[:, None, 0, :]) \
        + pts[None, :, 1, None] * (c[:, None, 2, :] - c[:, None, 0, :])
    W = w[None, :] * (2.0 * A[tris])[:, None]
    lam = np.column_stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]])
    return X, W, lam


def classify(ta, tb, same):
    """Vectorised quadrature.py:90-118 + kernels.py:246-254.
    ta, tb: (B, 3) vertex ids; same: (B,) bool (pa == pb).
    Returns code (B,) (#shared vertices, 3 if same) and perms (B, 3), (B, 3)."""
    B = len(ta)
    eq = ta[:, :, None] == tb[:, None, :]               # (B, 3, 3)
    code = eq.sum(axis=(1, 2))
    code = np.where(same, 3, code)
    pa = np.tile(np.arange(3), (B, 1))
    pb = pa.copy()
    for r in range(B):
        if same[r] or code[r] == 0:
            continue
        a, b = list(ta[r]), list(tb[r])
        sh = sorted(set(a) & set(b))
        ha = [a.index(s) for s in sh]
        hb = [b.index(s) for s in sh]
        pa[r] = ha + [i for i in range(3) if i not in ha]
        pb[r] = hb + [i for i in range(3) if i not in hb]
    return code, pa, pb


def touching_pairs(T, n_vertices):
    """Sorted keys pa*F + pb of all ordered pairs sharing a vertex -- kernels.py:333-343."""
    F = len(T)
    flat = T.reshape(-1)
    order = np.argsort(flat, kind="stable")
    fv = flat[order]
    tri = order // 3
    starts = np.searchsorted(fv, np.arange(n_vertices))
    ends = np.searchsorted(fv, np.arange(n_vertices), side="right")
    keys = []
    for v in range(n_vertices):
        inc = tri[starts[v] : ends[v]]
        keys.append((inc[:, None] * F + inc[None, :]).ravel())
    return np.unique(np.concatenate(keys))


def _chart(c, u, v):
    # chart(u, v) = P1 + u (P2 - P1) + v (P3 - P2)   quadrature.py:193-205
    return c[:, None, 0, :] + u[None, :, None] * (c[:, None, 1, :] - c[:, None, 0, :]) \
        + v[None, :, None] * (c[:, None, 2, :] - c[:, None, 1, :])


def singular_integrals(V, T, N, A, pa, pb, kind, q, chunk=200_000):
    """Regularised pair integrals -- kernels.py:260-319 (pair_integrals): any
    case, disjoint pairs by the tensor rule of quadrature.py:171-180.
    SLP: (B,); edge/vertex averaged with the orientation-swapped rule.
    DLP: (B, 3) per ORIGINAL local vertex of the column panel; identical -> 0."""
    pa = np.asarray(pa, dtype=np.int64)
    pb = np.asarray(pb, dtype=np.int64)
    B = len(pa)
    out = np.zeros((B, 3)) if kind == "dlp" else np.zeros(B)
    if B == 0:
        return out
    code, perm_a, perm_b = classify(T[pa], T[pb], pa == pb)
    for c, case in ((3, "identical"), (2, "edge"), (1, "vertex"), (0, "disjoint")):
        idx = np.flatnonzero(code == c)
        if len(idx) == 0 or (kind == "dlp" and case == "identical"):
            continue
        P, w = ss_rule(case, q)
        step = max(1, chunk // len(w))
        for lo in range(0, len(idx), step):
            sub = idx[lo : lo + step]
            ca = V[np.take_along_axis(T[pa[sub]], perm_a[sub], axis=1)]
            cb = V[np.take_along_axis(T[pb[sub]], perm_b[sub], axis=1)]
            scale = 4.0 * A[pa[sub]] * A[pb[sub]]
            X = _chart(ca, P[:, 0], P[:, 1])
            Y = _chart(cb, P[:, 2], P[:, 3])
            d = X - Y
            r = np.sqrt(np.einsum("bnk,bnk->bn", d, d))
            if kind == "slp":
                val = (INV4PI / r) @ w
                if case in ("edge", "vertex"):
                    d2 = _chart(ca, P[:, 2], P[:, 3]) - _chart(cb, P[:, 0], P[:, 1])
                    r2 = np.sqrt(np.einsum("bnk,bnk->bn", d2, d2))
                    val = 0.5 * (val + (INV4PI / r2) @ w)
                out[sub] = val * scale
            else:
                nb = N[pb[sub]]
                k = INV4PI * np.einsum("bnk,bk->bn", d, nb) / r**3
                lam = np.column_stack([1.0 - P[:, 2], P[:, 2] - P[:, 3], P[:, 3]])
                vals = (k * w[None, :]) @ lam * scale[:, None]
                res = np.zeros_like(vals)
                np.put_along_axis(res, perm_b[sub], vals, axis=1)
                out[sub] = res
    return out


class Table:
    """Singular values of all touching pairs, keyed like the reference's
    SingularTable (kernels.py:346-362)."""

    def __init__(self, V, T, N, A, kind, q):
        self.F = len(T)
        self.keys = touching_pairs(T, len(V))
        self.values = singular_integrals(V, T, N, A, self.keys // self.F, self.keys % self.F, kind, q)

    def lookup(self, pa, pb):
        key = np.asarray(pa) * self.F + np.asarray(pb)
        pos = np.searchsorted(self.keys, key)
        if not np.array_equal(self.keys[np.minimum(pos, len(self.keys) - 1)], key):
            raise KeyError("panel pair missing from the singular table")
        return self.values[pos]


def pair_matrix(V, T, N, A, rows, cols, kind, q, table=None):
    """All-pairs panel integrals -- kernels.py:365-434.  SLP (na, nb); DLP
    (na, nb, 3) per local vertex of the column panel.  Touching pairs take the
    table value (or raise when table is None and require_disjoint)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    Xa, Wa, _ = panel_points(V, T, A, rows, q)
    Xb, Wb, lam = panel_points(V, T, A, cols, q)
    d = Xa[:, :, None, None, :] - Xb[None, None, :, :, :]          # (na, Q, nb, Q, 3)
    r = np.sqrt(np.einsum("aibjk,aibjk->aibj", d, d))
    with np.errstate(divide="ignore", invalid="ignore"):  # touching pairs are overwritten below
        if kind == "slp":
            k = INV4PI / r
            out = np.einsum("ai,aibj,bj->ab", Wa, k, Wb)
        else:
            nb = N[cols]
            k = INV4PI * np.einsum("aibjk,bk->aibj", d, nb) / r**3
            out = np.einsum("ai,aibj,bj,jl->abl", Wa, k, Wb, lam)
    ta, tb = T[rows], T[cols]
    hit = (ta[:, None, :, None] == tb[None, :, None, :]).any(axis=(2, 3))
    sa, sb = np.nonzero(hit)
    if len(sa):
        if table is None:
            raise ValueError("expected well-separated panels, found touching pair")
        out[sa, sb] = table.lookup(rows[sa], cols[sb])
    return out


def slp_block(V, T, N, A, rows, cols, q, table=None):
    """kernels.py:437-445."""
    return pair_matrix(V, T, N, A, rows, cols, "slp", q, table)


def dlp_block(V, T, N, A, vt_ptr, vt_idx, rows, cols, q, table=None):
    """P0 rows x P1 vertex columns via incident panels -- kernels.py:448-468."""
    cols = np.asarray(cols, dtype=np.int64)
    pans = np.unique(np.concatenate([vt_idx[vt_ptr[v] : vt_ptr[v + 1]] for v in cols]))
    vals = pair_matrix(V, T, N, A, rows, pans, "dlp", q, table)
    pos = -np.ones(len(V), dtype=np.int64)
    pos[cols] = np.arange(len(cols))
    block = np.zeros((len(rows), len(cols)))
    cj = pos[T[pans]]
    for l in range(3):
        keep = np.flatnonzero(cj[:, l] >= 0)
        np.add.at(block.T, cj[keep, l], vals[:, keep, l].T)
    return block


def triangle_curls(V, T, A):
    """Surface curl of each P1 hat per panel, (F, 3, 3) -- kernels.py:229-239:
    curls[f, l] = (V_{l+1} - V_{l+2}) / (2 area_f)."""
    c = V[T]
    out = np.empty_like(c)
    for l in range(3):
        out[:, l, :] = c[:, (l + 1) % 3, :] - c[:, (l + 2) % 3, :]
    return out / (2.0 * A)[:, None, None]


def hyp_block(V, T, N, A, vt_ptr, vt_idx, rows, cols, q, table=None, curls=None):
    """Hypersingular P1 x P1 block through the surface-curl representation --
    kernels.py:471-511: w_ij = sum over incident panel pairs (a, b) of
    <curl_a(i), curl_b(j)> times the single-layer panel-pair integral."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if curls is None:
        curls = triangle_curls(V, T, A)
    pa = np.unique(np.concatenate([vt_idx[vt_ptr[v] : vt_ptr[v + 1]] for v in rows]))
    pb = np.unique(np.concatenate([vt_idx[vt_ptr[v] : vt_ptr[v + 1]] for v in cols]))
    vals = pair_matrix(V, T, N, A, pa, pb, "slp", q, table)
    rpos = -np.ones(len(V), dtype=np.int64)
    rpos[rows] = np.arange(len(rows))
    cpos = -np.ones(len(V), dtype=np.int64)
    cpos[cols] = np.arange(len(cols))
    ri, cj = rpos[T[pa]], cpos[T[pb]]
    ca, cb = curls[pa], curls[pb]
    block = np.zeros((len(rows), len(cols)))
    for la in range(3):
        ka = ri[:, la] >= 0
        if not ka.any():
            continue
        for lb in range(3):
            kb = cj[:, lb] >= 0
            if not kb.any():
                continue
            dots = ca[ka, la, :] @ cb[kb, lb, :].T
            np.add.at(block, (ri[ka, la][:, None], cj[kb, lb][None, :]), vals[np.ix_(ka, kb)] * dots)
    return block
