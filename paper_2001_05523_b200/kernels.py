"""Galerkin quadrature on the GPU.  API of h2bem.kernels (kernels.py:1-527)
for the operator kinds on the hot path (SLP, DLP).

Host side of the boundary: uploads the mesh once, builds the touching-pair
table (h2b_touch_count/fill: every ordered panel pair sharing a vertex with
its Sauter-Schwab case and vertex permutations), evaluates the singular
integrals of all touching pairs (h2b_singular) and packs dense-block jobs for
the pair-block kernels (h2b_pair_blocks_slp / _dlp).  Regular pairs use the
q_reg^2-point Duffy tensor rule per panel; touching pairs take the singular
table value (kernels.py:429-433), or make the call fail when the caller
requires disjoint panels (coupling matrices, kernels.py:441-444, 455-458).
"""

import ctypes

import numpy as np

from . import _lib
from . import device as D
from . import quadrature as quad

FOUR_PI = 4.0 * np.pi

SLP = "slp"
DLP = "dlp"
HYP = "hyp"

K_VALUE = "value"
K_DN_Z = "dn_z"
K_DN_X = "dn_x"
K_DN_X_DN_Z = "dn_x_dn_z"

TILE = 64           # max rows/cols of one device job (kernel tile)
DLP_MAX_PANELS = 128

_KIND_CODE = {SLP: _lib.H2B_SLP, DLP: _lib.H2B_DLP}


def kind_code(kind):
    if kind not in _KIND_CODE:
        raise ValueError(f"unknown operator kind {kind!r}")
    return _KIND_CODE[kind]


class DeviceMesh:
    """Mesh arrays resident in HBM + the ctypes descriptor."""

    def __init__(self, mesh):
        self.mesh = mesh
        ptr, idx = mesh.vertex_triangle_csr()
        self.vertices = D.dev(mesh.vertices, np.float64)
        self.triangles = D.dev(mesh.triangles, np.int32)
        self.normals = D.dev(mesh.normals, np.float64)
        self.areas = D.dev(mesh.areas, np.float64)
        self.vt_ptr = D.dev(ptr, np.int64)
        self.vt_idx = D.dev(idx, np.int32)
        self.c = _lib.Mesh(mesh.n_vertices, mesh.n_triangles, self.vertices.data_ptr(), self.triangles.data_ptr(),
                           self.normals.data_ptr(), self.areas.data_ptr(), self.vt_ptr.data_ptr(),
                           self.vt_idx.data_ptr())
        self._pp = {}
        self._touch = None

    def panel_points(self, q):
        """(4, F, q^2) device tensor: x, y, z, weight*2A per rule point."""
        if q not in self._pp:
            pts, w = quad.triangle_rule(q)
            Q = len(w)
            out = D.empty((4, self.mesh.n_triangles, Q))
            rxy, rw = D.dev(pts), D.dev(w)
            _lib.check(_lib.lib().h2b_panel_points(ctypes.byref(self.c), rxy.data_ptr(), rw.data_ptr(), Q,
                                                   out.data_ptr(), D.stream()))
            lam = np.column_stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]])
            self._pp[q] = (out, Q, D.dev(lam))
        return self._pp[q]

    def touch(self):
        if self._touch is None:
            self._touch = TouchTable(self)
        return self._touch

    def curls(self):
        """(3F, 3) device copy of triangle_curls (hypersingular blocks)."""
        if "curls" not in self._pp:
            self._pp["curls"] = D.dev(np.ascontiguousarray(triangle_curls(self.mesh).reshape(-1, 3)))
        return self._pp["curls"]


class TouchTable:
    """All ordered touching panel pairs (sharing >= 1 vertex, incl. identical),
    CSR by row panel with ascending columns -- the reference's sorted keys
    pa * F + pb (kernels.py:333-343) -- plus case codes and permutations."""

    def __init__(self, dmesh):
        L = _lib.lib()
        F = dmesh.mesh.n_triangles
        self.dmesh = dmesh
        self.row_ptr = D.empty((F + 1,), "int64")
        counts = np.zeros(4, dtype=np.int64)
        _lib.check(L.h2b_touch_count(ctypes.byref(dmesh.c), self.row_ptr.data_ptr(), _lib.ptr(counts), D.stream()))
        n = int(counts[3])
        self.n_pairs = n
        self.case_counts = counts[:3].copy()  # identical, edge, vertex
        self.col = D.empty((max(n, 1),), "int32")
        self.info = D.empty((max(n, 1),), "int32")
        self.case_list = D.empty((max(n, 1),), "int32")
        _lib.check(L.h2b_touch_fill(ctypes.byref(dmesh.c), self.row_ptr.data_ptr(), _lib.ptr(counts),
                                    self.col.data_ptr(), self.info.data_ptr(), self.case_list.data_ptr(),
                                    D.stream()))
        self.case_off = np.array([0, counts[0], counts[0] + counts[1], n], dtype=np.int64)
        self.c = _lib.Touch(F, n, self.row_ptr.data_ptr(), self.col.data_ptr(), self.info.data_ptr(),
                            self.case_list.data_ptr(), _lib.ptr(self.case_off), None, None)
        self.half_list = None

    def ensure_half(self):
        """Unordered-pair list (a < b) for the symmetric single-layer table."""
        if self.half_list is None:
            counts = self.case_counts
            nh = int(counts[0] + (counts[1] + counts[2]) // 2)
            self.half_list = D.empty((max(nh, 1),), "int32")
            self.half_off = np.zeros(4, dtype=np.int64)
            _lib.check(_lib.lib().h2b_touch_half(ctypes.byref(self.c), self.half_list.data_ptr(),
                                                 _lib.ptr(self.half_off), D.stream()))
            self.c.d_half_list = self.half_list.data_ptr()
            self.c.h_half_off = _lib.ptr(self.half_off)
        return self.half_list

    def subset(self, own_panels, half):
        """A descriptor whose pair lists keep only the pairs touching an owned
        panel (half: the unordered list, either panel owned; else the ordered
        list, row panel owned), case segments preserved.  Cached per mask."""
        t = D.torch()
        key = (bytes(np.packbits(np.asarray(own_panels, dtype=bool))), half)
        if getattr(self, "_subset", None) is not None and self._subset[0] == key:
            return self._subset[1]
        own = t.from_numpy(np.ascontiguousarray(own_panels, dtype=bool)).cuda()
        F = self.dmesh.mesh.n_triangles
        rows = t.repeat_interleave(t.arange(F, device="cuda", dtype=t.int32), t.diff(self.row_ptr))
        lst, off = (self.half_list, self.half_off) if half else (self.case_list, self.case_off)
        parts, new_off = [], [0]
        for k in range(3):
            seg = lst[int(off[k]) : int(off[k + 1])].long()
            m = own[rows[seg].long()]
            if half:
                m = m | own[self.col[seg].long()]
            parts.append(seg[m].to(t.int32))
            new_off.append(new_off[-1] + int(parts[-1].numel()))
        sub = t.cat(parts) if new_off[-1] else t.zeros(1, dtype=t.int32, device="cuda")
        sub_off = np.array(new_off, dtype=np.int64)
        c = _lib.Touch(self.c.n_panels, self.c.n_pairs, self.c.d_row_ptr, self.c.d_col, self.c.d_info,
                       sub.data_ptr() if not half else self.c.d_case_list,
                       _lib.ptr(sub_off) if not half else self.c.h_case_off,
                       sub.data_ptr() if half else None, _lib.ptr(sub_off) if half else None)
        self._subset = (key, c, sub, sub_off)
        return c

    def keys(self):
        """Sorted int64 keys pa * F + pb (reference SingularTable.keys)."""
        F = self.dmesh.mesh.n_triangles
        rp = D.host(self.row_ptr)
        rows = np.repeat(np.arange(F, dtype=np.int64), np.diff(rp))
        return rows * F + D.host(self.col[: self.n_pairs]).astype(np.int64)

    def codes_perms(self):
        """(codes, perms (n, 6)) decoded from the device info words."""
        info = D.host(self.info[: self.n_pairs]).astype(np.int64)
        perms = np.stack([(info >> s) & 3 for s in (2, 4, 6, 8, 10, 12)], axis=1)
        return info & 3, perms


class SingularTable:
    """Sauter-Schwab integrals of every touching pair at order q, on the device
    (reference: kernels.SingularTable, kernels.py:346-362)."""

    def __init__(self, mesh, kind, q, vertex_tris=None, compute=True):
        """mesh: the host SurfaceMesh (reference signature) or its DeviceMesh."""
        if kind not in (SLP, DLP):
            raise ValueError(f"unknown operator kind {kind!r}")
        dmesh = device_mesh(mesh)
        self.kind = kind
        self.q = q
        self.dmesh = dmesh
        self.touch = dmesh.touch()
        n = self.touch.n_pairs
        width = 3 if kind == DLP else 1
        self.values_dev = D.zeros((max(n, 1) * width,))
        self.rules = (_lib.Rule * 3)()
        self._keep = []
        for i, case in enumerate((quad.IDENTICAL, quad.SHARED_EDGE, quad.SHARED_VERTEX)):
            r = quad.sauter_schwab_rule(case, q)
            p, w = D.dev(r.points), D.dev(r.weights)
            self._keep += [p, w]
            self.rules[i] = _lib.Rule(len(r.weights), p.data_ptr(), w.data_ptr())
        self.n = dmesh.mesh.n_triangles
        self._keys = None
        if compute:
            self.compute()

    def compute(self, own_panels=None):
        """(Re)evaluate the touching pairs on the device (stream-ordered).
        Single layer: one evaluation per unordered pair (symmetric table).
        own_panels (bool per panel, row sharding): only the pairs this rank's
        blocks look up -- single layer: every unordered pair with an owned
        panel (both ordered entries are written); double layer: the ordered
        pairs whose row panel is owned.  Other entries are left untouched."""
        if self.kind == SLP:
            self.touch.ensure_half()
        c = self.touch.c
        if own_panels is not None:
            c = self.touch.subset(own_panels, half=self.kind == SLP)
        _lib.check(_lib.lib().h2b_singular(ctypes.byref(self.dmesh.c), ctypes.byref(c),
                                           kind_code(self.kind), self.rules, self.values_dev.data_ptr(),
                                           D.stream()))

    @property
    def keys(self):
        if self._keys is None:
            self._keys = self.touch.keys()
        return self._keys

    @property
    def values(self):
        v = D.host(self.values_dev)[: self.touch.n_pairs * (3 if self.kind == DLP else 1)]
        return v.reshape(-1, 3) if self.kind == DLP else v

    def lookup(self, pa, pb):
        key = np.asarray(pa, dtype=np.int64) * self.n + np.asarray(pb, dtype=np.int64)
        pos = np.searchsorted(self.keys, key)
        safe = np.minimum(pos, len(self.keys) - 1)
        if not np.array_equal(self.keys[safe], key):
            raise KeyError("panel pair missing from the singular table")
        return self.values[safe]


# ---------------------------------------------------------------------------
# job packing

def _as_job8(jobs):
    jobs = np.asarray(jobs, dtype=np.int64)
    if jobs.size == 0:
        return np.zeros((0, 8), dtype=np.int64)
    if jobs.ndim == 2 and jobs.shape[1] == 8:
        return jobs
    jobs = jobs.reshape(-1, 6)
    pad = np.zeros((len(jobs), 2), dtype=np.int64)
    pad[:, 0] = -1
    return np.hstack([jobs, pad])


def tile_jobs(jobs):
    """Split (row_off, nr, col_off, nc, out_off, ld[, mirror_off, mirror_ld])
    jobs into <= TILE x TILE tiles (8-word jobs out).  A mirrored tile also
    writes its transpose at mirror_off; a diagonal job (mirror_off == out_off)
    keeps its upper-triangle tiles only."""
    jobs = _as_job8(jobs)
    if len(jobs) == 0 or (jobs[:, 1].max() <= TILE and jobs[:, 3].max() <= TILE):
        return jobs
    out = []
    for r0, nr, c0, nc, o, ld, mo, mld in jobs:
        diag = mo == o and mo >= 0
        for i in range(0, max(nr, 1), TILE):
            for j in range(0, max(nc, 1), TILE):
                if diag and i > j:
                    continue
                m = mo + j * mld + i if mo >= 0 else -1
                oo = o + i * ld + j if o >= 0 else -1
                out.append((r0 + i, min(TILE, nr - i), c0 + j, min(TILE, nc - j), oo, ld, m, mld))
    return np.array(out, dtype=np.int64).reshape(-1, 8)


def block_partners(uids):
    """For every block (t, s) of a block list (n, 2), the index of block (s, t)
    in the same list, or -1; a diagonal block is its own partner.  Native
    (h2b_block_partners); same output as _block_partners_py."""
    uids = np.ascontiguousarray(uids, dtype=np.int64).reshape(-1, 2)
    out = np.empty(len(uids), dtype=np.int64)
    _lib.check(_lib.lib().h2b_block_partners(len(uids), _lib.ptr(uids), _lib.ptr(out)))
    return out


def block_jobs(uids, row_off, row_cnt, col_off, col_cnt, blk_off, blk_ld, partner=None):
    """(m, 8) pair-block jobs of the blocks (t, s) = uids[i]: rows
    row_off[t] .. + row_cnt[t], columns col_off[s] .. + col_cnt[s], stored at
    blk_off[i] / blk_ld[i].  With `partner` (block_partners of uids; symmetric
    single layer) one job per block pair that also writes the mirror -- the
    output of mirror_jobs on the stacked job columns, built in one native pass
    (h2b_block_jobs)."""
    c = lambda a: np.ascontiguousarray(a, dtype=np.int64)
    uids = c(uids).reshape(-1, 2)
    n = len(uids)
    arrs = [c(a) for a in (row_off, row_cnt, col_off, col_cnt, blk_off, blk_ld)]
    part = c(partner) if partner is not None else None
    jobs = np.empty((n, 8), dtype=np.int64)
    m = np.zeros(1, dtype=np.int64)
    _lib.check(_lib.lib().h2b_block_jobs(n, _lib.ptr(uids), *(_lib.ptr(a) for a in arrs), int(part is not None),
                                         _lib.ptr(part), _lib.ptr(jobs), _lib.ptr(m)))
    return jobs[: int(m[0])]


def _block_partners_py(uids):
    """numpy restatement of block_partners (tests)."""
    uids = np.asarray(uids, dtype=np.int64).reshape(-1, 2)
    n = len(uids)
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    key = uids[:, 0] * (uids.max() + 1) + uids[:, 1]
    tkey = uids[:, 1] * (uids.max() + 1) + uids[:, 0]
    order = np.argsort(key, kind="stable")
    pos = np.minimum(np.searchsorted(key[order], tkey), n - 1)
    return np.where(key[order][pos] == tkey, order[pos], -1)


def mirror_jobs(jobs, uids, partner=None):
    """Symmetric single-layer blocks (same tree and basis on both sides, so
    block (s, t) = block (t, s)^T): keep one job per block pair {(t, s), (s, t)}
    with the other written as its mirror; a diagonal block (t, t) keeps its
    upper triangle.  jobs: (n, 6) in the order of uids (n, 2)."""
    jobs = np.asarray(jobs, dtype=np.int64).reshape(-1, 6)
    uids = np.asarray(uids, dtype=np.int64).reshape(-1, 2)
    out = _as_job8(jobs)
    if len(jobs) == 0:
        return out
    if partner is None:
        partner = block_partners(uids)
    keep = (partner < 0) | (uids[:, 0] <= uids[:, 1])
    m = keep & (partner >= 0)
    out[m, 6] = jobs[partner[m], 4]
    out[m, 7] = jobs[partner[m], 5]
    return out[keep]


def mirror_jobs_owned(jobs, uids, dst_off, dst_ld, partner=None):
    """The jobs of mirror_jobs restricted to the blocks one rank stores (row
    sharding).  jobs (n, 6) / uids (n, 2): the FULL block list (integration
    geometry of every block); dst_off / dst_ld (n,): where this rank stores
    block i, or -1.  Every kept job integrates its block pair in the same
    orientation as the single-GPU job list, so the stored values are the same
    bits; a job whose direct block belongs to another rank becomes
    mirror-only (out_off = -1)."""
    jobs = np.asarray(jobs, dtype=np.int64).reshape(-1, 6)
    uids = np.asarray(uids, dtype=np.int64).reshape(-1, 2)
    if len(jobs) == 0:
        return np.zeros((0, 8), dtype=np.int64)
    if partner is None:
        partner = block_partners(uids)
    keep = (partner < 0) | (uids[:, 0] <= uids[:, 1])
    out = _as_job8(jobs)
    out[:, 4] = dst_off
    out[:, 5] = dst_ld
    m = keep & (partner >= 0)
    pm = partner[m]
    out[m, 6] = dst_off[pm]
    out[m, 7] = dst_ld[pm]
    out = out[keep]
    return out[(out[:, 4] >= 0) | (out[:, 6] >= 0)]


class SlpJobs:
    """SLP pair-block jobs resident on the device (tiled to TILE x TILE)."""

    def __init__(self, dmesh, q, jobs, row_idx, col_idx):
        self.dmesh = dmesh
        self.q = q
        self.jobs = tile_jobs(jobs)
        self.n = len(self.jobs)
        if self.n:
            tri = self.jobs[:, 6] == self.jobs[:, 4]
            full = self.jobs[:, 1] * self.jobs[:, 3]
            mult = np.where(self.jobs[:, 6] >= 0, 2, 1)
            # pairs integrated / pairs of the matrix written
            self.evaluated = int(np.where(tri, self.jobs[:, 3] * (self.jobs[:, 3] + 1) // 2, full).sum())
            self.pairs = int(np.where(tri, full, full * mult).sum())
        else:
            self.evaluated = self.pairs = 0
        if self.n == 0:
            return
        self.pp, self.Q, _ = dmesh.panel_points(q)
        self.dj = D.dev(self.jobs, np.int64)
        self.ri = row_idx if not isinstance(row_idx, np.ndarray) else D.dev(row_idx, np.int32)
        self.ci = col_idx if not isinstance(col_idx, np.ndarray) else D.dev(col_idx, np.int32)
        self.c = _lib.Jobs(self.n, self.dj.data_ptr(), self.ri.data_ptr(), self.ci.data_ptr())

    def run(self, table, out):
        if self.n == 0:
            return
        tptr = ctypes.byref(table.touch.c) if table is not None else None
        tv = table.values_dev.data_ptr() if table is not None else None
        _lib.check(_lib.lib().h2b_pair_blocks_slp(ctypes.byref(self.dmesh.c), self.pp.data_ptr(), self.Q,
                                                  ctypes.byref(self.c), tptr, tv, out.data_ptr(), D.stream()))


def run_slp_jobs(dmesh, q, jobs, row_idx, col_idx, table, out):
    """Device SLP pair blocks into `out` (device float64)."""
    SlpJobs(dmesh, q, jobs, row_idx, col_idx).run(table, out)


def build_dlp_jobs(mesh, blocks):
    """DLP jobs for dense blocks (row panels, column vertices, out_off, ld),
    built natively (h2b_dlp_jobs_build); same output as _build_dlp_jobs_py."""
    blocks = list(blocks)
    if not blocks:
        return None
    vptr, vidx = mesh.vertex_triangle_csr()
    tris = np.ascontiguousarray(mesh.triangles, dtype=np.int64)
    rows = [np.asarray(b[0], dtype=np.int64) for b in blocks]
    cols = [np.asarray(b[1], dtype=np.int64) for b in blocks]
    row_ptr = np.zeros(len(blocks) + 1, dtype=np.int64)
    np.cumsum([len(r) for r in rows], out=row_ptr[1:])
    col_ptr = np.zeros(len(blocks) + 1, dtype=np.int64)
    np.cumsum([len(c) for c in cols], out=col_ptr[1:])
    R = np.concatenate(rows) if row_ptr[-1] else np.zeros(1, dtype=np.int64)
    Cc = np.concatenate(cols) if col_ptr[-1] else np.zeros(1, dtype=np.int64)
    off = np.array([b[2] for b in blocks], dtype=np.int64)
    ld = np.array([b[3] for b in blocks], dtype=np.int64)
    vptr = np.ascontiguousarray(vptr, dtype=np.int64)
    vidx = np.ascontiguousarray(vidx, dtype=np.int64)
    L = _lib.lib()
    h = ctypes.c_void_p()
    _lib.check(L.h2b_dlp_jobs_build(mesh.n_vertices, _lib.ptr(vptr), _lib.ptr(vidx), _lib.ptr(tris), len(blocks),
                                    _lib.ptr(row_ptr), _lib.ptr(R), _lib.ptr(col_ptr), _lib.ptr(Cc), _lib.ptr(off),
                                    _lib.ptr(ld), ctypes.byref(h)))
    try:
        sz = np.zeros(6, dtype=np.int64)
        _lib.check(L.h2b_dlp_jobs_sizes(h, _lib.ptr(sz)))
        if sz[0] == 0:
            return None
        out = dict(jobs=np.empty((sz[0], 8), dtype=np.int64), row_idx=np.empty(sz[1], dtype=np.int32),
                   pan_idx=np.empty(sz[2], dtype=np.int32), inc_ptr=np.empty(sz[3], dtype=np.int32),
                   inc=np.empty(max(sz[4], 1), dtype=np.int32), inc_base=np.empty(sz[5], dtype=np.int64))
        if sz[4] == 0:
            out["inc"][:] = 0
        _lib.check(L.h2b_dlp_jobs_copy(h, *(_lib.ptr(out[k]) for k in
                                            ("jobs", "row_idx", "pan_idx", "inc_ptr", "inc", "inc_base"))))
        return out
    finally:
        L.h2b_dlp_jobs_free(h)


def _build_dlp_jobs_py(mesh, blocks):
    """DLP jobs for dense blocks (row panels, column vertices, out_off, ld):
    the column-panel set of each job is the sorted union of the panels incident
    to its column vertices (kernels.py:454), tiled so that a job holds at most
    TILE rows, TILE columns and DLP_MAX_PANELS panels; the incidence CSR lists,
    per column, (local panel, local vertex) contributions l-major then by
    panel -- the accumulation order of np.add.at in kernels.dlp_block."""
    vptr, vidx = mesh.vertex_triangle_csr()
    tris = mesh.triangles
    jobs, row_idx, pan_idx, inc_ptr, inc, inc_base = [], [], [], [], [], []
    nrow = npan = ninc = nptr = 0
    for rows, cols, out_off, ld in blocks:
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        # column tiles bounded by the panel budget
        c0 = 0
        while c0 < len(cols):
            c1 = min(len(cols), c0 + TILE)
            while True:
                sel = cols[c0:c1]
                pans = np.unique(np.concatenate([vidx[vptr[v] : vptr[v + 1]] for v in sel]))
                if len(pans) <= DLP_MAX_PANELS or c1 - c0 == 1:
                    break
                c1 = c0 + max(1, (c1 - c0) // 2)
            if len(pans) > DLP_MAX_PANELS:
                raise ValueError("vertex valence too large for the DLP panel tile")
            pos = {int(v): i for i, v in enumerate(sel)}
            trip = []
            t3 = tris[pans]
            for l in range(3):
                for p in range(len(pans)):
                    c = pos.get(int(t3[p, l]))
                    if c is not None:
                        trip.append((c, l, p))
            trip.sort()
            counts = np.zeros(len(sel) + 1, dtype=np.int64)
            for c, _, _ in trip:
                counts[c + 1] += 1
            cptr = np.cumsum(counts) + ninc
            codes = [(p << 2) | l for _, l, p in trip]
            for r0 in range(0, len(rows), TILE):
                r1 = min(len(rows), r0 + TILE)
                jobs.append((nrow, r1 - r0, npan, len(pans), c0, len(sel), out_off + r0 * ld + c0, ld))
                row_idx.append(rows[r0:r1])
                nrow += r1 - r0
                inc_base.append(nptr)
            pan_idx.append(pans)
            npan += len(pans)
            inc_ptr.append(cptr)
            nptr += len(cptr)
            inc.extend(codes)
            ninc += len(codes)
            c0 = c1
    if not jobs:
        return None
    # jobs of one column tile share pan/inc data; all row tiles point at it
    return dict(
        jobs=np.array(jobs, dtype=np.int64),
        row_idx=np.concatenate(row_idx).astype(np.int32),
        pan_idx=np.concatenate(pan_idx).astype(np.int32),
        inc_ptr=np.concatenate(inc_ptr).astype(np.int32),
        inc=np.array(inc, dtype=np.int32) if inc else np.zeros(1, dtype=np.int32),
        inc_base=np.array(inc_base, dtype=np.int64),
    )


def run_dlp_jobs(dmesh, q, packed, table, out):
    if packed is None:
        return
    pp, Q, lam = dmesh.panel_points(q)
    t = {k: D.dev(v) for k, v in packed.items()}
    cj = _lib.DlpJobs(len(packed["jobs"]), t["jobs"].data_ptr(), t["row_idx"].data_ptr(), t["pan_idx"].data_ptr(),
                      t["inc_ptr"].data_ptr(), t["inc"].data_ptr(), t["inc_base"].data_ptr())
    tptr = ctypes.byref(table.touch.c) if table is not None else None
    tv = table.values_dev.data_ptr() if table is not None else None
    _lib.check(_lib.lib().h2b_pair_blocks_dlp(ctypes.byref(dmesh.c), pp.data_ptr(), lam.data_ptr(), Q,
                                              ctypes.byref(cj), tptr, tv, out.data_ptr(), D.stream()))


def touching_pairs(mesh):
    """Sorted keys pa * F + pb of all touching ordered pairs (device classifier)."""
    return DeviceMesh(mesh).touch().keys()


# ---------------------------------------------------------------------------
# reference kernel-level entry points (kernels.py:260-319, 346-362, 365-468):
# same names and arguments, computed on the device.  `mesh` is the host
# SurfaceMesh (its device copy is cached); `pq` (host panel points) is
# accepted for signature compatibility -- the device builds its own points at
# order q, bit-identical to quadrature.triangle_points -- and `singular` is a
# SingularTable of this module (AssemblyContext.singular_table).

def device_mesh(mesh):
    """The DeviceMesh of a host mesh, cached on the mesh object (its lifetime
    follows the mesh), or the DeviceMesh itself."""
    if isinstance(mesh, DeviceMesh):
        return mesh
    dm = getattr(mesh, "_h2b_device_mesh", None)
    if dm is None:
        dm = DeviceMesh(mesh)
        mesh._h2b_device_mesh = dm
    return dm


def _table_for(dm, kind, q, singular):
    if singular is None:
        # the reference integrates touching pairs on the fly at order q
        # (pair_integrals); the device table of the mesh at order q holds the
        # same values
        key = ("table", kind, q)
        if key not in dm._pp:
            dm._pp[key] = SingularTable(dm, kind, q)
        return dm._pp[key]
    if not isinstance(singular, SingularTable):
        raise ValueError("singular must be a device SingularTable (AssemblyContext.singular_table)")
    if singular.kind != kind:
        raise ValueError(f"singular table of kind {singular.kind!r} used for {kind!r}")
    return singular


def pair_integrals(mesh, pa, pb, kind, q, chunk=None):
    """Galerkin double integrals over panel pairs (pa[i], pb[i]) with the
    regularising rule of each pair's case (kernels.py:260-319): SLP (B,),
    DLP (B, 3) per original local vertex of the column panel (identical pairs
    0).  Any case, disjoint included (tensor rule through the charts)."""
    if kind not in (SLP, DLP):
        raise ValueError(f"unknown operator kind {kind!r}")
    dm = device_mesh(mesh)
    pa = np.asarray(pa, dtype=np.int64)
    pb = np.asarray(pb, dtype=np.int64)
    B = len(pa)
    if len(pb) != B:
        raise ValueError("pa and pb differ in length")
    width = 3 if kind == DLP else 1
    if B == 0:
        return np.zeros((0, 3)) if kind == DLP else np.zeros(0)
    F = dm.mesh.n_triangles
    if pa.min() < 0 or pb.min() < 0 or pa.max() >= F or pb.max() >= F:
        raise ValueError("panel index out of range")
    rules = (_lib.Rule * 4)()
    keep = []
    for i, case in enumerate((quad.IDENTICAL, quad.SHARED_EDGE, quad.SHARED_VERTEX, quad.DISJOINT)):
        r = quad.sauter_schwab_rule(case, q)
        p, w = D.dev(r.points), D.dev(r.weights)
        keep += [p, w]
        rules[i] = _lib.Rule(len(r.weights), p.data_ptr(), w.data_ptr())
    da, db = D.dev(pa, np.int32), D.dev(pb, np.int32)
    out = D.empty((B * width,))
    _lib.check(_lib.lib().h2b_pair_integrals(ctypes.byref(dm.c), B, da.data_ptr(), db.data_ptr(), kind_code(kind),
                                             rules, out.data_ptr(), D.stream()))
    h = D.host(out)
    return h.reshape(B, 3) if kind == DLP else h


def _dlp_pair_jobs(na, nb):
    """DLP jobs whose output columns are (column panel, local vertex) pairs,
    one contribution each: the kernel's vertex scatter becomes the identity
    and out (na x 3 nb) holds panel_pair_matrix(..., DLP) (na, nb, 3)."""
    per = TILE // 3
    jobs, row_idx, pan_idx, inc_ptr, inc, inc_base = [], [], [], [], [], []
    nptr = ninc = 0
    for p0 in range(0, nb, per):
        p1 = min(nb, p0 + per)
        w = p1 - p0
        pan_idx.append(np.arange(p0, p1))
        codes = [(p << 2) | l for p in range(w) for l in range(3)]
        ptr0 = nptr
        inc_ptr.append(ninc + np.arange(3 * w + 1))
        nptr += 3 * w + 1
        inc.extend(codes)
        ninc += len(codes)
        for r0 in range(0, na, TILE):
            r1 = min(na, r0 + TILE)
            jobs.append((r0, r1 - r0, p0, w, 3 * p0, 3 * w, r0 * 3 * nb + 3 * p0, 3 * nb))
            inc_base.append(ptr0)
    return dict(jobs=np.array(jobs, dtype=np.int64), pan_local=np.concatenate(pan_idx),
                inc_ptr=np.concatenate(inc_ptr).astype(np.int32), inc=np.array(inc, dtype=np.int32),
                inc_base=np.array(inc_base, dtype=np.int64))


def panel_pair_matrix(mesh, panels_a, panels_b, kind, q, chunk=None, pq=None, singular=None):
    """All-pairs Galerkin integrals between two panel sets (kernels.py:365-434):
    regular pairs by the q^2-point tensor rule, touching pairs from the
    singular table (its order is the Sauter-Schwab order; without a table the
    touching pairs are integrated at order q).  SLP (Pa, Pb); DLP (Pa, Pb, 3)
    per local vertex of the column panel."""
    if kind not in (SLP, DLP):
        raise ValueError(f"unknown operator kind {kind!r}")
    dm = device_mesh(mesh)
    pa = np.asarray(panels_a, dtype=np.int64)
    pb = np.asarray(panels_b, dtype=np.int64)
    na, nb = len(pa), len(pb)
    if na == 0 or nb == 0:
        return np.zeros((na, nb, 3) if kind == DLP else (na, nb))
    table = _table_for(dm, kind, q, singular)
    if kind == SLP:
        out = D.zeros((na * nb,))
        run_slp_jobs(dm, q, np.array([[0, na, 0, nb, 0, nb]], dtype=np.int64), pa.astype(np.int32),
                     pb.astype(np.int32), table, out)
        return D.host(out).reshape(na, nb)
    J = _dlp_pair_jobs(na, nb)
    packed = dict(jobs=J["jobs"], row_idx=pa.astype(np.int32), pan_idx=pb[J["pan_local"]].astype(np.int32),
                  inc_ptr=J["inc_ptr"], inc=J["inc"], inc_base=J["inc_base"])
    out = D.zeros((na * nb * 3,))
    run_dlp_jobs(dm, q, packed, table, out)
    return D.host(out).reshape(na, nb, 3)


def slp_block(mesh, rows, cols, q, require_disjoint=False, pq=None, singular=None):
    """Dense single-layer block rows x cols (panel ids) (kernels.py:437-445);
    ValueError on a touching pair when require_disjoint."""
    dm = device_mesh(mesh)
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if len(rows) == 0 or len(cols) == 0:
        return np.zeros((len(rows), len(cols)))
    table = None if require_disjoint else _table_for(dm, SLP, q, singular)
    out = D.zeros((len(rows) * len(cols),))
    run_slp_jobs(dm, q, np.array([[0, len(rows), 0, len(cols), 0, len(cols)]], dtype=np.int64),
                 rows.astype(np.int32), cols.astype(np.int32), table, out)
    return D.host(out).reshape(len(rows), len(cols))


def dlp_block(mesh, rows, cols, q, vertex_tris=None, require_disjoint=False, pq=None, singular=None):
    """Dense double-layer block: P0 rows (panels) x P1 columns (vertices)
    through the panels incident to the column vertices with the barycentric
    scatter fused in (kernels.py:448-468); ValueError on a touching pair when
    require_disjoint."""
    dm = device_mesh(mesh)
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if len(rows) == 0 or len(cols) == 0:
        return np.zeros((len(rows), len(cols)))
    table = None if require_disjoint else _table_for(dm, DLP, q, singular)
    out = D.zeros((len(rows) * len(cols),))
    run_dlp_jobs(dm, q, build_dlp_jobs(dm.mesh, [(rows, cols, 0, len(cols))]), table, out)
    return D.host(out).reshape(len(rows), len(cols))


# ---------------------------------------------------------------------------
# hypersingular operator (surface-curl representation, kernels.py:229-239,
# 471-511): single-layer panel-pair values of each block's incident panels
# (k_blocks_slp) contracted with the P1 hat curls (k_hyp_scatter)

def triangle_curls(mesh):
    """Surface curl n x grad of each P1 hat, constant per panel (kernels.py:
    229-239): (F, 3, 3), curls[f, l] = (V_{l+1} - V_{l+2}) / (2 area_f)."""
    c = mesh.vertices[mesh.triangles]
    out = np.empty_like(c)
    for l in range(3):
        out[:, l, :] = c[:, (l + 1) % 3, :] - c[:, (l + 2) % 3, :]
    return out / (2.0 * mesh.areas)[:, None, None]


def _vertex_incidence(mesh, verts, panels):
    """Per vertex (in order) its incident panels, ascending: counts, position
    in `panels` (sorted) and 3 * panel + local vertex index."""
    vptr, vidx = mesh.vertex_triangle_csr()
    verts = np.asarray(verts, dtype=np.int64)
    counts = vptr[verts + 1] - vptr[verts]
    starts = np.repeat(vptr[verts], counts)
    flat = vidx[starts + (np.arange(int(counts.sum())) - np.repeat(np.cumsum(counts) - counts, counts))]
    owner = np.repeat(verts, counts)
    local = np.argmax(mesh.triangles[flat] == owner[:, None], axis=1)
    return counts, np.searchsorted(panels, flat), 3 * flat + local


def hyp_jobs(mesh, blocks):
    """Host job description of hypersingular blocks (row vertices, column
    vertices, out_off, ld): the single-layer pair jobs over each block's
    incident panels and the incidence lists of k_hyp_scatter."""
    vptr, vidx = mesh.vertex_triangle_csr()

    def incident(v):
        v = np.asarray(v, dtype=np.int64)
        if len(v) == 0:
            return np.zeros(0, dtype=np.int64)
        return np.unique(np.concatenate([vidx[vptr[a] : vptr[a + 1]] for a in v]))

    jobs, desc, pa_l, pb_l = [], [], [], []
    rp, rpos, rcl, cp, cpos, ccl = [], [], [], [], [], []
    v_off = pa_off = pb_off = rbase = cbase = rinc = cinc = 0
    for rows, cols, off, ld in blocks:
        pa, pb = incident(rows), incident(cols)
        rc, rps, rcls = _vertex_incidence(mesh, rows, pa)
        cc, cps, ccls = _vertex_incidence(mesh, cols, pb)
        jobs.append((pa_off, len(pa), pb_off, len(pb), v_off, len(pb)))
        desc.append((len(rows), len(cols), v_off, len(pb), rbase, cbase, off, ld))
        rp.append(rinc + np.concatenate([[0], np.cumsum(rc)]))
        cp.append(cinc + np.concatenate([[0], np.cumsum(cc)]))
        rpos.append(rps)
        rcl.append(rcls)
        cpos.append(cps)
        ccl.append(ccls)
        pa_l.append(pa)
        pb_l.append(pb)
        rinc += int(rc.sum())
        cinc += int(cc.sum())
        rbase += len(rows) + 1
        cbase += len(cols) + 1
        v_off += len(pa) * len(pb)
        pa_off += len(pa)
        pb_off += len(pb)
    cat = lambda a, dt: np.concatenate(a).astype(dt) if a and sum(len(x) for x in a) else np.zeros(1, dtype=dt)
    return dict(jobs=np.array(jobs, dtype=np.int64).reshape(-1, 6), desc=np.array(desc, dtype=np.int64).reshape(-1, 8),
                pa=cat(pa_l, np.int32), pb=cat(pb_l, np.int32), v_total=v_off,
                r_ptr=cat(rp, np.int32), r_pos=cat(rpos, np.int32), r_cl=cat(rcl, np.int32),
                c_ptr=cat(cp, np.int32), c_pos=cat(cpos, np.int32), c_cl=cat(ccl, np.int32))


def run_hyp_blocks(dmesh, q, blocks, table, out):
    """Hypersingular blocks into `out` (device float64); table None: touching
    pairs rejected (ValueError), else taken from the single-layer table."""
    blocks = list(blocks)
    if not blocks:
        return
    J = hyp_jobs(dmesh.mesh, blocks)
    vals = D.zeros((max(J["v_total"], 1),))
    run_slp_jobs(dmesh, q, J["jobs"], J["pa"], J["pb"], table, vals)
    t = {k: D.dev(J[k], np.int32) for k in ("r_ptr", "r_pos", "r_cl", "c_ptr", "c_pos", "c_cl")}
    desc = D.dev(J["desc"], np.int64)
    _lib.check(_lib.lib().h2b_hyp_scatter(len(J["desc"]), desc.data_ptr(), t["r_ptr"].data_ptr(),
                                          t["r_pos"].data_ptr(), t["r_cl"].data_ptr(), t["c_ptr"].data_ptr(),
                                          t["c_pos"].data_ptr(), t["c_cl"].data_ptr(), dmesh.curls().data_ptr(),
                                          vals.data_ptr(), out.data_ptr(), D.stream()))


def hyp_block(mesh, rows, cols, q, vertex_tris=None, curls=None, require_disjoint=False, pq=None, singular=None):
    """Dense hypersingular block, P1 rows x P1 columns (vertex ids), through
    the surface-curl representation (kernels.py:471-511); ValueError on a
    touching pair when require_disjoint.  `vertex_tris` / `curls` / `pq` are
    accepted for signature compatibility (the device mesh holds its own)."""
    dm = device_mesh(mesh)
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if len(rows) == 0 or len(cols) == 0:
        return np.zeros((len(rows), len(cols)))
    table = None if require_disjoint else _table_for(dm, SLP, q, singular)
    out = D.zeros((len(rows) * len(cols),))
    run_hyp_blocks(dm, q, [(rows, cols, 0, len(cols))], table, out)
    return D.host(out).reshape(len(rows), len(cols))
