"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package (`h2bem`, /root/reference/pkg/src) in this container.

Test infrastructure only: nothing in the product imports this file, and it
cannot run on the GPU box (the reference is not there).  Re-run with

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [--skip-large]

OPENBLAS_NUM_THREADS=1 is mandatory: multithreaded OpenBLAS inside the
reference's thread pool corrupts double-layer blocks.

What is pinned (all produced by the reference's own public functions):
  rules.npz        Gauss-Legendre / Duffy / Sauter-Schwab tables (quadrature.py:49-190)
  mesh.npz         sphere level 2 in full, sha256 digests of levels 4..9 (mesh.py:146-154)
  struct_cfg{0,1}.npz  cluster trees + block trees in full (clustering.py:78-160)
  struct_large.json    digests of the cfg2 / cfg3 trees and block lists
  touch.npz        touching pair keys, case codes and permutations (kernels.py:246-343,
                   quadrature.py:90-118)
  singular.npz     pair_integrals samples, SLP/DLP, q_ss 4 and 5 (kernels.py:260-319)
  pairs.npz        pair_integrals on mixed pair lists (disjoint included), and
                   panel_pair_matrix / slp_block / dlp_block without a table
  near_cfg0.npz    sampled split-order nearfield blocks (kernels.py:365-468)
  h2_cfg0.npz      full GCA basis + sampled couplings + matvec x/y of config 0
  h2_cfg1.npz      pivots/ranks digests + matvec x/y of config 1
  h2_cfg3p.npz     config-3 parameters (m=5, eta=1.5, leaf 64, q 3/4) at sphere
                   level 6: pivots/ranks + matvec / rmatvec x/y + samples
  cfg3_basis.npz   config-3 (sphere level 9, m=5) reference GCA basis: rank and
                   pivot-list digest per cluster (device-basis agreement)
  h2_dlp4.npz      level-4 double-layer H^2 (P0 x P1) matvec x/y + basis
  sample_l8.npz    config-2 size (sphere level 8): a seeded sample of single- and
                   double-layer near blocks with the split orders (regular 3,
                   Sauter-Schwab 5) and of touching-pair integrals
  cube4.npz        config-4 geometry at n=4 (this repo's cube_shell_mesh arrays fed
                   to the reference): trees + block trees (grid-aligned: exact
                   ties in the splits), SLP/DLP GCA H^2 matvec x/y, SLP basis
"""

import argparse
import hashlib
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
if os.environ["OPENBLAS_NUM_THREADS"] != "1":
    sys.exit("OPENBLAS_NUM_THREADS must be 1 (reference DLP race)")

sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from h2bem import gca, kernels, quadrature as quad  # noqa: E402
from h2bem import spaces  # noqa: E402
from h2bem.clustering import BlockTree, build_cluster_tree  # noqa: E402
from h2bem.containers import AssemblyContext, H2Matrix, dense_block  # noqa: E402
from h2bem.mesh import sphere_mesh  # noqa: E402
from h2bem._util import pmap  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
THREADS = os.cpu_count() or 1


def digest(a, dtype=None):
    a = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    return hashlib.sha256(a.tobytes()).hexdigest()


def log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


# ---------------------------------------------------------------------------
def tree_arrays(tree):
    n = len(tree.nodes)
    start = np.array([c.start for c in tree.nodes], dtype=np.int64)
    end = np.array([c.end for c in tree.nodes], dtype=np.int64)
    depth = np.array([c.depth for c in tree.nodes], dtype=np.int64)
    left = np.full(n, -1, dtype=np.int64)
    right = np.full(n, -1, dtype=np.int64)
    for c in tree.nodes:
        assert tree.nodes[c.uid] is c
        if c.children:
            left[c.uid] = c.children[0].uid
            right[c.uid] = c.children[1].uid
    boxes = np.stack([c.box for c in tree.nodes])
    return dict(perm=tree.perm.astype(np.int64), start=start, end=end, depth=depth,
                left=left, right=right, boxes=boxes)


def block_arrays(bt):
    far = np.array([[b.row.uid, b.col.uid] for b in bt.far], dtype=np.int64).reshape(-1, 2)
    near = np.array([[b.row.uid, b.col.uid] for b in bt.near], dtype=np.int64).reshape(-1, 2)
    return far, near


def structure_digest(mesh, r_leaf, eta, row_space, col_space):
    rb = spaces.DofSpace(row_space, mesh).support_boxes()
    rt = build_cluster_tree(rb, r_leaf)
    if col_space == row_space:
        ct = rt
    else:
        ct = build_cluster_tree(spaces.DofSpace(col_space, mesh).support_boxes(), r_leaf)
    bt = BlockTree(rt, ct, eta)
    far, near = block_arrays(bt)
    out = {"n_far": int(len(far)), "n_near": int(len(near)), "far": digest(far), "near": digest(near)}
    for name, t in (("row", rt), ("col", ct)):
        ta = tree_arrays(t)
        out[f"{name}_nodes"] = int(len(ta["start"]))
        out[f"{name}_perm"] = digest(ta["perm"])
        out[f"{name}_ranges"] = digest(np.stack([ta["start"], ta["end"], ta["depth"], ta["left"], ta["right"]]))
        out[f"{name}_boxes"] = digest(ta["boxes"])
    return out


# ---------------------------------------------------------------------------
def split_nearfield(ctx, kind, bt, q_reg, q_ss):
    """Nearfield payloads with regular order q_reg and singular order q_ss, through
    the reference's kernel-level entry points (slp_block / dlp_block with an
    explicit SingularTable); bit-identical to assemble_nearfield when q_reg == q_ss."""
    pq = ctx.panel_quad(q_reg)
    table = ctx.singular_table(kind, q_ss)
    rt, ct = bt.row_tree, bt.col_tree

    def build(b):
        rows, cols = rt.dofs(b.row), ct.dofs(b.col)
        if kind == kernels.SLP:
            return kernels.slp_block(ctx.mesh, rows, cols, q_reg, pq=pq, singular=table)
        if kind == kernels.HYP:
            return kernels.hyp_block(ctx.mesh, rows, cols, q_reg, ctx.vertex_tris, ctx.curls, pq=pq,
                                     singular=table)
        return kernels.dlp_block(ctx.mesh, rows, cols, q_reg, ctx.vertex_tris, pq=pq, singular=table)

    return pmap(build, bt.near, THREADS)


def split_h2(ctx, kind, bt, rb, cb, q_reg, q_ss):
    def couple(b):
        return dense_block(ctx, kind, rb.pivots[b.row.uid], cb.pivots[b.col.uid], q_reg, require_disjoint=True)

    couplings = pmap(couple, bt.far, THREADS)
    near = split_nearfield(ctx, kind, bt, q_reg, q_ss)
    return H2Matrix(bt, rb, cb, couplings, near)


def basis_arrays(prefix, basis, tree):
    uids = [c.uid for c in tree.nodes]
    ranks = np.array([basis.rank[u] for u in uids], dtype=np.int64)
    piv = np.concatenate([np.asarray(basis.pivots[u], dtype=np.int64) for u in uids])
    out = {f"{prefix}ranks": ranks, f"{prefix}pivots": piv}
    vs = [basis.V[c.uid].ravel() for c in tree.nodes if c.is_leaf]
    es = [basis.E[c.uid].ravel() for c in tree.nodes if c.uid in basis.E]
    out[f"{prefix}V"] = np.concatenate(vs)
    out[f"{prefix}E"] = np.concatenate(es) if es else np.zeros(0)
    return out


# ---------------------------------------------------------------------------
def gen_rules():
    out = {}
    for q in range(1, 9):
        g = quad.gauss_legendre(q)
        out[f"gl{q}_x"] = g.points
        out[f"gl{q}_w"] = g.weights
    for q in (2, 3, 4, 5):
        p, w = quad.triangle_rule(q)
        out[f"tri{q}_p"] = p
        out[f"tri{q}_w"] = w
    for case in (quad.IDENTICAL, quad.SHARED_EDGE, quad.SHARED_VERTEX, quad.DISJOINT):
        for q in (3, 4, 5):
            r = quad.sauter_schwab_rule(case, q)
            out[f"ss_{case}_{q}_p"] = r.points
            out[f"ss_{case}_{q}_w"] = r.weights
    np.savez_compressed(os.path.join(HERE, "rules.npz"), **out)


def gen_mesh(levels):
    m2 = sphere_mesh(2)
    out = {"l2_vertices": m2.vertices, "l2_triangles": m2.triangles, "l2_normals": m2.normals, "l2_areas": m2.areas}
    meta = {}
    for lv in levels:
        m = sphere_mesh(lv)
        meta[str(lv)] = {
            "n_vertices": int(m.n_vertices), "n_triangles": int(m.n_triangles),
            "vertices": digest(m.vertices), "triangles": digest(m.triangles, np.int64),
            "normals": digest(m.normals), "areas": digest(m.areas),
        }
        log(f"mesh level {lv}")
    np.savez_compressed(os.path.join(HERE, "mesh.npz"), **out)
    with open(os.path.join(HERE, "mesh_digests.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def gen_structure_small():
    for name, level, leaf, eta in (("cfg0", 4, 32, 2.0), ("cfg1", 6, 64, 2.0)):
        mesh = sphere_mesh(level)
        out = {}
        for sp_name, sp in (("p0", spaces.P0), ("p1", spaces.P1)):
            boxes = spaces.DofSpace(sp, mesh).support_boxes()
            out[f"{sp_name}_support"] = boxes
            t = build_cluster_tree(boxes, leaf)
            for k, v in tree_arrays(t).items():
                out[f"{sp_name}_{k}"] = v
            if sp == spaces.P0:
                tp0 = t
            else:
                tp1 = t
        far, near = block_arrays(BlockTree(tp0, tp0, eta))
        out["slp_far"], out["slp_near"] = far, near
        far, near = block_arrays(BlockTree(tp0, tp1, eta))
        out["dlp_far"], out["dlp_near"] = far, near
        np.savez_compressed(os.path.join(HERE, f"struct_{name}.npz"), **out)
        log(f"structure {name}")


def gen_structure_large():
    meta = {}
    meta["cfg2_slp"] = structure_digest(sphere_mesh(8), 64, 2.0, spaces.P0, spaces.P0)
    log("cfg2 slp structure")
    meta["cfg2_dlp"] = structure_digest(sphere_mesh(8), 64, 2.0, spaces.P0, spaces.P1)
    log("cfg2 dlp structure")
    meta["cfg3_slp"] = structure_digest(sphere_mesh(9), 64, 1.5, spaces.P0, spaces.P0)
    log("cfg3 slp structure")
    with open(os.path.join(HERE, "struct_large.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


def gen_touch():
    out = {}
    for level in (2, 4):
        mesh = sphere_mesh(level)
        keys = kernels.touching_pairs(mesh)
        F = mesh.n_triangles
        pa, pb = keys // F, keys % F
        codes = kernels._classify_pairs(mesh, pa, pb).astype(np.int64)
        perms = np.zeros((len(keys), 6), dtype=np.int64)
        for i, (a, b) in enumerate(zip(pa, pb)):
            _, qa, qb = quad.classify_panel_pair(mesh.triangles[a], mesh.triangles[b])
            perms[i, :3] = qa
            perms[i, 3:] = qb
        out[f"l{level}_keys"] = keys
        out[f"l{level}_codes"] = codes
        out[f"l{level}_perms"] = perms
    np.savez_compressed(os.path.join(HERE, "touch.npz"), **out)


def gen_singular():
    mesh = sphere_mesh(4)
    F = mesh.n_triangles
    keys = kernels.touching_pairs(mesh)
    pa, pb = keys // F, keys % F
    codes = kernels._classify_pairs(mesh, pa, pb)
    rng = np.random.default_rng(20261020)
    pick = []
    for code, cnt in ((3, 48), (2, 96), (1, 96)):
        idx = np.flatnonzero(codes == code)
        pick.append(np.sort(rng.choice(idx, cnt, replace=False)))
    pick = np.concatenate(pick)
    out = {"pa": pa[pick], "pb": pb[pick], "code": codes[pick].astype(np.int64)}
    for q in (3, 4, 5):
        out[f"slp_q{q}"] = kernels.pair_integrals(mesh, pa[pick], pb[pick], kernels.SLP, q)
        out[f"dlp_q{q}"] = kernels.pair_integrals(mesh, pa[pick], pb[pick], kernels.DLP, q)
    # regular (disjoint) panel pairs through panel_pair_matrix's bulk path
    ra = np.array([0, 5, 77, 300, 1023, 2047])
    rb = np.array([1500, 900, 33, 640, 12, 1800, 7])
    for q in (3, 4):
        out[f"reg_slp_q{q}"] = kernels.panel_pair_matrix(mesh, ra, rb, kernels.SLP, q)
        out[f"reg_dlp_q{q}"] = kernels.panel_pair_matrix(mesh, ra, rb, kernels.DLP, q)
    out["reg_rows"], out["reg_cols"] = ra, rb
    np.savez_compressed(os.path.join(HERE, "singular.npz"), **out)


def build_world(level, leaf, eta, m, eps, kind):
    mesh = sphere_mesh(level)
    ctx = AssemblyContext(mesh)
    t0 = build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), leaf)
    if kind == kernels.SLP:
        bt = BlockTree(t0, t0, eta)
        rb = gca.build_basis(ctx, t0, gca.P0_SLP, m, eps, threads=THREADS)
        cb = rb
    elif kind == kernels.HYP:
        t1 = build_cluster_tree(spaces.DofSpace(spaces.P1, mesh).support_boxes(), leaf)
        bt = BlockTree(t1, t1, eta)
        rb = gca.build_basis(ctx, t1, gca.P1_CURL, m, eps, threads=THREADS)
        cb = rb
    else:
        t1 = build_cluster_tree(spaces.DofSpace(spaces.P1, mesh).support_boxes(), leaf)
        bt = BlockTree(t0, t1, eta)
        rb = gca.build_basis(ctx, t0, gca.P0_SLP, m, eps, threads=THREADS)
        cb = gca.build_basis(ctx, t1, gca.P1_DLP, m, eps, threads=THREADS)
    return mesh, ctx, bt, rb, cb


def gen_h2_cfg0():
    mesh, ctx, bt, rb, cb = build_world(4, 32, 2.0, 3, 1e-4, kernels.SLP)
    log("cfg0 basis")
    H = split_h2(ctx, kernels.SLP, bt, rb, cb, 3, 4)
    log("cfg0 h2 assembled")
    x = np.random.default_rng(0).uniform(-1.0, 1.0, H.shape[1])
    y = H.matvec(x)
    # dense product with the same split orders (oracle for accuracy, not parity)
    allp = np.arange(mesh.n_triangles)
    A = kernels.panel_pair_matrix(mesh, allp, allp, kernels.SLP, 3, pq=ctx.panel_quad(3),
                                  singular=ctx.singular_table(kernels.SLP, 4))
    out = basis_arrays("", rb, bt.row_tree)
    rng = np.random.default_rng(7)
    nsel = rng.choice(len(H.near), 24, replace=False)
    fsel = rng.choice(len(H.far), 48, replace=False)
    out["near_sel"] = np.sort(nsel)
    out["near_vals"] = np.concatenate([H.near[i][1].ravel() for i in np.sort(nsel)])
    out["far_sel"] = np.sort(fsel)
    out["far_vals"] = np.concatenate([H.far[i][1].ravel() for i in np.sort(fsel)])
    out["near_sum"] = np.array([float(sum(d.sum() for _, d in H.near))])
    out["far_sum"] = np.array([float(sum(s.sum() for _, s in H.far))])
    out["x"], out["y"], out["y_dense"] = x, y, A @ x
    out["diag"] = H.diagonal()
    rep = H.storage_report()
    out["storage"] = np.array([rep["basis"], rep["coupling"], rep["lowrank"], rep["nearfield"]], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "h2_cfg0.npz"), **out)


def gen_h2_cfg1():
    mesh, ctx, bt, rb, cb = build_world(6, 64, 2.0, 4, 1e-4, kernels.SLP)
    log("cfg1 basis")
    H = split_h2(ctx, kernels.SLP, bt, rb, cb, 3, 4)
    log("cfg1 h2 assembled")
    rng = np.random.default_rng(1)
    xs = [rng.standard_normal(H.shape[1]) for _ in range(2)]
    out = {"x0": xs[0], "y0": H.matvec(xs[0]), "x1": xs[1], "y1": H.matvec(xs[1])}
    ba = basis_arrays("", rb, bt.row_tree)
    out["ranks"] = ba["ranks"]
    out["pivots"] = ba["pivots"]
    out["V_sum"] = np.array([ba["V"].sum(), np.abs(ba["V"]).sum()])
    out["E_sum"] = np.array([ba["E"].sum(), np.abs(ba["E"]).sum()])
    rep = H.storage_report()
    out["storage"] = np.array([rep["basis"], rep["coupling"], rep["lowrank"], rep["nearfield"]], dtype=np.int64)
    out["diag"] = H.diagonal()
    np.savez_compressed(os.path.join(HERE, "h2_cfg1.npz"), **out)


def gen_h2_cfg3p():
    """BASELINE.json config-3 parameters (GCA m=5, eta=1.5, leaf 64, orders
    3/4, single layer) at a reference-tractable size: sphere level 6."""
    mesh, ctx, bt, rb, cb = build_world(6, 64, 1.5, 5, 1e-4, kernels.SLP)
    log("cfg3p basis")
    H = split_h2(ctx, kernels.SLP, bt, rb, cb, 3, 4)
    log("cfg3p h2 assembled")
    rng = np.random.default_rng(3)
    xs = [rng.standard_normal(H.shape[1]) for _ in range(2)]
    out = {"x0": xs[0], "y0": H.matvec(xs[0]), "x1": xs[1], "y1": H.matvec(xs[1])}
    out["yt0"] = H.rmatvec(xs[0])
    ba = basis_arrays("", rb, bt.row_tree)
    out["ranks"] = ba["ranks"]
    out["pivots"] = ba["pivots"]
    out["V_sum"] = np.array([ba["V"].sum(), np.abs(ba["V"]).sum()])
    out["E_sum"] = np.array([ba["E"].sum(), np.abs(ba["E"]).sum()])
    rep = H.storage_report()
    out["storage"] = np.array([rep["basis"], rep["coupling"], rep["lowrank"], rep["nearfield"]], dtype=np.int64)
    out["diag"] = H.diagonal()
    rng = np.random.default_rng(11)
    nsel = np.sort(rng.choice(len(H.near), 16, replace=False))
    fsel = np.sort(rng.choice(len(H.far), 32, replace=False))
    out["near_sel"], out["far_sel"] = nsel, fsel
    out["near_vals"] = np.concatenate([H.near[i][1].ravel() for i in nsel])
    out["far_vals"] = np.concatenate([H.far[i][1].ravel() for i in fsel])
    np.savez_compressed(os.path.join(HERE, "h2_cfg3p.npz"), **out)


def gen_cfg3_basis():
    """The reference GCA basis at config 3 (sphere level 9, leaf 64, m=5,
    eps 1e-4): per cluster (uid order) its rank and a digest of its pivot
    list (first 8 bytes of sha256 over the int64 pivots), so the device basis
    can be compared with the reference's cluster by cluster.  Also the
    tree/block-list digests it was built on."""
    mesh = sphere_mesh(9)
    ctx = AssemblyContext(mesh)
    t0 = build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), 64)
    log("cfg3 tree")
    rb = gca.build_basis(ctx, t0, gca.P0_SLP, 5, 1e-4, threads=THREADS)
    log("cfg3 basis")
    uids = [c.uid for c in t0.nodes]
    ranks = np.array([rb.rank[u] for u in uids], dtype=np.int16)
    dig = np.array([int.from_bytes(hashlib.sha256(np.asarray(rb.pivots[u], dtype=np.int64).tobytes()).digest()[:8],
                                   "little", signed=True) for u in uids], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "cfg3_basis.npz"), ranks=ranks, pivot_digest=dig,
                        perm_digest=np.array([digest(t0.perm)]))


def gen_h2_dlp4():
    mesh, ctx, bt, rb, cb = build_world(4, 32, 2.0, 3, 1e-4, kernels.DLP)
    log("dlp4 bases")
    H = split_h2(ctx, kernels.DLP, bt, rb, cb, 3, 5)
    log("dlp4 h2 assembled")
    x = np.random.default_rng(2).uniform(-1.0, 1.0, H.shape[1])
    out = {"x": x, "y": H.matvec(x)}
    out.update(basis_arrays("row_", rb, bt.row_tree))
    out.update(basis_arrays("col_", cb, bt.col_tree))
    rng = np.random.default_rng(9)
    nsel = np.sort(rng.choice(len(H.near), 24, replace=False))
    fsel = np.sort(rng.choice(len(H.far), 32, replace=False))
    out["near_sel"], out["far_sel"] = nsel, fsel
    out["near_vals"] = np.concatenate([H.near[i][1].ravel() for i in nsel])
    out["far_vals"] = np.concatenate([H.far[i][1].ravel() for i in fsel])
    out["near_sum"] = np.array([float(sum(d.sum() for _, d in H.near))])
    np.savez_compressed(os.path.join(HERE, "h2_dlp4.npz"), **out)


def gen_h2_hyp4():
    """Hypersingular H^2 operator (P1 x P1, curl representation) at sphere
    level 4, leaf 32, eta 2, m 3, q 3 / 4: bases, samples, one matvec."""
    mesh, ctx, bt, rb, cb = build_world(4, 32, 2.0, 3, 1e-4, kernels.HYP)
    log("hyp4 basis")
    H = split_h2(ctx, kernels.HYP, bt, rb, cb, 3, 4)
    log("hyp4 h2 assembled")
    x = np.random.default_rng(11).uniform(-1.0, 1.0, H.shape[1])
    out = {"x": x, "y": H.matvec(x), "yt": H.rmatvec(x)}
    out.update(basis_arrays("", rb, bt.row_tree))
    rng = np.random.default_rng(12)
    nsel = np.sort(rng.choice(len(H.near), 24, replace=False))
    fsel = np.sort(rng.choice(len(H.far), 32, replace=False))
    out["near_sel"], out["far_sel"] = nsel, fsel
    out["near_vals"] = np.concatenate([H.near[i][1].ravel() for i in nsel])
    out["far_vals"] = np.concatenate([H.far[i][1].ravel() for i in fsel])
    out["near_sum"] = np.array([float(sum(d.sum() for _, d in H.near))])
    # one dense hypersingular block through the kernel-level entry point
    rows, cols = np.array([0, 3, 17, 100, 511]), np.array([0, 1, 2, 40, 300, 1025])
    out["hb_rows"], out["hb_cols"] = rows, cols
    out["hb_q3"] = kernels.hyp_block(mesh, rows, cols, 3, singular=ctx.singular_table(kernels.HYP, 3))
    np.savez_compressed(os.path.join(HERE, "h2_hyp4.npz"), **out)


class _OnDemandTable:
    """Stands in for kernels.SingularTable on a sampled block: the reference's
    panel_pair_matrix looks touching pairs up through .lookup, answered by the
    reference's own pair_integrals at the Sauter-Schwab order."""

    def __init__(self, mesh, kind, q):
        self.mesh, self.kind, self.q = mesh, kind, q

    def lookup(self, pa, pb):
        return kernels.pair_integrals(self.mesh, np.asarray(pa), np.asarray(pb), self.kind, self.q)


def gen_sample_l8():
    """Config-2 size parity sample (the full reference nearfield takes hours)."""
    mesh = sphere_mesh(8)
    ctx = AssemblyContext(mesh)
    t0 = build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), 64)
    t1 = build_cluster_tree(spaces.DofSpace(spaces.P1, mesh).support_boxes(), 64)
    bs, bd = BlockTree(t0, t0, 2.0), BlockTree(t0, t1, 2.0)
    log("l8 structure")
    rng = np.random.default_rng(8)
    pq = ctx.panel_quad(3)
    vt = mesh.vertex_triangles()
    out = {}
    for name, bt, n_sel in (("slp", bs, 40), ("dlp", bd, 24)):
        sel = np.sort(rng.choice(len(bt.near), n_sel, replace=False))
        vals = []
        for i in sel:
            b = bt.near[i]
            rows = t0.perm[b.row.start : b.row.end]
            cols = bt.col_tree.perm[b.col.start : b.col.end]
            if name == "slp":
                blk = kernels.slp_block(mesh, rows, cols, 3, pq=pq, singular=_OnDemandTable(mesh, kernels.SLP, 5))
            else:
                blk = kernels.dlp_block(mesh, rows, cols, 3, vertex_tris=vt, pq=pq,
                                        singular=_OnDemandTable(mesh, kernels.DLP, 5))
            vals.append(blk.ravel())
        out[f"{name}_sel"] = sel
        out[f"{name}_vals"] = np.concatenate(vals)
        log(f"l8 {name} blocks")
    keys = kernels.touching_pairs(mesh, vt)
    pick = np.sort(rng.choice(len(keys), 5000, replace=False))
    pa, pb = keys[pick] // mesh.n_triangles, keys[pick] % mesh.n_triangles
    out["pa"], out["pb"] = pa, pb
    out["slp_pairs"] = kernels.pair_integrals(mesh, pa, pb, kernels.SLP, 5)
    out["dlp_pairs"] = kernels.pair_integrals(mesh, pa, pb, kernels.DLP, 5)
    np.savez_compressed(os.path.join(HERE, "sample_l8.npz"), **out)


def gen_cube():
    """Config 4 geometry (3x3x3 unit cubes minus the centre, merged surface) at
    n=4: 1920 flat panels on a lattice -- the split coordinates tie exactly."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2001_05523_b200.mesh import cube_shell_mesh  # the input geometry only
    from h2bem.mesh import SurfaceMesh

    ours = cube_shell_mesh(4)
    mesh = SurfaceMesh(ours.vertices, ours.triangles)
    ctx = AssemblyContext(mesh)
    out = {"vertices": mesh.vertices, "triangles": mesh.triangles}
    t0 = build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), 32)
    t1 = build_cluster_tree(spaces.DofSpace(spaces.P1, mesh).support_boxes(), 32)
    for name, t in (("p0", t0), ("p1", t1)):
        for k, v in tree_arrays(t).items():
            out[f"{name}_{k}"] = v
    bs, bd = BlockTree(t0, t0, 2.0), BlockTree(t0, t1, 2.0)
    out["slp_far"], out["slp_near"] = block_arrays(bs)
    out["dlp_far"], out["dlp_near"] = block_arrays(bd)
    rb = gca.build_basis(ctx, t0, gca.P0_SLP, 3, 1e-4, threads=THREADS)
    cb = gca.build_basis(ctx, t1, gca.P1_DLP, 3, 1e-4, threads=THREADS)
    log("cube bases")
    ba = basis_arrays("", rb, t0)
    out["slp_ranks"], out["slp_pivots"] = ba["ranks"], ba["pivots"]
    rng = np.random.default_rng(4)
    Hs = split_h2(ctx, kernels.SLP, bs, rb, rb, 3, 4)
    out["x_slp"] = rng.uniform(-1.0, 1.0, Hs.shape[1])
    out["y_slp"] = Hs.matvec(out["x_slp"])
    Hd = split_h2(ctx, kernels.DLP, bd, rb, cb, 3, 4)
    out["x_dlp"] = rng.uniform(-1.0, 1.0, Hd.shape[1])
    out["y_dlp"] = Hd.matvec(out["x_dlp"])
    np.savez_compressed(os.path.join(HERE, "cube4.npz"), **out)


def gen_pairs():
    """pair_integrals on separated (disjoint-case) and mixed pair lists, and
    panel_pair_matrix / slp_block / dlp_block without a singular table (the
    touching pairs integrated on the fly at order q) -- the kernel-level
    entry points (kernels.py:260-319, 365-468)."""
    mesh = sphere_mesh(3)
    F = mesh.n_triangles
    rng = np.random.default_rng(7)
    pa = rng.integers(0, F, 400)
    pb = rng.integers(0, F, 400)
    pb[:20] = pa[:20]  # a few identical pairs in the mixed list
    codes = kernels._classify_pairs(mesh, pa, pb)
    out = {"pa": pa, "pb": pb, "code": codes.astype(np.int64)}
    for q in (2, 3, 4):
        out[f"slp_q{q}"] = kernels.pair_integrals(mesh, pa, pb, kernels.SLP, q)
        out[f"dlp_q{q}"] = kernels.pair_integrals(mesh, pa, pb, kernels.DLP, q)
    ra = np.array([0, 1, 2, 3, 40, 41, 200, 511])
    rb = np.array([0, 2, 5, 9, 40, 300, 301, 17, 510])
    verts = np.array([0, 1, 5, 17, 100, 255])
    for q in (3, 4):
        out[f"ppm_slp_q{q}"] = kernels.panel_pair_matrix(mesh, ra, rb, kernels.SLP, q)
        out[f"ppm_dlp_q{q}"] = kernels.panel_pair_matrix(mesh, ra, rb, kernels.DLP, q)
        out[f"slpb_q{q}"] = kernels.slp_block(mesh, ra, rb, q)
        out[f"dlpb_q{q}"] = kernels.dlp_block(mesh, ra, verts, q)
    out["ra"], out["rb"], out["verts"] = ra, rb, verts
    np.savez_compressed(os.path.join(HERE, "pairs.npz"), **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-large", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    steps = [
        ("rules", gen_rules),
        ("mesh", lambda: gen_mesh([4, 6] if args.skip_large else [4, 6, 8, 9])),
        ("struct", gen_structure_small),
        ("touch", gen_touch),
        ("singular", gen_singular),
        ("pairs", gen_pairs),
        ("h2_cfg0", gen_h2_cfg0),
        ("h2_dlp4", gen_h2_dlp4),
        ("h2_hyp4", gen_h2_hyp4),
        ("h2_cfg1", gen_h2_cfg1),
        ("h2_cfg3p", gen_h2_cfg3p),
        ("cube", gen_cube),
        ("sample_l8", gen_sample_l8),
    ]
    if not args.skip_large:
        steps.append(("struct_large", gen_structure_large))
        steps.append(("cfg3_basis", gen_cfg3_basis))
    for name, fn in steps:
        if args.only and name not in args.only.split(","):
            continue
        t = time.time()
        fn()
        log(f"{name} done in {time.time() - t:.1f}s")


if __name__ == "__main__":
    main()
