"""Config 4 of BASELINE.json on one GPU: the closed surface of a 3x3x3 block
of unit cubes with the centre cube removed (mesh.cube_shell_mesh(n): 60 unit
faces x 2 n^2 right triangles; n=64 -> 491 520 triangles, the literal reading;
n=108 -> 1 399 680, the "~1.4M"), single-layer (P0 x P0) and double-layer
(P0 rows x P1 columns) operators, GCA m=4, eta=2, leaf 64, eps_aca 1e-4,
q 3/4, x ~ U(-1,1) seed 4, 100 matvecs per operator.  Bases, nearfield and
couplings are built on the device.

    python tools/config4.py [n]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2001_05523_b200 import clustering as C  # noqa: E402
from paper_2001_05523_b200 import gca, spaces  # noqa: E402
from paper_2001_05523_b200.containers import AssemblyContext  # noqa: E402
from paper_2001_05523_b200.mesh import cube_shell_mesh  # noqa: E402

nc_ = int(sys.argv[1]) if len(sys.argv) > 1 else 64
m, eta, leaf, eps, q_reg, q_ss = 4, 2.0, 64, 1e-4, 3, 4
T = {}


def sync_time(t0):
    torch.cuda.synchronize()
    return round(time.perf_counter() - t0, 3)


t0 = time.perf_counter()
mesh = cube_shell_mesh(nc_)
mesh.validate()
T["mesh_s"] = sync_time(t0)
ctx = AssemblyContext(mesh)
t0 = time.perf_counter()
t_p0 = C.build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), leaf)
t_p1 = C.build_cluster_tree(spaces.DofSpace(spaces.P1, mesh).support_boxes(), leaf)
T["trees_s"] = sync_time(t0)
t0 = time.perf_counter()
b0 = gca.build_basis(ctx, t_p0, gca.P0_SLP, m, eps, device=True)
b1 = gca.build_basis(ctx, t_p1, gca.P1_DLP, m, eps, device=True)
T["bases_device_s"] = sync_time(t0)
out = {"config": f"cube shell n={nc_}: {mesh.n_triangles} triangles, {mesh.n_vertices} vertices; "
                  f"GCA m={m} eta={eta} leaf={leaf} eps={eps}, q {q_reg}/{q_ss}", "setup": T}
pk = bench.peaks()
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for kind, rt, ct, rb, cb in (("slp", t_p0, t_p0, b0, b0), ("dlp", t_p0, t_p1, b0, b1)):
    t0 = time.perf_counter()
    bt = C.BlockTree(rt, ct, eta)
    H = gca.assemble_h2(ctx, kind, bt, rb, cb, q_reg, q_singular=q_ss)
    t_asm = sync_time(t0)
    plan = H.plan()
    nr, ncol = H.shape
    x = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, ncol)).cuda()
    z = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, ncol)).cuda()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for k in range(13):
        flush.fill_(float(k))
        ev[0].record()
        plan.apply_device(x)
        ev[1].record()
        torch.cuda.synchronize()
        if k >= 3:
            ts.append(ev[0].elapsed_time(ev[1]) / 1e3)
    t = float(np.median(ts))
    # the config's 100 matvecs back to back (no flush: what a solver loop sees)
    y = torch.empty(nr, dtype=torch.float64, device="cuda")
    ev[0].record()
    for _ in range(100):
        plan.apply_device(x, y)
    ev[1].record()
    torch.cuda.synchronize()
    t100 = ev[0].elapsed_time(ev[1]) / 1e3
    mv_bytes = H.matvec_bytes()
    y1 = plan.apply_device(x).clone()
    y2 = plan.apply_device(x).clone()
    lin = plan.apply_device(0.7 * x - 1.3 * z) - (0.7 * plan.apply_device(x) - 1.3 * plan.apply_device(z))
    out[kind] = {"rows": int(nr), "cols": int(ncol), "far": int(len(bt.far_uids)), "near": int(len(bt.near_uids)),
                 "assembly_s": t_asm, "matvec_ms": t * 1e3, "dofs_per_s": nr / t, "bytes": mv_bytes,
                 "achieved_gbs": mv_bytes / t / 1e9, "hbm_frac": mv_bytes / t / 1e9 / pk[0],
                 "100_matvecs_ms": t100 * 1e3, "bitwise_repeat": bool(torch.equal(y1, y2)),
                 "linearity_rel": float(lin.norm() / y1.norm())}
    del H, plan
    torch.cuda.empty_cache()
out["memory_gb"] = round(torch.cuda.max_memory_allocated() / 1e9, 2)
print(json.dumps(out), flush=True)
