"""Config 3 of BASELINE.json on one GPU: sphere refined 9x (2 097 152
triangles), single-layer operator, GCA m=5, eta=1.5, leaf 64, eps_aca 1e-4,
q 3/4; nearfield assembly, couplings, matvec vs the HBM roofline, and the CG
solve of G x = b with b = P0 load of x1^2 - x2^2 (eps_solver = eps_aca/10,
Jacobi).  Every stage after the mesh runs on the device (GCA basis included).
Size-independent checks: linearity, bitwise repeat, symmetry x.Ay = y.Ax,
residual of the returned solution through an independent matvec.

    python tools/config3.py [level] [m] [eta]
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
from paper_2001_05523_b200 import gca, kernels, solver, spaces  # noqa: E402
from paper_2001_05523_b200.containers import (AssemblyContext, H2Matrix, assemble_couplings,  # noqa: E402
                                              near_layout, near_slp_jobs)
from paper_2001_05523_b200.mesh import sphere_mesh  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 9
m = int(sys.argv[2]) if len(sys.argv) > 2 else 5
eta = float(sys.argv[3]) if len(sys.argv) > 3 else 1.5
q_reg, q_ss, leaf, eps = 3, 4, 64, 1e-4
out = {"config": f"sphere L{level} SLP P0, GCA m={m} eta={eta} leaf={leaf} eps={eps}, q {q_reg}/{q_ss}"}
T = {}


def tick(name, t0):
    torch.cuda.synchronize()
    T[name] = round(time.perf_counter() - t0, 3)


t0 = time.perf_counter()
mesh = sphere_mesh(level)
tick("mesh_s", t0)
t0 = time.perf_counter()
ctx = AssemblyContext(mesh)
tree = C.build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), leaf)
bt = C.BlockTree(tree, tree, eta)
tick("trees_s", t0)
t0 = time.perf_counter()
basis = gca.build_basis(ctx, tree, gca.P0_SLP, m, eps, device=True)
tick("basis_device_s", t0)
n = mesh.n_triangles
out.update(n=int(n), nodes=int(tree.n_nodes), far=int(len(bt.far_uids)), near=int(len(bt.near_uids)),
           rank_mean=float(np.mean([basis.rank[u] for u in range(tree.n_nodes)])),
           rank_max=int(max(basis.rank.values())))

# nearfield (timed on the device)
lay = near_layout(bt)
Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
sj = kernels.SlpJobs(ctx.dmesh, q_reg, near_slp_jobs(bt), tree.perm.astype(np.int32), tree.perm.astype(np.int32))
tab = kernels.SingularTable(ctx.dmesh, "slp", q_ss, compute=False)
tab.compute()
sj.run(tab, Dn)
t_sing = bench.ev_time(torch, tab.compute, 3)
t_reg = bench.ev_time(torch, lambda: sj.run(tab, Dn), 3)
fc = bench.flop_counts(ctx, bt, dict(q_reg=q_reg, q_ss=q_ss), sj)
fp64, _ = bench.measure_fp64_peak()
out["nearfield"] = {"ms": (t_sing + t_reg) * 1e3, "pairs": fc["pairs"], "pairs_per_s": fc["pairs"] / (t_sing + t_reg),
                    "singular_ms": t_sing * 1e3, "regular_ms": t_reg * 1e3,
                    "tflops": (fc["reg_flops"] + fc["sing_flops"]) / (t_sing + t_reg) / 1e12,
                    "fp64_frac": (fc["reg_flops"] + fc["sing_flops"]) / (t_sing + t_reg) / 1e12 / fp64}
t0 = time.perf_counter()
S = assemble_couplings(ctx, "slp", bt, basis, basis, q_reg)
tick("couplings_s", t0)
t0 = time.perf_counter()
H = H2Matrix.from_device(bt, basis, basis, S, Dn)
plan = H.plan()
tick("plan_s", t0)

x = torch.from_numpy(np.random.default_rng(3).standard_normal(n)).cuda()
z = torch.from_numpy(np.random.default_rng(4).standard_normal(n)).cuda()
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for k in range(13):
    flush.fill_(float(k))
    ev[0].record()
    y = plan.apply_device(x)
    ev[1].record()
    torch.cuda.synchronize()
    if k >= 3:
        ts.append(ev[0].elapsed_time(ev[1]) / 1e3)
t = float(np.median(ts))
mv_bytes = H.matvec_bytes()
pk = bench.peaks()
y1 = plan.apply_device(x).clone()
y2 = plan.apply_device(x).clone()
lin = plan.apply_device(0.7 * x - 1.3 * z) - (0.7 * plan.apply_device(x) - 1.3 * plan.apply_device(z))
sym = float(torch.dot(z, plan.apply_device(x)) - torch.dot(x, plan.apply_device(z)))
out["matvec"] = {"ms": t * 1e3, "dofs_per_s": n / t, "bytes": mv_bytes, "achieved_gbs": mv_bytes / t / 1e9,
                 "hbm_frac": mv_bytes / t / 1e9 / pk[0], "bitwise_repeat": bool(torch.equal(y1, y2)),
                 "linearity_rel": float(lin.norm() / y1.norm()),
                 "symmetry_rel": abs(sym) / float(torch.dot(z, y1).abs())}

# CG solve of the Galerkin system (solver.cg, device-resident)
b = spaces.load_vector(spaces.DofSpace(spaces.P0, mesh), lambda X, tt: X[..., 0] ** 2 - X[..., 1] ** 2)
bd = torch.from_numpy(b).cuda()
diag = H.diagonal()
torch.cuda.synchronize()
t0 = time.perf_counter()
res = solver.cg(lambda v: plan.apply_device(v), bd, eps / 10.0, 2000, precond_diag=diag)
torch.cuda.synchronize()
t_cg = time.perf_counter() - t0
chk = float((plan.apply_device(res.x) - bd).norm() / bd.norm())
out["cg"] = {"iterations": res.iterations, "converged": res.converged, "residual": res.residual,
             "independent_residual": chk, "s": round(t_cg, 3), "ms_per_iteration": t_cg / res.iterations * 1e3}
out["setup"] = T
out["memory_gb"] = round(torch.cuda.max_memory_allocated() / 1e9, 2)
print(json.dumps(out), flush=True)
