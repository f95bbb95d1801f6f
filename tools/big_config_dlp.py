"""Config 2 double-layer part on one GPU: P0 rows x P1 columns (sphere level
`argv[1]`, default 8 = 524 288 triangles / 262 146 vertices): operator
assembly through the public API, matvec time vs the HBM roofline, and
size-independent checks (bitwise repeat, linearity)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np
import torch
import bench
from paper_2001_05523_b200 import clustering as C, gca, spaces
from paper_2001_05523_b200.containers import AssemblyContext
from paper_2001_05523_b200.mesh import sphere_mesh

level = int(sys.argv[1]) if len(sys.argv) > 1 else 8
t0 = time.time()
mesh = sphere_mesh(level)
ctx = AssemblyContext(mesh)
t_r = C.build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), 64)
t_c = C.build_cluster_tree(spaces.DofSpace(spaces.P1, mesh).support_boxes(), 64)
bt = C.BlockTree(t_r, t_c, 2.0)
th = os.cpu_count() or 8
rb = gca.build_basis(ctx, t_r, gca.P0_SLP, 4, bench.EPS_ACA, threads=th)
cb = gca.build_basis(ctx, t_c, gca.P1_DLP, 4, bench.EPS_ACA, threads=th)
t_setup = time.time() - t0
torch.cuda.synchronize()
t1 = time.time()
H = gca.assemble_h2(ctx, "dlp", bt, rb, cb, 3, q_singular=5)
torch.cuda.synchronize()
t_asm = time.time() - t1
plan = H.plan()
nr, nc = H.shape
x = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, nc)).cuda()
z = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, nc)).cuda()
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for k in range(25):
    flush.fill_(float(k))
    ev[0].record(); plan.apply_device(x); ev[1].record(); torch.cuda.synchronize()
    if k >= 5:
        ts.append(ev[0].elapsed_time(ev[1]) / 1e3)
t = float(np.median(ts))
mv_bytes = H.matvec_bytes()
y1 = plan.apply_device(x).clone(); y2 = plan.apply_device(x).clone()
lin = plan.apply_device(0.7 * x - 1.3 * z) - (0.7 * plan.apply_device(x) - 1.3 * plan.apply_device(z))
pk = bench.peaks()
print(json.dumps({
    "operator": f"DLP sphere L{level}: {nr} P0 rows x {nc} P1 columns, m=4 eta=2 leaf=64, q 3/5",
    "setup_s": round(t_setup, 1), "assembly_s": round(t_asm, 3),
    "matvec_ms": t * 1e3, "row_dofs_per_s": nr / t, "matvec_bytes": mv_bytes,
    "achieved_gbs": mv_bytes / t / 1e9, "hbm_frac": mv_bytes / t / 1e9 / pk[0],
    "bitwise_repeat": bool(torch.equal(y1, y2)), "linearity_rel": float(lin.norm() / y1.norm()),
}))
