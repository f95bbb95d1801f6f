"""Small driver for profiling: build config 1 (or --config) once, run a few
nearfield assemblies and matvecs (no timing).  Used under ncu."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np
from paper_2001_05523_b200.containers import near_slp_jobs
import torch
import bench
from paper_2001_05523_b200 import kernels
from paper_2001_05523_b200.containers import H2Matrix, assemble_couplings, near_layout

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="1")
ap.add_argument("--matvecs", type=int, default=3)
ap.add_argument("--nearfield", type=int, default=1)
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
mesh, ctx, tree, bt, basis = bench.build_problem(cfg, os.cpu_count() or 8)
lay = near_layout(bt)
Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
nu = bt.near_uids
jobs = near_slp_jobs(bt)
sj = kernels.SlpJobs(ctx.dmesh, cfg["q_reg"], jobs, tree.perm.astype(np.int32), tree.perm.astype(np.int32))
tab = kernels.SingularTable(ctx.dmesh, "slp", cfg["q_ss"], compute=False)
for _ in range(a.nearfield):
    tab.compute(); sj.run(tab, Dn)
S = assemble_couplings(ctx, "slp", bt, basis, basis, cfg["q_reg"])
H = H2Matrix.from_device(bt, basis, basis, S, Dn)
x = torch.randn(H.shape[1], dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for k in range(a.matvecs):
    flush.fill_(float(k))
    y = H.matvec(x)
torch.cuda.synchronize()
print("done", H.shape, float(y.abs().sum()))
