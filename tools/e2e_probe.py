"""Breakdown of the end-to-end matvec call (host numpy in/out) on config 1."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np
import torch
import bench
from paper_2001_05523_b200.containers import H2Matrix, assemble_couplings, near_layout

cfg = bench.CONFIGS["1"]
mesh, ctx, tree, bt, basis = bench.build_problem(cfg, os.cpu_count() or 8)
lay = near_layout(bt)
Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
S = assemble_couplings(ctx, "slp", bt, basis, basis, cfg["q_reg"])
H = H2Matrix.from_device(bt, basis, basis, S, Dn)
plan = H.plan()
n = H.shape[0]
xh = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).pin_memory().numpy()
xd = torch.from_numpy(xh).cuda()
yd = torch.empty(n, dtype=torch.float64, device="cuda")
yp = torch.empty(n, dtype=torch.float64).pin_memory()


def wall(f, k=200):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k * 1e6


print(f"H.matvec(numpy)           {wall(lambda: H.matvec(xh)):7.1f} us")
print(f"plan.apply(numpy)         {wall(lambda: plan.apply(xh)):7.1f} us")
print(f"kernel (apply_device)+sync {wall(lambda: (plan.apply_device(xd, yd), torch.cuda.synchronize())):7.1f} us")
print(f"H2D pinned 262KB + sync    {wall(lambda: (xd.copy_(torch.from_numpy(xh), non_blocking=True), torch.cuda.synchronize())):7.1f} us")
print(f"D2H pinned + sync          {wall(lambda: (yp.copy_(yd, non_blocking=True), torch.cuda.synchronize())):7.1f} us")
print(f"np.empty + D2H pageable    {wall(lambda: torch.from_numpy(np.empty(n)).copy_(yd)):7.1f} us")
