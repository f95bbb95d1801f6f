"""Config 2 (single-layer part, sphere L8, 524 288 triangles) on one GPU:
nearfield assembly, matvec time vs the HBM roofline, and size-independent
checks (linearity, determinism) -- the reference is too slow at this size to
produce goldens."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np
from paper_2001_05523_b200.containers import near_slp_jobs
import torch
import bench
from paper_2001_05523_b200 import kernels
from paper_2001_05523_b200.containers import H2Matrix, assemble_couplings, near_layout

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "2s"]
t0 = time.time()
mesh, ctx, tree, bt, basis = bench.build_problem(cfg, os.cpu_count() or 8)
t_setup = time.time() - t0
lay = near_layout(bt)
Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
nu = bt.near_uids
jobs = near_slp_jobs(bt)
sj = kernels.SlpJobs(ctx.dmesh, cfg["q_reg"], jobs, tree.perm.astype(np.int32), tree.perm.astype(np.int32))
tab = kernels.SingularTable(ctx.dmesh, "slp", cfg["q_ss"], compute=False)
for _ in range(2):
    tab.compute(); sj.run(tab, Dn)
t_sing = bench.ev_time(torch, tab.compute, 5)
t_reg = bench.ev_time(torch, lambda: sj.run(tab, Dn), 5)
fc = bench.flop_counts(ctx, bt, cfg, sj)
S = assemble_couplings(ctx, "slp", bt, basis, basis, cfg["q_reg"])
H = H2Matrix.from_device(bt, basis, basis, S, Dn)
plan = H.plan()
n = H.shape[0]
x = torch.from_numpy(np.random.default_rng(cfg["seed"]).standard_normal(n)).cuda()
z = torch.from_numpy(np.random.default_rng(cfg["seed"] + 1).standard_normal(n)).cuda()
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for k in range(25):
    flush.fill_(float(k))
    ev[0].record(); y = plan.apply_device(x); ev[1].record(); torch.cuda.synchronize()
    if k >= 5:
        ts.append(ev[0].elapsed_time(ev[1]) / 1e3)
t = float(np.median(ts))
mv_bytes = H.matvec_bytes()
y1 = plan.apply_device(x).clone(); y2 = plan.apply_device(x).clone()
lin = plan.apply_device(0.7 * x - 1.3 * z) - (0.7 * plan.apply_device(x) - 1.3 * plan.apply_device(z))
pk = bench.peaks()
print(json.dumps({
    "config": cfg["desc"], "n": n, "setup_s": round(t_setup, 1),
    "matvec_ms": t * 1e3, "dofs_per_s": n / t, "matvec_bytes": mv_bytes, "achieved_gbs": mv_bytes / t / 1e9,
    "hbm_frac": mv_bytes / t / 1e9 / pk[0],
    "nearfield_ms": (t_sing + t_reg) * 1e3, "pairs_per_s": fc["pairs"] / (t_sing + t_reg),
    "singular_ms": t_sing * 1e3, "regular_ms": t_reg * 1e3, "evaluated_regular": fc["regular_evaluated"],
    "nearfield_tflops": (fc["reg_flops"] + fc["sing_flops"]) / (t_sing + t_reg) / 1e12,
    "bitwise_repeat": bool(torch.equal(y1, y2)),
    "linearity_rel": float(lin.norm() / y1.norm()),
}))
