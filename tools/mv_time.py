"""Time the plan's matvec alone (CUDA events, L2 flushed between launches);
used for A/B runs of library variants (H2B_LIB_PATH) and plan options (env)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np
import torch
import bench
from paper_2001_05523_b200 import kernels
from paper_2001_05523_b200.containers import H2Matrix, assemble_couplings, near_layout

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "1"]
mesh, ctx, tree, bt, basis = bench.build_problem(cfg, os.cpu_count() or 8)
lay = near_layout(bt)
Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
S = assemble_couplings(ctx, "slp", bt, basis, basis, cfg["q_reg"])
H = H2Matrix.from_device(bt, basis, basis, S, Dn)
x = torch.randn(H.shape[1], dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
plan = H.plan()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for k in range(40):
    flush.fill_(float(k))
    ev[0].record()
    plan.apply_device(x)
    ev[1].record()
    torch.cuda.synchronize()
    if k >= 5:
        ts.append(ev[0].elapsed_time(ev[1]))
print(f"matvec {np.median(ts)*1e3:.1f} us (median of {len(ts)})")
