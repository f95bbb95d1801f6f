"""Save the matvec result of a configuration (seeded x) for a bitwise A/B of two library builds:
    H2B_LIB_PATH=a.so python tools/ab_bits.py 1 out_a.npy; H2B_LIB_PATH=b.so python tools/ab_bits.py 1 out_b.npy
    python tools/ab_bits.py cmp out_a.npy out_b.npy"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np
if sys.argv[1] == "cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    print("bitwise equal" if np.array_equal(a, b) else f"DIFFER: max rel {np.abs(a - b).max() / np.abs(a).max():.3e}")
    sys.exit(0)
import torch, bench
from paper_2001_05523_b200 import kernels
from paper_2001_05523_b200.containers import H2Matrix, assemble_couplings, near_layout, near_slp_jobs
cfg = bench.CONFIGS[sys.argv[1]]
mesh, ctx, tree, bt, basis = bench.build_problem(cfg, os.cpu_count() or 8)
lay = near_layout(bt)
Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
sj = kernels.SlpJobs(ctx.dmesh, cfg["q_reg"], near_slp_jobs(bt), tree.perm.astype(np.int32), tree.perm.astype(np.int32))
tab = kernels.SingularTable(ctx.dmesh, "slp", cfg["q_ss"])
sj.run(tab, Dn)
S = assemble_couplings(ctx, "slp", bt, basis, basis, cfg["q_reg"])
H = H2Matrix.from_device(bt, basis, basis, S, Dn)
x = torch.from_numpy(np.random.default_rng(7).standard_normal(H.shape[1])).cuda()
ys = [H.plan().apply_device(x).cpu().numpy() for _ in range(3)]
assert all(np.array_equal(ys[0], y) for y in ys), "not repeatable"
np.save(sys.argv[2], ys[0])
print("saved", sys.argv[2], float(np.abs(ys[0]).sum()))
