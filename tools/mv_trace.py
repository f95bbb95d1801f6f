"""Per-CTA timeline of one matvec (H2B_TRACE=1): role windows and SM occupancy."""
import os, sys
os.environ["H2B_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import ctypes
import numpy as np
import torch
import bench
from paper_2001_05523_b200 import kernels, _lib
from paper_2001_05523_b200.containers import H2Matrix, assemble_couplings, near_layout

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "1"]
mesh, ctx, tree, bt, basis = bench.build_problem(cfg, os.cpu_count() or 8)
lay = near_layout(bt)
Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
nu = bt.near_uids
jobs = np.stack([tree.start[nu[:, 0]], lay.blk_rows, tree.start[nu[:, 1]], lay.blk_cols, lay.blk_off, lay.blk_ld], 1)
sj = kernels.SlpJobs(ctx.dmesh, cfg["q_reg"], jobs, tree.perm.astype(np.int32), tree.perm.astype(np.int32))
tab = kernels.SingularTable(ctx.dmesh, "slp", cfg["q_ss"])
sj.run(tab, Dn)
S = assemble_couplings(ctx, "slp", bt, basis, basis, cfg["q_reg"])
H = H2Matrix.from_device(bt, basis, basis, S, Dn)
x = torch.randn(H.shape[1], dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
plan = H.plan()
for k in range(5):
    flush.fill_(float(k))
    y = plan.apply_device(x)
torch.cuda.synchronize()
n = 8 * 200000
buf = np.zeros(n, dtype=np.uint64)
_lib.check(_lib.lib().h2b_plan_trace(plan.handle, buf.ctypes.data, n))
total = None
# boundaries appended after 3*total words; find total by scanning: we know c_leaves etc from plan
nt = len(tree.leaf_uids())
# brute: the last 5 written words
nfwd = len(tree.leaf_uids())
# boundaries sit right after the 3*tot per-CTA words; tot is unknown here, scan for it
tot = None
for cand in range(1, n // 8):
    if 8 * cand + 4 < n and buf[8 * cand + 3] == cand and buf[8 * cand + 4] == cand and buf[8 * cand] == nfwd:
        tot = cand
        break
b = buf[8 * tot : 8 * tot + 5].astype(np.int64)
tr = buf[: 8 * tot].reshape(tot, 8).astype(np.int64)
t0 = tr[:, 0].min()
st, en, sm = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, tr[:, 2]
names = ["forward", "bands", "-", "-"]
bounds = [0, int(b[0]), tot, tot, tot]
print(f"matvec span {en.max():.1f} us, CTAs {tot}")
for i, nm in enumerate(names):
    a, z = bounds[i], bounds[i + 1]
    if z <= a:
        continue
    d = en[a:z] - st[a:z]
    print(f"{nm:8s} n={z-a:5d} start [{st[a:z].min():6.1f},{st[a:z].max():6.1f}] end [{en[a:z].min():6.1f},{en[a:z].max():6.1f}] dur mean {d.mean():6.2f} max {d.max():6.2f} sum {d.sum():8.1f}")
# concurrency profile
grid = np.linspace(0, en.max(), 40)
for g in grid[::4]:
    act = [(int(((st[a:z] <= g) & (en[a:z] > g)).sum())) for a, z in zip(bounds[:-1], bounds[1:])]
    print(f"t={g:6.1f} active fwd/near/cpl/desc = {act}")

# phase marks (relative to CTA start), means per role
for i, nm in enumerate(names):
    a, z = bounds[i], bounds[i + 1]
    if z <= a:
        continue
    m = tr[a:z, 3:8]
    ok = m[:, 0] > 0
    if ok.any():
        rel = (m[ok] - tr[a:z, 0][ok, None]) / 1e3
        rel[m[ok] == 0] = np.nan
        print(nm, "marks (us from start):", np.round(np.nanmean(np.where(np.isnan(rel), np.nan, rel), axis=0), 2).tolist())

# concurrency / throughput timeline of band CTAs
a, z = bounds[1], tot
edges = np.arange(0, en.max() + 5, 5.0)
for lo in edges[:-1]:
    hi = lo + 5
    act = ((st[a:z] < hi) & (en[a:z] > lo)).sum()
    fin = ((en[a:z] >= lo) & (en[a:z] < hi)).sum()
    print(f"[{lo:5.0f},{hi:5.0f}) bands active {act:4d} finished {fin:4d}")
