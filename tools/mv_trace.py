"""Per-CTA timeline of one matvec (H2B_TRACE=1): role windows and SM occupancy."""
import os, sys
os.environ["H2B_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import ctypes
import numpy as np
from paper_2001_05523_b200.containers import near_slp_jobs
import torch
import bench
from paper_2001_05523_b200 import kernels, _lib
from paper_2001_05523_b200.containers import H2Matrix, assemble_couplings, near_layout

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "1"]
mesh, ctx, tree, bt, basis = bench.build_problem(cfg, os.cpu_count() or 8)
lay = near_layout(bt)
Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
nu = bt.near_uids
jobs = near_slp_jobs(bt)
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
info = plan.info()
n = 8 * (info['near_tasks'] + info['coupling_tasks'] + len(tree.leaf_uids()) + 64)
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
tr = buf[: 8 * tot].reshape(tot, 8).astype(np.int64)
t0 = tr[:, 0].min()
st, en = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3
kind = (tr[:, 2] >> 16) & 0xff
nclimb = (tr[:, 2] >> 24) & 0xff
print(f"matvec span {en.max():.1f} us, tasks {tot}")
for kd, nm in ((2, "forward"), (0, "near"), (1, "coupling"), (3, "descent"), (4, "nearsym")):
    sel = kind == kd
    if not sel.any():
        continue
    d = en[sel] - st[sel]
    print(f"{nm:8s} n={sel.sum():5d} start [{st[sel].min():6.1f},{st[sel].max():6.1f}] end [{en[sel].min():6.1f},{en[sel].max():6.1f}] dur mean {d.mean():6.2f} max {d.max():6.2f}")
    m = tr[sel, 3:8].astype(np.float64)
    m[m == 0] = np.nan
    dm = np.diff(np.concatenate([tr[sel, 0:1].astype(np.float64), m], axis=1), axis=1)
    with np.errstate(all="ignore"):
        print(f"{'':8s} phase ns (start->m0->..->m4):", np.round(np.nanmean(dm, axis=0), 0).tolist())
sel = kind == 2
for c in range(int(nclimb[sel].max()) + 1 if sel.any() else 0):
    m = sel & (nclimb == c)
    if m.any():
        print(f"forward climb {c:2d}: n={m.sum():4d} dur mean {(en[m]-st[m]).mean():6.2f} us, end max {en[m].max():6.1f}")
is_last = (tr[:, 2] >> 41) & 1
ddepth = (tr[:, 2] >> 32) & 0xff
sel = ((kind == 1) | (kind == 3)) & (is_last == 1)
for dd in range(int(ddepth[sel].max()) + 1 if sel.any() else 0):
    m = sel & (ddepth == dd)
    if m.any():
        mk = tr[m, 3:8].astype(np.float64)
        mk[mk == 0] = np.nan
        with np.errstate(all="ignore"):
            ph = np.round(np.nanmean(mk - tr[m, 0:1], axis=0) / 1e3, 2).tolist()
        print(f"descent depth {dd:2d}: n={m.sum():4d} start [{st[m].min():6.1f},{st[m].max():6.1f}] end [{en[m].min():6.1f},{en[m].max():6.1f}] dur mean {(en[m]-st[m]).mean():5.2f} marks(us from start: ycpl, E-step, store, -, parent) {ph}")
edges = np.arange(0, en.max() + 5, 5.0)
for lo in edges[:-1]:
    hi = lo + 5
    row = []
    for kd in (2, 0, 1, 3):
        sel = (kind == kd) | ((kind == 4) & (kd == 0))
        row.append(int(((en[sel] >= lo) & (en[sel] < hi)).sum()))
    print(f"[{lo:5.0f},{hi:5.0f}) finished fwd/near/cpl/desc {row}")
