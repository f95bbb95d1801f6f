"""Block product throughput: H2Matrix.matmat on nrhs right-hand sides vs nrhs
single-vector matvecs (L2 flushed before each timed call).  Reports
DoF*rhs/s and the HBM roofline of the operator stream (the operator bytes of
one matvec, read once per block).

    python tools/matmat_time.py [config|sphere LEVEL M ETA] [nrhs ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2001_05523_b200 import clustering as C  # noqa: E402
from paper_2001_05523_b200 import gca, spaces  # noqa: E402
from paper_2001_05523_b200.containers import AssemblyContext, H2Matrix, assemble_couplings, near_layout  # noqa: E402
from paper_2001_05523_b200.mesh import sphere_mesh  # noqa: E402

args = sys.argv[1:]
if args and args[0] == "sphere":
    level, m, eta = int(args[1]), int(args[2]), float(args[3])
    mesh = sphere_mesh(level)
    ctx = AssemblyContext(mesh)
    tree = C.build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), 64)
    bt = C.BlockTree(tree, tree, eta)
    basis = gca.build_basis(ctx, tree, gca.P0_SLP, m, 1e-4, device=True)
    name, rest = f"sphere L{level} m={m} eta={eta}", args[4:]
else:
    cfg = bench.CONFIGS[args[0] if args else "1"]
    mesh, ctx, tree, bt, basis = bench.build_problem(cfg, os.cpu_count() or 8)
    name, rest = cfg["desc"], args[1:]
lay = near_layout(bt)
Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
S = assemble_couplings(ctx, "slp", bt, basis, basis, 3)
H = H2Matrix.from_device(bt, basis, basis, S, Dn)
n = H.shape[0]
plan = H.plan()
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn, reps=30):
    ts = []
    for k in range(reps):
        flush.fill_(float(k))
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]) / 1e3)
    ts = np.sort(ts[5:])[: int(0.8 * (reps - 5))]
    return float(np.mean(ts))


mv_bytes = H.matvec_bytes()
hbm = bench.peaks()[0]
x = torch.randn(n, dtype=torch.float64, device="cuda")
t_mv = timed(lambda: plan.apply_device(x))
res = {"workload": name, "n": n, "matvec_ms": t_mv * 1e3, "matvec_dofs_per_s": n / t_mv, "runs": []}
for nrhs in [int(a) for a in rest] or [8, 16]:
    X = torch.randn((n, nrhs), dtype=torch.float64, device="cuda")
    H.matmat(X)
    t = timed(lambda: H.matmat(X))
    res["runs"].append({"nrhs": nrhs, "ms": t * 1e3, "dof_rhs_per_s": n * nrhs / t,
                        "speedup_vs_matvecs": nrhs * t_mv / t,
                        "operator_gbs": mv_bytes / t / 1e9, "hbm_frac": mv_bytes / t / 1e9 / hbm,
                        "fp64_tflops": 2.0 * (mv_bytes / 8) * nrhs / t / 1e12})
print(json.dumps(res), flush=True)
