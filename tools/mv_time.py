"""Time the plan's matvec alone (CUDA events, L2 flushed between launches);
used for A/B runs of library variants (H2B_LIB_PATH) and plan options (env).

    python tools/mv_time.py [config]            config of bench.CONFIGS (host basis)
    python tools/mv_time.py sphere LEVEL M ETA  any sphere, device basis
"""
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

if len(sys.argv) > 1 and sys.argv[1] == "sphere":
    level, m, eta = int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
    mesh = sphere_mesh(level)
    ctx = AssemblyContext(mesh)
    tree = C.build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), 64)
    bt = C.BlockTree(tree, tree, eta)
    basis = gca.build_basis(ctx, tree, gca.P0_SLP, m, 1e-4, device=True)
else:
    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "1"]
    mesh, ctx, tree, bt, basis = bench.build_problem(cfg, os.cpu_count() or 8)
lay = near_layout(bt)
Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
S = assemble_couplings(ctx, "slp", bt, basis, basis, 3)
H = H2Matrix.from_device(bt, basis, basis, S, Dn)
x = torch.randn(H.shape[1], dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
plan = H.plan()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for k in range(105):
    flush.fill_(float(k))
    ev[0].record()
    plan.apply_device(x)
    ev[1].record()
    torch.cuda.synchronize()
    if k >= 5:
        ts.append(ev[0].elapsed_time(ev[1]))
ts = np.sort(ts)[: int(0.8 * len(ts))]  # drop the slowest 20 %; mean resolves below the 2 us event tick
t = float(np.mean(ts)) * 1e-3
b = H.matvec_bytes()
sb = H.streamed_bytes()
print(f"matvec {t*1e6:.1f} us (mean of fastest {len(ts)}), {b/t/1e9:.0f} GB/s algorithmic = "
      f"{b/t/1e9/bench.peaks()[0]*100:.1f} % of HBM; streamed {sb/1e6:.1f} MB = {sb/t/1e9:.0f} GB/s")
print("plan", plan.info())
