"""Double-layer nearfield quadrature on one GPU (config 2: sphere L8, P0 rows x
P1 columns, q_reg 3, Sauter-Schwab 5): host job building, the Sauter-Schwab
table (k_singular<DLP>) and the regular pair-block kernel with the fused
vertex scatter (k_blocks_dlp), timed separately, against the FP64 roofline
(25 flops per regular evaluation, q_reg^4 evaluations per
(row panel, incident column panel) pair; 51 flops per Sauter-Schwab
evaluation, edge 5 q^4, vertex 2 q^4, identical 0).

    python tools/dlp_nearfield.py [level] [q_reg] [q_ss]
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2001_05523_b200 import _lib  # noqa: E402
from paper_2001_05523_b200 import clustering as C  # noqa: E402
from paper_2001_05523_b200 import device as D  # noqa: E402
from paper_2001_05523_b200 import kernels, spaces  # noqa: E402
from paper_2001_05523_b200.containers import AssemblyContext, _near_blocks, near_layout  # noqa: E402
from paper_2001_05523_b200.mesh import sphere_mesh  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 8
q, qs = (int(sys.argv[2]) if len(sys.argv) > 2 else 3), (int(sys.argv[3]) if len(sys.argv) > 3 else 5)
mesh = sphere_mesh(level)
ctx = AssemblyContext(mesh)
t_r = C.build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), 64)
t_c = C.build_cluster_tree(spaces.DofSpace(spaces.P1, mesh).support_boxes(), 64)
bt = C.BlockTree(t_r, t_c, 2.0)
lay = near_layout(bt)
t0 = time.perf_counter()
packed = kernels.build_dlp_jobs(mesh, _near_blocks(bt, lay))
t_jobs = time.perf_counter() - t0
jobs = packed["jobs"]
pairs = int((jobs[:, 1] * jobs[:, 3]).sum())
# touching (row panel, column panel) incidences inside the jobs (looked up, not integrated)
T = mesh.triangles
touch_inc = 0
for j in jobs:
    rp = packed["row_idx"][j[0] : j[0] + j[1]]
    cp = packed["pan_idx"][j[2] : j[2] + j[3]]
    a, b = T[rp], T[cp]
    touch_inc += int((a[:, None, :, None] == b[None, :, None, :]).any(axis=(2, 3)).sum())
out = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
tab = kernels.SingularTable(ctx.dmesh, "dlp", qs, compute=False)
pp, Q, lam = ctx.dmesh.panel_points(q)
t = {k: D.dev(v) for k, v in packed.items()}
cj = _lib.DlpJobs(len(jobs), t["jobs"].data_ptr(), t["row_idx"].data_ptr(), t["pan_idx"].data_ptr(),
                  t["inc_ptr"].data_ptr(), t["inc"].data_ptr(), t["inc_base"].data_ptr())


def regular():
    _lib.check(_lib.lib().h2b_pair_blocks_dlp(ctypes.byref(ctx.dmesh.c), pp.data_ptr(), lam.data_ptr(), Q,
                                              ctypes.byref(cj), ctypes.byref(tab.touch.c), tab.values_dev.data_ptr(),
                                              out.data_ptr(), D.stream()))


tab.compute()
regular()
t_sing = bench.ev_time(torch, tab.compute, 5)
t_reg = bench.ev_time(torch, regular, 5)
n_id, n_edge, n_vert = (int(c) for c in tab.touch.case_counts)
reg_flops = 25.0 * (pairs - touch_inc) * q**4
sing_flops = 51.0 * (n_edge * 5 + n_vert * 2) * qs**4
fp64, _ = bench.measure_fp64_peak()
print(json.dumps({
    "operator": f"DLP nearfield sphere L{level}: {mesh.n_triangles} P0 rows x {mesh.n_vertices} P1 columns, "
                f"leaf 64, eta 2, q {q}/{qs}",
    "near_blocks": int(len(bt.near_uids)), "entries": int(lay.entries), "jobs": int(len(jobs)),
    "panel_pairs": pairs, "touching_incidences": touch_inc, "host_job_build_s": round(t_jobs, 3),
    "singular": {"ms": t_sing * 1e3, "pairs": int(tab.touch.n_pairs), "tflops": sing_flops / t_sing / 1e12,
                 "fp64_frac": sing_flops / t_sing / 1e12 / fp64},
    "regular": {"ms": t_reg * 1e3, "pairs_per_s": pairs / t_reg, "tflops": reg_flops / t_reg / 1e12,
                "fp64_frac": reg_flops / t_reg / 1e12 / fp64},
    "entries_per_s": lay.entries / (t_sing + t_reg),
    "fp64_frac": (reg_flops + sing_flops) / (t_sing + t_reg) / 1e12 / fp64,
}))
