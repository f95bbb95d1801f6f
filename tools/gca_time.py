"""GCA basis construction: host (reference-identical numpy, thread pool) vs
device (h2b_gca_columns + h2b_gca_aca), pivot agreement, per config.

    python tools/gca_time.py [level leaf m [host]] ...
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2001_05523_b200 import clustering as C  # noqa: E402
from paper_2001_05523_b200 import gca, spaces  # noqa: E402
from paper_2001_05523_b200.containers import AssemblyContext  # noqa: E402
from paper_2001_05523_b200.mesh import sphere_mesh  # noqa: E402

args = sys.argv[1:] or ["6", "64", "4", "host"]
i = 0
while i < len(args):
    level, leaf, m = int(args[i]), int(args[i + 1]), int(args[i + 2])
    host = i + 3 < len(args) and args[i + 3] == "host"
    i += 4 if host else 3
    mesh = sphere_mesh(level)
    ctx = AssemblyContext(mesh)
    tree = C.build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), leaf)
    gca.build_basis(AssemblyContext(sphere_mesh(3)), C.build_cluster_tree(
        spaces.DofSpace(spaces.P0, sphere_mesh(3)).support_boxes(), 16), gca.P0_SLP, m, 1e-4, device=True)  # warm-up
    torch.cuda.synchronize()
    t = time.perf_counter()
    bd = gca.build_basis(ctx, tree, gca.P0_SLP, m, 1e-4, device=True)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t
    out = {"level": level, "n": int(mesh.n_triangles), "leaf": leaf, "m": m, "nodes": int(tree.n_nodes),
           "device_s": round(t_dev, 3),
           "rank_mean": float(np.mean([bd.rank[u] for u in range(tree.n_nodes)]))}
    if host:
        t = time.perf_counter()
        bh = gca.build_basis(ctx, tree, gca.P0_SLP, m, 1e-4, threads=os.cpu_count() or 8)
        out["host_s"] = round(time.perf_counter() - t, 3)
        out["host_threads"] = os.cpu_count()
        out["pivots_identical_frac"] = float(np.mean(
            [bh.rank[u] == bd.rank[u] and np.array_equal(bh.pivots[u], bd.pivots[u]) for u in range(tree.n_nodes)]))
    print(json.dumps(out), flush=True)
