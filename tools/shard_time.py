"""Per-rank device time of the row-sharded matvec at N ranks, measured on ONE
GPU rank by rank (the ranks' kernels do not depend on each other within a
matvec: only the all-gathered inputs connect them, which are prepared here by
running every rank's forward launch first).  Reports, per N, the max over
ranks of (forward launch + pack) + (x_hat import + spanning climbs + bands
launch) -- the kernel part of one matvec on N GPUs, collectives excluded --
and the DoF/s it implies, next to the single-GPU launch.

    python tools/shard_time.py [config] [N ...]     (GPU box; default config 3, N = 1 2 4 8)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2001_05523_b200 import _lib  # noqa: E402
from paper_2001_05523_b200 import distributed as DD  # noqa: E402
from paper_2001_05523_b200.containers import H2Matrix, assemble_couplings, near_layout  # noqa: E402
from paper_2001_05523_b200.containers import assemble_nearfield_device  # noqa: E402

args = sys.argv[1:]
cfg = bench.CONFIGS[args[0] if args else "3"]
worlds = [int(a) for a in args[1:]] or [1, 2, 4, 8]
mesh, ctx, tree, bt, basis = bench.build_problem(cfg, os.cpu_count() or 8)
n = tree.n_dofs
L, st = _lib.lib(), _lib.stream_ptr()
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
x = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).cuda()
xp = x[torch.from_numpy(tree.perm).cuda()]


class _Fake:
    def all_gather_into_tensor(self, buf, loc):
        raise RuntimeError("not used")


def ev(fn, reps=20):
    ts = []
    for k in range(reps + 3):
        flush.fill_(float(k))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if k >= 3:
            ts.append(a.elapsed_time(b) / 1e3)
    return float(np.median(ts))


out = {"workload": cfg["desc"], "n": n, "runs": []}
for world in worlds:
    if world == 1:
        Dn = assemble_nearfield_device(ctx, "slp", bt, cfg["q_reg"], cfg["q_ss"])  # symmetric: streamed once per pair
        S = assemble_couplings(ctx, "slp", bt, basis, basis, cfg["q_reg"])
        H = H2Matrix.from_device(bt, basis, basis, S, Dn)
        p = H.plan()
        t = ev(lambda: p.apply_device(x))
        out["runs"].append({"ranks": 1, "matvec_ms": t * 1e3, "dofs_per_s": n / t})
        print(json.dumps(out["runs"][-1]), flush=True)
        del H, p, S, Dn
        continue
    ranks = []
    for r in range(world):
        sh = DD.RowShard(bt, basis, basis, r, world)
        sh.assemble(ctx, "slp", cfg["q_reg"], cfg["q_ss"])
        full = torch.zeros(world * sh.chunk, dtype=torch.float64, device="cuda")
        full[torch.from_numpy(sh.pad_index).cuda()] = xp
        op = DD.ShardedMatvec(sh, r, world, _Fake(), xhat=True)
        ranks.append((sh, op, full))
    for sh, op, full in ranks:  # the gathered coefficients
        _lib.check(L.h2b_xhat_forward(op.plan.handle, full.data_ptr(), op.xsend.data_ptr(), st))
    recv = torch.cat([op.xsend for _, op, _ in ranks])
    res = []
    for sh, op, full in ranks:
        y = torch.zeros(sh.hi - sh.lo, dtype=torch.float64, device="cuda")
        tf = ev(lambda: L.h2b_xhat_forward(op.plan.handle, full.data_ptr(), op.xsend.data_ptr(), st))
        tm = ev(lambda: L.h2b_xhat_main(op.plan.handle, full.data_ptr(), recv.data_ptr(), y.data_ptr(), st))
        res.append((tf, tm, op.info()["near_bytes"] + op.info()["coupling_bytes"]))
    worst = max(range(world), key=lambda i: res[i][0] + res[i][1])
    t = res[worst][0] + res[worst][1]
    out["runs"].append({"ranks": world, "max_rank_ms": t * 1e3, "forward_ms": res[worst][0] * 1e3,
                        "bands_ms": res[worst][1] * 1e3, "dofs_per_s_kernels": n / t,
                        "per_rank_ms": [round((a + b) * 1e3, 3) for a, b, _ in res],
                        "per_rank_stream_gb": [round(c / 1e9, 3) for _, _, c in res]})
    print(json.dumps(out["runs"][-1]), flush=True)
    del ranks, recv
    torch.cuda.empty_cache()
print(json.dumps(out))
