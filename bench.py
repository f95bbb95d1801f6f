"""Benchmark: H^2-matvec DoF/s + nearfield quadrature pairs/s, fp64, B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 3]

Workload (default, BASELINE.json configs[3] -- the configuration the metric
is quoted on at 1/2/4/8 GPUs; it fits one GPU): sphere refined 9x
(2 097 152 triangles), piecewise-constant single-layer operator, GCA H^2 with
m = 5, eta = 1.5, leaf 64, eps_aca = 1e-4 (reference default), regular Gauss
order 3, Sauter-Schwab order 4; x ~ N(0,1) seed 3; CG right-hand side the P0
load of x1^2 - x2^2.  Synthetic mesh, no dataset.  The GCA basis is built on
the device (k_gca_columns + k_gca_aca); its per-cluster agreement with the
reference's own basis is reported (tests/golden/cfg3_basis.npz).

A step is one H^2 matvec y = A x (inputs resident in HBM; 14.9 GB of operator
per matvec, far above the 126 MB L2, and L2 flushed by a 256 MiB write
between steps).  `value` = DoF x K / (sum of step times), max over ranks.
The nearfield assembly (touching-pair classification, Sauter-Schwab table,
regular pair blocks) and the coupling assembly are timed in the same run
(`nearfield`, pairs/s, FP64 roofline), and so is the CG solve (`cg`).  `e2e`
is the same matvec through the public API on a plain (pageable) numpy vector
-- the call a reference user makes: H2Matrix.matvec(x) with the H2D copy,
the kernel and the D2H copy inside the timed region.

Multi-GPU: `--gpus N` launches N ranks itself (torch.distributed.run) unless
WORLD_SIZE is set, in which case it must equal N.  Rows are sharded by
contiguous row-leaf ranges (distributed.RowShard): each rank assembles and
stores only its own share of the operator (nearfield, couplings, touching
pairs), x is all-gathered over NCCL once per matvec, each rank writes its own
rows; weak in memory, strong in work ("scaling": "strong": the problem is
fixed); timing = max over ranks; CG with all-reduced scalars.

--impl reference: the reference's CPU algorithm on this host's cores (the
oracle port in oracle/: the reference cannot travel to the GPU box), on the
same configuration, through oracle code only (it never imports
paper_2001_05523_b200): structure by oracle/structure.py (pinned bit-exact
to the reference), each step the reference matvec restricted to bounded row
slices (oracle.h2.RowSlice, one slice per core in parallel), plus a seeded
sample of near blocks through the oracle quadrature.
"""

import argparse
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

CONFIGS = {
    # name: level, leaf, eta, m, q_reg, q_ss, kind, seed, dist, basis
    "3": dict(level=9, leaf=64, eta=1.5, m=5, q_reg=3, q_ss=4, kind="slp", seed=3, dist="normal", basis="device",
              golden="cfg3_basis.npz",
              desc="config 3: sphere L9 (2097152 tri) SLP P0, GCA m=5 eta=1.5 leaf=64 eps=1e-4, q 3/4, CG"),
    "1": dict(level=6, leaf=64, eta=2.0, m=4, q_reg=3, q_ss=4, kind="slp", seed=1, dist="normal", basis="host",
              golden="h2_cfg1.npz",
              desc="config 1: sphere L6 (32768 tri) SLP P0, GCA m=4 eta=2 leaf=64 eps=1e-4, q 3/4"),
    "0": dict(level=4, leaf=32, eta=2.0, m=3, q_reg=3, q_ss=4, kind="slp", seed=0, dist="uniform", basis="host",
              golden="h2_cfg0.npz",
              desc="config 0: sphere L4 (2048 tri) SLP P0, GCA m=3 eta=2 leaf=32 eps=1e-4, q 3/4"),
    "2s": dict(level=8, leaf=64, eta=2.0, m=4, q_reg=3, q_ss=5, kind="slp", seed=2, dist="uniform", basis="device",
               golden=None,
               desc="config 2 (single layer): sphere L8 (524288 tri) SLP P0, GCA m=4 eta=2 leaf=64 eps=1e-4, q 3/5"),
}
DEFAULT_CONFIG = "3"
EPS_ACA = 1e-4
METRIC = "H2-matvec DoF/s (fp64), + nearfield quad pairs/s"
PROFILE = os.path.join(ROOT, "profiles", "r02bx_ncu_full_raw.csv")


# ---------------------------------------------------------------------------
# measurement helpers

def peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        return 6650.0, "B200_PROFILING.md fallback"


def measure_fp64_peak():
    """DFMA-chain microbenchmark (tools/fp64_probe) run live on this GPU."""
    exe = os.path.join(ROOT, "tools", "_bin", "fp64_probe")
    if os.path.exists(exe):
        try:
            out = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout
            return float(json.loads(out.strip().splitlines()[-1])["fp64_dfma_tflops"]), "tools/fp64_probe (measured live)"
        except Exception:
            pass
    return 34.23, "profiles/r01_fp64_probe.json (measured earlier on this pool)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks
    line).  One sampler per run: sub-intervals are cut out of its record by
    timestamp (mark / stop(t0, t1)) -- a second nvidia-smi would double the
    perturbation, and its start-up (NVML init) stalls driver calls for tens of
    milliseconds."""

    def __init__(self, gpu_index=0):
        self.proc = None
        self.path = f"/tmp/h2b_clocks_{os.getpid()}.csv"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={gpu_index}",
                 "--query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    @staticmethod
    def mark():
        return time.time()

    def stop(self, t0=None, t1=None):
        """Stop the sampler (first call) and summarise the samples, all of
        them or those stamped within [t0, t1] (time.time() values)."""
        import datetime

        if self.proc is None:
            return None
        if self.proc.poll() is None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            if t0 is not None:
                try:
                    ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    continue
                if ts < t0 - 0.05 or ts > t1 + 0.05:
                    continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(kernel, path=PROFILE):
    """DRAM bytes (read + write) of one launch of `kernel` in the committed
    ncu --set full capture (profiles/), or None."""
    import csv

    if not os.path.exists(path):
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    with open(path) as f:
        rows = list(csv.reader(f))
    if len(rows) < 3:
        return None
    head, units = rows[0], rows[1]
    try:
        ik = head.index("Kernel Name")
        ir, iw = head.index("dram__bytes_read.sum"), head.index("dram__bytes_write.sum")
    except ValueError:
        return None
    for r in rows[2:]:
        if kernel in r[ik]:
            return float(r[ir].replace(",", "")) * scale.get(units[ir], 1) + \
                float(r[iw].replace(",", "")) * scale.get(units[iw], 1)
    return None


def ev_time(torch, fn, reps=1):
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / reps


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def h2b_env():
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("H2B_")}


def draw_x(cfg, n):
    rng = np.random.default_rng(cfg["seed"])
    return rng.standard_normal(n) if cfg["dist"] == "normal" else rng.uniform(-1.0, 1.0, n)


# ---------------------------------------------------------------------------
# our arm

def flop_counts(table_pairs, slp_jobs, cfg):
    """SURVEY.md 8(d) convention: 12 flops per regular SLP kernel evaluation,
    36 per Sauter-Schwab evaluation; pair counts as integrated (the symmetric
    single-layer matrix integrates one pair per entry pair)."""
    n_id, n_edge, n_vert = table_pairs
    q, qs = cfg["q_reg"], cfg["q_ss"]
    touch_eval = n_id + n_edge + n_vert
    reg_eval = slp_jobs.evaluated - touch_eval
    ev_sing = n_id * 6 * qs**4 + n_edge * 2 * 5 * qs**4 + n_vert * 2 * 2 * qs**4
    return dict(regular_evaluated=reg_eval, singular_evaluated=touch_eval, reg_flops=12.0 * reg_eval * q**4,
                sing_flops=36.0 * ev_sing)


def build_problem(cfg, threads):
    """Mesh, assembly context, cluster tree, block tree and GCA basis of a
    configuration (tools/ profiling drivers; run_ours times the same steps)."""
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import gca, spaces
    from paper_2001_05523_b200.containers import AssemblyContext
    from paper_2001_05523_b200.mesh import sphere_mesh

    mesh = sphere_mesh(cfg["level"])
    ctx = AssemblyContext(mesh)
    tree = C.build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), cfg["leaf"])
    bt = C.BlockTree(tree, tree, cfg["eta"])
    basis = gca.build_basis(ctx, tree, gca.P0_SLP, cfg["m"], EPS_ACA, device=cfg["basis"] == "device",
                            threads=threads)
    return mesh, ctx, tree, bt, basis


def run_ours(args, cfg):
    import torch

    ws, rank, local = dist_env()
    backend = os.environ.get("H2B_DIST_BACKEND", "nccl")
    if backend != "nccl":  # orchestration check on fewer GPUs (not a measurement)
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as tdist

        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(backend)
        dist = tdist
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import distributed as DD
    from paper_2001_05523_b200 import gca, kernels, solver, spaces
    from paper_2001_05523_b200.containers import (AssemblyContext, H2Matrix, assemble_couplings,
                                                  assemble_nearfield_sharded, coupling_slp_jobs, near_layout,
                                                  near_slp_jobs, near_slp_jobs_sharded)
    from paper_2001_05523_b200.mesh import sphere_mesh

    torch.cuda.reset_peak_memory_stats()
    threads = max(1, (os.cpu_count() or 8) // ws)
    T = {}
    t0 = time.perf_counter()
    mesh = sphere_mesh(cfg["level"])
    T["mesh_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ctx = AssemblyContext(mesh)
    tree = C.build_cluster_tree(spaces.DofSpace(spaces.P0, mesh).support_boxes(), cfg["leaf"])
    bt = C.BlockTree(tree, tree, cfg["eta"])
    T["trees_s"] = time.perf_counter() - t0
    device_basis = cfg["basis"] == "device"
    if device_basis:
        gca.build_basis(ctx, tree, gca.P0_SLP, cfg["m"], EPS_ACA, device=True)  # warm (first-use costs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    basis = gca.build_basis(ctx, tree, gca.P0_SLP, cfg["m"], EPS_ACA, device=device_basis, threads=threads)
    torch.cuda.synchronize()
    T["basis_s"] = time.perf_counter() - t0
    n = tree.n_dofs
    perm = tree.perm

    shard = DD.RowShard(bt, basis, basis, rank, ws) if ws > 1 else None
    view = shard.view if shard is not None else bt
    lo, hi = (shard.lo, shard.hi) if shard is not None else (0, n)

    # ---- nearfield assembly on the device (timed) ----------------------------
    clocks = Clocks(local)
    time.sleep(1.0)  # nvidia-smi's start-up (NVML init) stalls driver calls for tens of ms: keep it out of the timings
    dm = ctx.dmesh
    kernels.TouchTable(dm)  # warm-up (allocator)
    t_touch = ev_time(torch, lambda: kernels.TouchTable(dm), 3)  # classification of all touching pairs
    dm.touch()
    table = kernels.SingularTable(dm, "slp", cfg["q_ss"], compute=False)
    own = shard.own_panels if shard is not None else None
    jobs = near_slp_jobs_sharded(view) if shard is not None else near_slp_jobs(bt)
    sj = kernels.SlpJobs(dm, cfg["q_reg"], jobs, perm.astype(np.int32), perm.astype(np.int32))
    lay = near_layout(view)
    Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
    for _ in range(2):
        table.compute(own)
        sj.run(table, Dn)
    nf_reps = 3 if n > 1_000_000 else 10
    nf_m0 = clocks.mark()  # clocks during the FP64-bound quadrature alone: a slice of the one sampler's record
    t_sing = ev_time(torch, lambda: table.compute(own), nf_reps)
    t_reg = ev_time(torch, lambda: sj.run(table, Dn), nf_reps)
    t_reg_each = [ev_time(torch, lambda: sj.run(table, Dn), 1) for _ in range(nf_reps)]
    nf_m1 = clocks.mark()
    touch = dm.touch()
    if own is not None:
        touch.subset(own, half=True)
        so = touch._subset[3]
        case = (int(so[1] - so[0]), int(so[2] - so[1]), int(so[3] - so[2]))
    else:
        touch.ensure_half()
        ho = touch.half_off
        case = (int(ho[1] - ho[0]), int(ho[2] - ho[1]), int(ho[3] - ho[2]))
    fc = flop_counts(case, sj, cfg)
    near_pairs = lay.entries
    # couplings: end to end (host job list + kernel) and the kernel alone
    t1 = time.perf_counter()
    S = assemble_couplings(ctx, "slp", view, basis, basis, cfg["q_reg"])
    torch.cuda.synchronize()
    t_cpl_e2e = time.perf_counter() - t1
    cj, rp, cp, flay = coupling_slp_jobs(view, basis, basis)
    cjobs = kernels.SlpJobs(dm, cfg["q_reg"], cj, rp, cp)
    Sc = torch.zeros_like(S)
    cjobs.run(None, Sc)
    t_cpl = ev_time(torch, lambda: cjobs.run(None, Sc), nf_reps)
    assert torch.equal(Sc, S)
    cpl_pairs = flay.entries
    cpl_flops = 12.0 * cjobs.evaluated * cfg["q_reg"] ** 4

    # ---- operator + matvec ------------------------------------------------------
    if shard is not None:
        shard.S, shard.D = S, Dn
        # the timed assembly above is the rank's sharded assembly; check it is
        assert torch.equal(Dn, assemble_nearfield_sharded(ctx, "slp", view, cfg["q_reg"], cfg["q_ss"], own))
        # H2B_COMM=native: the x all-gather runs inside the C-ABI call
        # (h2b_plan_set_comm + h2b_matvec_sharded, libh2b's own NCCL
        # communicator); default: torch.distributed's all_gather_into_tensor
        comm = DD.NativeComm(rank, ws, local, dist) if os.environ.get("H2B_COMM") == "native" else None
        # the x_hat exchange (SURVEY 8(e) better variant: each rank
        # forward-transforms only its own column subtrees, coefficients
        # all-gathered) unless H2B_XHAT=0
        xhat = os.environ.get("H2B_XHAT", "1") != "0" and comm is None
        op = DD.ShardedMatvec(shard, rank, ws, dist, comm=comm, xhat=xhat)
        plan = op.plan
        H = None
    else:
        H = H2Matrix.from_device(bt, basis, basis, S, Dn)
        op = DD.LocalMatvec(H)
        plan = op.plan
    info = plan.info()
    x_host = draw_x(cfg, n)
    x = torch.from_numpy(x_host).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    warm = max(args.warmup, 3)
    for _ in range(warm):
        op.apply(x, y)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    K = args.steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    torch.cuda.synchronize()
    for k in range(K):
        flush.fill_(float(k))
        starts[k].record()
        op.apply(x, y)
        ends[k].record()
    torch.cuda.synchronize()
    step_s = np.array([s.elapsed_time(e) / 1e3 for s, e in zip(starts, ends)])
    # the kernel alone (k_matvec: one launch per step), same stream
    from paper_2001_05523_b200 import _lib

    xin = op.xbuf if shard is not None else x
    yout = op.yloc if shard is not None else y
    kst = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ken = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    for k in range(K):
        flush.fill_(float(k))
        kst[k].record()
        if shard is not None and op.xhat:  # the bands launch (+ x_hat import) of the x_hat exchange
            _lib.check(_lib.lib().h2b_xhat_main(plan.handle, xin.data_ptr(), op.xrecv.data_ptr(), yout.data_ptr(),
                                                _lib.stream_ptr()))
        else:
            _lib.check(_lib.lib().h2b_matvec(plan.handle, xin.data_ptr(), yout.data_ptr(), _lib.stream_ptr()))
        ken[k].record()
    torch.cuda.synchronize()
    kern_s = float(np.mean([s.elapsed_time(e) / 1e3 for s, e in zip(kst, ken)]))
    clk = clocks.stop()
    nf_clk = clocks.stop(nf_m0, nf_m1)
    total = float(step_s.sum())
    tmax = {"total": total, "touch": t_touch, "sing": t_sing, "reg": t_reg, "cpl": t_cpl, "cpl_e2e": t_cpl_e2e}
    sums = {"near_pairs": float(near_pairs), "cpl_pairs": float(cpl_pairs),
            "flops": fc["reg_flops"] + fc["sing_flops"], "cpl_flops": cpl_flops}
    if dist:
        tt = torch.tensor(list(tmax.values()), dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tmax = dict(zip(tmax, tt.tolist()))
        ss = torch.tensor(list(sums.values()), dtype=torch.float64, device="cuda")
        dist.all_reduce(ss, op=dist.ReduceOp.SUM)
        sums = dict(zip(sums, ss.tolist()))
    mean_step = tmax["total"] / K
    dofs_per_s = n * K / tmax["total"]

    # ---- e2e through the public API ------------------------------------------
    e2e = None
    if ws == 1:
        xh = np.ascontiguousarray(x_host)  # plain pageable numpy: the reference caller's vector
        for _ in range(5):
            yh = H.matvec(xh)  # keeps the previous result alive, as the timed loop does: both pinned blocks exist
        ke = max(10, min(K, 50))
        import gc

        gc.collect()  # a full collection over the setup's ~1e6 objects inside the loop costs 10+ ms
        each = []
        t1 = time.perf_counter()
        for _ in range(ke):
            t2 = time.perf_counter()
            yh = H.matvec(xh)
            each.append(time.perf_counter() - t2)
        dt = time.perf_counter() - t1
        xpin = torch.from_numpy(x_host).pin_memory().numpy()
        for _ in range(3):
            H.matvec(xpin)
        t1 = time.perf_counter()
        for _ in range(ke):
            H.matvec(xpin)
        dtp = time.perf_counter() - t1
        e2e = {"value": n * ke / dt, "unit": "DoF/s", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
               "timer": "host wall clock around H2Matrix.matvec(numpy, pageable) incl. H2D/D2H, synchronised",
               "calls": ke, "ms_per_call": {"mean": dt / ke * 1e3, "median": float(np.median(each)) * 1e3,
                                            "min": float(np.min(each)) * 1e3, "max": float(np.max(each)) * 1e3},
               "pinned_input_value": n * ke / dtp}
        del yh
    else:
        xp = torch.from_numpy(x_host).pin_memory()
        yp = torch.empty(hi - lo, dtype=torch.float64).pin_memory()
        xd = torch.empty_like(x)

        def e2e_step():
            xd.copy_(xp, non_blocking=True)
            op.apply(xd, y)
            yp.copy_(y[op.perm_dev], non_blocking=True)
            torch.cuda.synchronize()

        for _ in range(3):
            e2e_step()
        dist.barrier()
        ke = max(10, min(K, 50))
        t1 = time.perf_counter()
        for _ in range(ke):
            e2e_step()
        dt = torch.tensor([time.perf_counter() - t1], dtype=torch.float64, device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": n * ke / float(dt.item()), "unit": "DoF/s", "h2d_bytes_per_step": 8 * n,
               "d2h_bytes_per_step": 8 * (hi - lo),
               "timer": "host wall clock per rank around H2D of x (pinned) + ShardedMatvec.apply + D2H of own "
                        "rows, max over ranks"}

    # ---- CG solve of the Galerkin system --------------------------------------
    b = spaces.load_vector(spaces.DofSpace(spaces.P0, mesh), lambda X, tt: X[..., 0] ** 2 - X[..., 1] ** 2)
    if ws == 1:
        bd = torch.from_numpy(b).cuda()
        diag = H.diagonal()
        run_cg = lambda: solver.cg(plan.apply_device, bd, EPS_ACA / 10.0, 2000, precond_diag=diag)  # noqa: E731
    else:
        bd = torch.from_numpy(b[perm[lo:hi]].copy()).cuda()
        dloc = op.diagonal_local()
        red = DD.allreduce_sum(dist)
        run_cg = lambda: solver.cg(op.apply_local, bd, EPS_ACA / 10.0, 2000, precond_diag=dloc,  # noqa: E731
                                   allreduce=red)
    run_cg()  # warm
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t1 = time.perf_counter()
    res = run_cg()
    torch.cuda.synchronize()
    t_cg = time.perf_counter() - t1
    if dist:
        tt = torch.tensor([t_cg], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_cg = float(tt.item())
    cg = {"iterations": res.iterations, "converged": res.converged, "residual": res.residual, "s": t_cg,
          "ms_per_iteration": t_cg * 1e3 / max(res.iterations, 1),
          "rhs": "P0 load of x1^2 - x2^2, Jacobi, eps_solver = eps_aca / 10 (solver.cg, device-resident)"}

    # ---- rooflines -------------------------------------------------------------
    hbm, hbm_src = peaks()
    fp64_peak, fp64_src = measure_fp64_peak() if rank == 0 else (None, None)
    # every operator entry once, each basis in both roles, x and
    # y -- for this rank: its nearfield + couplings, the whole column basis
    # (forward), its row clusters' basis, all of x, its rows of y
    rflo = basis.storage_floats()
    rb_own = rflo
    if shard is not None:
        own_nodes = set(shard.owned.tolist())
        rb_own = sum(basis.V[u].size for u in basis.V if u in own_nodes) + \
            sum(basis.E[u].size for u in basis.E if u in own_nodes)
    alg_bytes = 8 * (lay.entries + flay.entries + rflo + rb_own + n + (hi - lo))
    streamed = alg_bytes - 8 * (lay.entries + flay.entries) + info["near_bytes"] + info["coupling_bytes"]
    achieved = alg_bytes / kern_s / 1e9
    nf_time = tmax["sing"] + tmax["reg"]
    result = {
        "metric": METRIC,
        "value": dofs_per_s,
        "unit": "DoF/s",
        "n_gpus": ws,
        "steps": K,
        "warmup": warm,
        "ms_per_step": mean_step * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": f"synthetic (generated sphere mesh, x ~ {'N(0,1)' if cfg['dist'] == 'normal' else 'U(-1,1)'} "
                f"seed {cfg['seed']})",
        "config": {"workload": cfg["desc"], "n_dofs": n, "matvec_bytes_algorithmic": alg_bytes if ws == 1 else None,
                   "operator_gb": round(8 * (near_layout(bt).entries + flay.entries) / 1e9, 3) if ws == 1 else None,
                   "l2": "inputs far above L2 (operator streamed from HBM) and L2 flushed (256 MiB write) "
                         "between timed steps",
                   "basis": "device GCA (k_gca_columns + k_gca_aca)" if device_basis else
                            "host GCA (reference-identical pivots)",
                   "parallelism": (f"row-shard x{ws} (sharded assembly + storage, NCCL all-gather of x"
                                   + (" and of the ranks' own x_hat: forward transform split over the ranks)"
                                      if ws > 1 and op.xhat else ")")) if ws > 1 else "single GPU",
                   "env": h2b_env()},
        "gpu_launches": K,
        "roofline": {"bound": "hbm", "kernel": "k_matvec (fused forward + coupling + backward + nearfield)",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": ncu_traffic("k_matvec"),
                     "traffic_source": os.path.relpath(PROFILE, ROOT) + " (ncu --set full, one launch, dram read+write)",
                     "algorithmic_bytes": alg_bytes, "kernel_ms": kern_s * 1e3, "peak_source": hbm_src,
                     "streamed_bytes": streamed, "streamed_gbs": streamed / kern_s / 1e9,
                     "note": "achieved = SURVEY 8(d) algorithmic bytes (every operator entry once) / mean k_matvec "
                             "launch time (CUDA events, rank 0); the plan streams the symmetric single-layer "
                             "nearfield once per block pair (streamed_bytes < algorithmic bytes)"},
        "nearfield": {
            "pairs_per_s": sums["near_pairs"] / nf_time,
            "pairs_per_s_incl_classification": sums["near_pairs"] / (nf_time + tmax["touch"]),
            "pairs": int(sums["near_pairs"]), "ms": nf_time * 1e3, "touch_classify_ms": tmax["touch"] * 1e3,
            "singular": {"ms": tmax["sing"] * 1e3, "pairs_integrated": fc["singular_evaluated"],
                         "tflops": fc["sing_flops"] / t_sing / 1e12,
                         "frac": fc["sing_flops"] / t_sing / 1e12 / fp64_peak if fp64_peak else None},
            "regular": {"ms": tmax["reg"] * 1e3, "pairs_integrated": fc["regular_evaluated"],
                        "tflops": fc["reg_flops"] / t_reg / 1e12,
                        "frac": fc["reg_flops"] / t_reg / 1e12 / fp64_peak if fp64_peak else None,
                        "ms_each_launch": [round(t * 1e3, 3) for t in t_reg_each]},
            "clocks": nf_clk,
            "roofline": {"bound": "fp64", "achieved": sums["flops"] / nf_time / 1e12, "peak": fp64_peak,
                         "unit": "TFLOP/s", "frac": sums["flops"] / nf_time / 1e12 / fp64_peak if fp64_peak else None,
                         "peak_source": fp64_src,
                         "flops": "SURVEY 8(d): 12 per regular, 36 per Sauter-Schwab evaluation, on the pairs "
                                  "integrated (symmetric single layer: one per entry pair)"},
            "couplings": {"pairs": int(sums["cpl_pairs"]), "kernel_ms": tmax["cpl"] * 1e3,
                          "pairs_per_s": sums["cpl_pairs"] / tmax["cpl"],
                          "tflops": sums["cpl_flops"] / tmax["cpl"] / 1e12,
                          "end_to_end_ms": tmax["cpl_e2e"] * 1e3,
                          "note": "S_b = G[pivots_t, pivots_s] (gca.py:194-205); end to end includes the host "
                                  "job list"},
        },
        "e2e": e2e,
        "cg": cg,
        "plan": info,
        "memory_gb_per_rank": round(torch.cuda.max_memory_allocated() / 1e9, 2),
        "clocks": clk,
        "setup": {k: round(v, 3) for k, v in T.items()},
    }
    if device_basis and cfg.get("golden"):
        result["basis_vs_reference"] = basis_agreement(cfg, tree, basis)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(H, cfg, x_host, mesh, budget_s=args.cpu_budget)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def basis_agreement(cfg, tree, basis):
    """Per-cluster agreement of the (device) basis with the reference's own
    GCA basis (rank, and the pivot list by digest), tests/golden/*."""
    import hashlib

    path = os.path.join(ROOT, "tests", "golden", cfg["golden"])
    if not os.path.exists(path):
        return None
    g = np.load(path)
    if "pivot_digest" not in g:
        return None
    ranks = np.array([basis.rank[u] for u in range(tree.n_nodes)])
    dig = np.array([int.from_bytes(hashlib.sha256(np.asarray(basis.pivots[u], dtype=np.int64).tobytes()).digest()[:8],
                                   "little", signed=True) for u in range(tree.n_nodes)], dtype=np.int64)
    return {"clusters": int(tree.n_nodes), "rank_equal_frac": float(np.mean(ranks == g["ranks"])),
            "pivots_equal_frac": float(np.mean(dig == g["pivot_digest"])),
            "source": "tests/golden/" + cfg["golden"] + " (reference gca.build_basis run by make_golden.py)"}


def cpu_baseline(H, cfg, x, mesh, budget_s=15.0):
    """The oracle (numpy restatement of containers.py:254-270) on the SAME
    operator exported from the device, one thread: one full matvec at least;
    plus a seeded sample of near blocks through the oracle quadrature
    (kernels.py:260-468 restated), single thread."""
    from oracle import h2 as OH

    t0 = time.perf_counter()
    bt, b = H.block_tree, H.row_basis
    S = [s for _, s in H.far]
    Dn = [d for _, d in H.near]
    ot = OH.Tree(bt.row_tree.perm, bt.row_tree.start, bt.row_tree.end, bt.row_tree.depth_of, bt.row_tree.left,
                 bt.row_tree.right)
    t_export = time.perf_counter() - t0
    n = H.shape[0]
    k, t = 0, time.perf_counter()
    while True:
        OH.matvec(ot, ot, b.V, b.E, b.rank, b.V, b.E, b.rank, bt.far_uids, S, bt.near_uids, Dn, x)
        k += 1
        if time.perf_counter() - t > budget_s:
            break
    dt = time.perf_counter() - t
    del S, Dn
    out = {"value": n * k / dt, "unit": "DoF/s", "cores": 1, "kind": "port",
           "sample": f"{k} full oracle matvec(s) of the same {n}-DoF operator exported from the device "
                     f"({dt:.1f} s; export {t_export:.1f} s; OPENBLAS_NUM_THREADS=1)"}
    out["nearfield_sample"] = oracle_near_sample(mesh, bt, cfg, budget_s=max(5.0, budget_s / 2))
    out["coupling_sample"] = oracle_coupling_sample(mesh, bt, b, cfg, budget_s=max(3.0, budget_s / 4))
    return out


def oracle_coupling_sample(mesh, bt, basis, cfg, budget_s=4.0, seed=11):
    """Seeded sample of coupling blocks S_b = G[pivots_t, pivots_s]
    (gca.py:194-205) through the oracle's regular tensor rule (require_disjoint:
    no singular table); pairs/s on one thread."""
    from oracle import quad as OQ

    V, T, N, A = mesh.vertices, mesh.triangles, mesh.normals, mesh.areas
    rng = np.random.default_rng(seed)
    order = rng.permutation(len(bt.far_uids))
    pairs = blocks = 0
    t0 = time.perf_counter()
    for i in order:
        if time.perf_counter() - t0 > budget_s:
            break
        t, s_ = bt.far_uids[i]
        rows = np.asarray(basis.pivots[int(t)], dtype=np.int64)
        cols = np.asarray(basis.pivots[int(s_)], dtype=np.int64)
        OQ.slp_block(V, T, N, A, rows, cols, cfg["q_reg"], None)
        pairs += len(rows) * len(cols)
        blocks += 1
    dt = time.perf_counter() - t0
    return {"pairs_per_s": pairs / dt if dt else None, "pairs": pairs, "blocks": blocks, "cores": 1,
            "sample": f"{blocks} seeded random far blocks of {len(bt.far_uids)} (oracle tensor rule, q "
                      f"{cfg['q_reg']}, pivots of the bench's basis)"}


def oracle_near_sample(mesh, bt, cfg, budget_s=8.0, seed=7):
    """Seeded sample of near blocks through the oracle quadrature: touching
    pairs by the Sauter-Schwab restatement (only those of the sampled
    blocks), regular pairs by the tensor rule; pairs/s on one thread."""
    from oracle import quad as OQ

    V, T, N, A = mesh.vertices, mesh.triangles, mesh.normals, mesh.areas
    return _near_sample(V, T, N, A, bt.row_tree, bt.near_uids, cfg, budget_s, seed)


class _PairTable:
    """Singular values of given pairs, looked up like the reference's table."""

    def __init__(self, F, pa, pb, vals):
        self.F = F
        self.keys = pa * F + pb
        o = np.argsort(self.keys)
        self.keys, self.vals = self.keys[o], vals[o]

    def lookup(self, pa, pb):
        return self.vals[np.searchsorted(self.keys, np.asarray(pa) * self.F + np.asarray(pb))]


def _near_sample(V, T, N, A, tree, near_uids, cfg, budget_s, seed):
    from oracle import quad as OQ

    rng = np.random.default_rng(seed)
    order = rng.permutation(len(near_uids))
    F = len(T)
    pairs = blocks = 0
    t_sing = t_reg = 0.0
    for i in order:
        if t_sing + t_reg > budget_s:
            break
        a, s = near_uids[i]
        rows = tree.perm[tree.start[a] : tree.end[a]]
        cols = tree.perm[tree.start[s] : tree.end[s]]
        t1 = time.perf_counter()
        hit = (T[rows][:, None, :, None] == T[cols][None, :, None, :]).any(axis=(2, 3))
        ra, cb = np.nonzero(hit)
        vals = OQ.singular_integrals(V, T, N, A, rows[ra], cols[cb], "slp", cfg["q_ss"])
        t2 = time.perf_counter()
        OQ.slp_block(V, T, N, A, rows, cols, cfg["q_reg"], _PairTable(F, rows[ra], cols[cb], vals))
        t3 = time.perf_counter()
        t_sing += t2 - t1
        t_reg += t3 - t2
        pairs += len(rows) * len(cols)
        blocks += 1
    tt = t_sing + t_reg
    return {"pairs_per_s": pairs / tt if tt else None, "pairs": pairs, "blocks": blocks, "cores": 1,
            "s_singular": round(t_sing, 2), "s_regular": round(t_reg, 2),
            "sample": f"{blocks} seeded random near blocks of {len(near_uids)} (oracle quadrature, q "
                      f"{cfg['q_reg']}/{cfg['q_ss']})"}


# ---------------------------------------------------------------------------
# reference arm (oracle only; never imports paper_2001_05523_b200)

_REF = {}


def _ref_slice(root):
    """Worker: the row slice under `root` with shape-exact seeded values."""
    from oracle import h2 as OH

    st = _REF
    if root not in st.setdefault("slices", {}):
        tree, far, near, rank = st["tree"], st["far"], st["near"], st["rank"]
        size = tree.end - tree.start
        rng = np.random.default_rng(1000 + int(root))

        def V(u):
            return rng.standard_normal((int(size[u]), int(rank[u])))

        def E(u):
            return rng.standard_normal((int(rank[u]), int(rank[tree.parent[u]])))

        def S(i):
            return rng.standard_normal((int(rank[far[i, 0]]), int(rank[far[i, 1]])))

        def Dn(i):
            return rng.standard_normal((int(size[near[i, 0]]), int(size[near[i, 1]])))

        st["slices"][root] = OH.RowSlice(tree, int(root), far, near, rank, V, E, S, Dn)
    return st["slices"][root]


def _ref_step(root):
    sl = _ref_slice(root)
    t = time.perf_counter()
    sl.matvec(_REF["x"])
    return sl.n_rows, time.perf_counter() - t


def _ref_near(args):
    i0, budget = args
    st = _REF
    V, T, N, A = st["mesh"]
    return _near_sample(V, T, N, A, st["tree"], st["near"], st["cfg"], budget, seed=100 + i0)


def _ref_cpl(args):
    """Worker: seeded far blocks through the oracle tensor rule, pivot sets
    drawn from each cluster's dofs with the reference basis's ranks."""
    from oracle import quad as OQ

    i0, budget = args
    st = _REF
    V, T, N, A = st["mesh"]
    tree, far, rank = st["tree"], st["far"], st["rank"]
    rng = np.random.default_rng(200 + i0)
    pairs = blocks = 0
    t0 = time.perf_counter()
    for i in rng.permutation(len(far)):
        if time.perf_counter() - t0 > budget:
            break
        piv = []
        for u in far[i]:
            dofs = tree.perm[tree.start[u] : tree.end[u]]
            piv.append(rng.choice(dofs, size=min(int(rank[u]), len(dofs)), replace=False))
        OQ.slp_block(V, T, N, A, piv[0], piv[1], st["cfg"]["q_reg"], None)
        pairs += len(piv[0]) * len(piv[1])
        blocks += 1
    return {"pairs": pairs, "blocks": blocks, "s": time.perf_counter() - t0}


def run_reference(args, cfg):
    """The reference's CPU algorithm (oracle port) on this host's cores, same
    configuration: each step = the reference matvec restricted to one row
    slice per core (oracle.h2.RowSlice), run in parallel; value = rows of all
    slices / step wall time."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp

    from oracle import structure as OS

    cores = os.cpu_count() or 8
    t0 = time.perf_counter()
    V, T, N, A = OS.sphere(cfg["level"])
    tree = OS.cluster_tree(OS.p0_boxes(V, T), cfg["leaf"])
    far, near = OS.block_tree(tree, tree, cfg["eta"])
    t_struct = time.perf_counter() - t0
    g = np.load(os.path.join(ROOT, "tests", "golden", cfg["golden"]))
    rank_arr = np.asarray(g["ranks"], dtype=np.int64)
    assert len(rank_arr) == tree.n_nodes
    x = draw_x(cfg, len(tree.perm))
    # row slices: the clusters at the depth where a slice holds ~1/64 of the rows
    d = int(np.clip(np.round(np.log2(max(len(tree.perm) // 32768, 2))), 1, 8))
    roots = np.flatnonzero(tree.depth == d)
    rng = np.random.default_rng(cfg["seed"])
    roots = rng.permutation(roots)[: min(cores, len(roots))]
    _REF.update(tree=tree, far=far, near=near, rank=rank_arr, x=x, mesh=(V, T, N, A), cfg=cfg)
    ctx = mp.get_context("fork")
    with ctx.Pool(len(roots)) as pool:
        t1 = time.perf_counter()
        pool.map(_ref_slice_warm, roots, chunksize=1)  # build the slice operators (untimed)
        t_build = time.perf_counter() - t1
        for _ in range(max(args.warmup, 1)):
            pool.map(_ref_step, roots, chunksize=1)
        K = args.steps
        walls, rows_total = [], 0
        for _ in range(K):
            t1 = time.perf_counter()
            res = pool.map(_ref_step, roots, chunksize=1)
            walls.append(time.perf_counter() - t1)
            rows_total = sum(r for r, _ in res)
        near_res = pool.map(_ref_near, [(i, 6.0) for i in range(len(roots))], chunksize=1)
        cpl_res = pool.map(_ref_cpl, [(i, 3.0) for i in range(len(roots))], chunksize=1)
    dt = float(np.sum(walls))
    val = rows_total * K / dt
    npairs = sum(r["pairs"] for r in near_res)
    nwall = max(r["s_singular"] + r["s_regular"] for r in near_res)
    out = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "DoF/s", "n_gpus": ws, "steps": K,
        "warmup": max(args.warmup, 1), "ms_per_step": dt / K * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (generated sphere mesh, x ~ {'N(0,1)' if cfg['dist'] == 'normal' else 'U(-1,1)'} "
                f"seed {cfg['seed']})",
        "config": {"workload": cfg["desc"], "n_dofs": int(len(tree.perm))},
        "cpu_baseline": {"value": val, "unit": "DoF/s", "cores": len(roots), "kind": "port",
                         "sample": f"each step: the reference matvec (oracle.h2.RowSlice, containers.py:254-270 "
                                   f"restricted to a row subtree: its far/near blocks, its ancestors' far blocks, "
                                   f"the forward transform of every column cluster they read) on {len(roots)} "
                                   f"row slices of depth {d} ({rows_total} of {len(tree.perm)} rows) in parallel, "
                                   f"one per core; structure from oracle/structure.py (bit-exact with the "
                                   f"reference), ranks from the reference's basis ({cfg['golden']}), operator "
                                   f"values seeded random (the CPU cost does not depend on them)"},
        "e2e": {"value": val, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "couplings": {"pairs_per_s": sum(r["pairs"] for r in cpl_res) / max(r["s"] for r in cpl_res),
                      "pairs": int(sum(r["pairs"] for r in cpl_res)), "cores": len(roots),
                      "sample": "seeded random far blocks through the oracle tensor rule (pivot sets of the "
                                "reference basis's ranks), one process per core"},
        "nearfield": {"pairs_per_s": npairs / nwall if nwall else None, "pairs": int(npairs), "cores": len(roots),
                      "sample": "seeded random near blocks through the oracle quadrature (Sauter-Schwab for the "
                                "sampled touching pairs, tensor rule otherwise), one process per core"},
        "setup_s": {"structure": round(t_struct, 1), "slice_operators": round(t_build, 1)},
    }
    print(json.dumps(out), flush=True)


def _ref_slice_warm(root):
    _ref_slice(root)
    return 0


# ---------------------------------------------------------------------------

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return 0
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1:
        # launch one rank per GPU ourselves (the driver uses torchrun directly)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if ws is not None and int(ws) != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}")
    run_ours(args, cfg)
    return 0


if __name__ == "__main__":
    sys.exit(main())
