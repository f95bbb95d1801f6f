"""Where the end-to-end (numpy in / numpy out) matvec time goes (config from argv, default 1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np
import torch
import bench
from paper_2001_05523_b200 import _lib
from paper_2001_05523_b200.containers import H2Matrix, assemble_couplings, near_layout

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "1"]
mesh, ctx, tree, bt, basis = bench.build_problem(cfg, os.cpu_count() or 8)
lay = near_layout(bt)
Dn = torch.zeros(max(lay.total, 1), dtype=torch.float64, device="cuda")
S = assemble_couplings(ctx, "slp", bt, basis, basis, 3)
H = H2Matrix.from_device(bt, basis, basis, S, Dn)
n = H.shape[1]
plan = H.plan()
xh = torch.randn(n, dtype=torch.float64).pin_memory().numpy()
yh = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
xd = torch.from_numpy(xh).cuda()
L = _lib.lib()


REPS = 300 if cfg["level"] <= 6 else 40


def wall(fn, reps=None):
    reps = reps or REPS
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    ts = np.sort(ts)
    return f"median {np.median(ts)*1e6:.1f} us, p10 {ts[len(ts)//10]*1e6:.1f} us"


def dev():
    plan.apply_device(xd)
    torch.cuda.synchronize()


print("H.matvec(numpy)            ", wall(lambda: H.matvec(xh)))
print("raw h2b_matvec_host         ", wall(lambda: L.h2b_matvec_host(plan.handle, _lib.ptr(xh), _lib.ptr(yh), None)))
print("device in/out + sync        ", wall(dev))
print("pinned alloc                ", wall(lambda: torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()))
xpg = np.array(xh)  # pageable copy, made once
print("pageable x (staged)         ", wall(lambda: L.h2b_matvec_host(plan.handle, _lib.ptr(xpg), _lib.ptr(yh), None)))
print("H.matvec(pageable numpy)    ", wall(lambda: H.matvec(xpg)))


def copies():
    xd.copy_(torch.from_numpy(xh), non_blocking=True)
    y = plan.apply_device(xd)
    torch.from_numpy(yh).copy_(y, non_blocking=True)
    torch.cuda.synchronize()


print("H2D + device + D2H (torch)  ", wall(copies))


xpage = np.array(xh)


def copies_pageable():
    xd.copy_(torch.from_numpy(xpage))
    y = plan.apply_device(xd)
    out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    out.copy_(y, non_blocking=True)
    torch.cuda.synchronize()
    return out.numpy()


print("pageable H2D (torch) + device + D2H pinned ", wall(copies_pageable))
t0 = time.perf_counter()
for _ in range(20):
    z = np.array(xh)
print("numpy copy of x (one core)  ", f"{(time.perf_counter() - t0) / 20 * 1e6:.1f} us")
