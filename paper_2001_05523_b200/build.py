"""Build libh2b.so in-tree: nvcc for sm_100a (cross-compiles without a GPU).

    python -m paper_2001_05523_b200.build          # incremental
    python -m paper_2001_05523_b200.build --force  # full rebuild

The shared library lands in paper_2001_05523_b200/_lib/libh2b.so (git-ignored,
shipped to the GPU box with the working tree).
"""

import argparse
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
LIB = os.path.join(OUT_DIR, "libh2b.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["errors.cpp", "structure.cpp", "dlp_jobs.cpp", "block_jobs.cpp", "comm.cpp", "quadrature.cu", "matvec.cu", "gca.cu", "solver.cu",
           "matmat.cu", "basis.cu", "tree_dev.cu"]
HEADERS = ["h2b_internal.h", "device_common.cuh", "nccl_api.h"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _flags(src):
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
    if src.endswith(".cu"):
        # no --use_fast_math: fp64 quadrature keeps IEEE division/sqrt semantics
        return common + ARCH + ["-lineinfo", "-Xptxas", "-v"] + ["--expt-relaxed-constexpr"]
    # host-only translation units: exact IEEE evaluation (bit-exact structure)
    return common + ["-Xcompiler", "-ffp-contract=off", "-x", "c++"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    os.makedirs(OBJ_DIR, exist_ok=True)
    cc = nvcc()
    headers = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "h2b.h")]
    objs = []
    logs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OBJ_DIR, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + headers + [__file__]):
            cmd = [cc, "-c", path, "-o", obj] + _flags(src)
            res = subprocess.run(cmd, capture_output=True, text=True)
            logs.append((src, res.stdout + res.stderr))
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
    if force or _stale(LIB, objs):
        cmd = [cc, "-shared", "-o", LIB] + objs + ARCH + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    # measurement probes used by bench.py (FP64 peak) and tools/
    tools = os.path.join(ROOT, "tools")
    tbin = os.path.join(tools, "_bin")
    os.makedirs(tbin, exist_ok=True)
    for name in ("fp64_probe", "stream_probe"):
        src = os.path.join(tools, name + ".cu")
        exe = os.path.join(tbin, name)
        if os.path.exists(src) and (force or _stale(exe, [src])):
            res = subprocess.run([cc, "-O3", "-std=c++17", "-o", exe, src] + ARCH, capture_output=True, text=True)
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed for {name}:\n{res.stdout}\n{res.stderr}")
    if verbose:
        for src, text in logs:
            print(f"== {src}\n{text}")
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    args = ap.parse_args()
    print(build(force=args.force, verbose=args.verbose))


if __name__ == "__main__":
    sys.exit(main())
