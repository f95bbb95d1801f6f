"""Device plumbing: torch owns device memory and streams, libh2b does the work.

`require_cuda()` is the loud failure every GPU entry point goes through: no
CUDA device or no built library -> RuntimeError, never a CPU fallback."""

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_2001_05523_b200: a CUDA device is required (no CPU fallback)")
    _lib.lib()
    return t


def dev(a, dtype=None):
    """numpy -> contiguous CUDA tensor."""
    t = require_cuda()
    a = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    if not a.flags.writeable:
        a = a.copy()
    return t.from_numpy(a).to("cuda", non_blocking=False)


def empty(shape, dtype="float64"):
    t = require_cuda()
    return t.empty(shape, dtype=getattr(t, dtype), device="cuda")


def zeros(shape, dtype="float64"):
    t = require_cuda()
    return t.zeros(shape, dtype=getattr(t, dtype), device="cuda")


def host(x):
    return x.detach().cpu().numpy()


def stream():
    return _lib.stream_ptr()
