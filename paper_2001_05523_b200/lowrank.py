"""Fully pivoted cross approximation with inverse core (host).  Same pivot
rule and arithmetic as h2bem.lowrank.aca_inverse_core (lowrank.py:154-184):
largest-modulus residual entry (first occurrence in C order), rank-one
downdate R - R[:, mu] R[nu, :] / pivot, stop when ||R||_F <= eps ||S||_F.
Pivot indices are integers and must match the reference exactly, so every
floating-point step below is the same numpy operation the reference uses."""

import numpy as np


def aca_inverse_core(S, eps):
    """(tau, sigma, C, ok) with C = inv(S[tau, sigma])."""
    S = np.asarray(S, dtype=float)
    if not np.isfinite(S).all():
        raise ValueError("matrix contains non-finite entries")
    R = S.copy()
    total = np.linalg.norm(R)
    rows, cols = [], []
    if total == 0.0:
        return np.zeros(0, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros((0, 0)), True
    limit = min(S.shape)
    converged = True
    threshold = eps * total
    while np.linalg.norm(R) > threshold:
        flat = int(np.argmax(np.abs(R)))
        i, j = divmod(flat, R.shape[1])
        pivot = R[i, j]
        if pivot == 0.0 or len(rows) == limit:
            converged = False
            break
        rows.append(i)
        cols.append(j)
        R = R - np.outer(R[:, j], R[i, :]) / pivot
    tau = np.asarray(rows, dtype=np.int64)
    sigma = np.asarray(cols, dtype=np.int64)
    C = np.linalg.inv(S[np.ix_(tau, sigma)]) if len(tau) else np.zeros((0, 0))
    return tau, sigma, C, converged
