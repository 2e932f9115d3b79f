"""Plain conjugate gradients (oracle; test infra).

PAPER.md P:86 only says matrix-free methods need "a suitable iterative
solver"; reading L15 fixes unpreconditioned Hestenes-Stiefel CG, x0 given
(zero in the configs), stopping when ||r_k||_2 <= rtol ||b||_2 on the
recursively updated residual.
"""
from __future__ import annotations

import numpy as np

CG_CONVERGED, CG_NOT_CONVERGED, CG_BREAKDOWN = 0, 1, -1


def cg(apply, b: np.ndarray, x0: np.ndarray | None = None, rtol: float = 1e-10,
       maxit: int = 10000):
    """Returns (x, iterations, recursive relative residual, status)."""
    x = np.zeros_like(b) if x0 is None else x0.astype(np.float64).copy()
    r = b - apply(x)
    p = r.copy()
    rr = float(r @ r)
    bnorm = float(np.sqrt(b @ b))
    if bnorm == 0.0:
        return x, 0, 0.0, CG_CONVERGED
    it = 0
    while np.sqrt(rr) > rtol * bnorm:
        if it >= maxit:
            return x, it, np.sqrt(rr) / bnorm, CG_NOT_CONVERGED
        q = apply(p)
        pq = float(p @ q)
        if pq <= 0.0:
            return x, it, np.sqrt(rr) / bnorm, CG_BREAKDOWN
        alpha = rr / pq
        x = x + alpha * p
        r = r - alpha * q
        rr_new = float(r @ r)
        p = r + (rr_new / rr) * p
        rr = rr_new
        it += 1
    return x, it, np.sqrt(rr) / bnorm, CG_CONVERGED
