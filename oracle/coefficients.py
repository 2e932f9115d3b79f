"""Material coefficients m(x) / M(x) of the benchmark configs (oracle; test infra).

PAPER.md P:185 (WP coefficient m uniformly positive), P:306-311 (EL tensor M
uniformly positive definite and bounded).  The closed forms are those of
BASELINE.json ``configs``; readings L19-L22 fix the unstated parts.  Kind
codes match synth/configs.py and include/dogip.h.
"""
from __future__ import annotations

import numpy as np

from synth.configs import (COEF_ANISO_FOURIER, COEF_CONST, COEF_CONST_TENSOR,
                           COEF_PER_CELL, COEF_SINCOS2D, COEF_TANH_RADIAL,
                           Coefficient)


def rodrigues(omega: np.ndarray) -> np.ndarray:
    """Rotation by axis-angle vectors omega (n,3): R = I + sin t K + (1-cos t) K^2,
    K the cross-product matrix of omega/|omega| (I + [omega]_x for |omega|<1e-12)."""
    n = omega.shape[0]
    t = np.linalg.norm(omega, axis=1)
    small = t < 1e-12
    k = omega / np.where(small, 1.0, t)[:, None]
    K = np.zeros((n, 3, 3))
    K[:, 0, 1], K[:, 0, 2] = -k[:, 2], k[:, 1]
    K[:, 1, 0], K[:, 1, 2] = k[:, 2], -k[:, 0]
    K[:, 2, 0], K[:, 2, 1] = -k[:, 1], k[:, 0]
    I = np.broadcast_to(np.eye(3), (n, 3, 3))
    R = I + np.sin(t)[:, None, None] * K + (1.0 - np.cos(t))[:, None, None] * (K @ K)
    if small.any():
        W = np.zeros((int(small.sum()), 3, 3))
        o = omega[small]
        W[:, 0, 1], W[:, 0, 2] = -o[:, 2], o[:, 1]
        W[:, 1, 0], W[:, 1, 2] = o[:, 2], -o[:, 0]
        W[:, 2, 0], W[:, 2, 1] = -o[:, 1], o[:, 0]
        R[small] = np.eye(3) + W
    return R


def evaluate(coef: Coefficient, d: int, x: np.ndarray, cell: np.ndarray) -> np.ndarray:
    """Coefficient at physical points x (n, d) lying in cells ``cell`` (n,).

    Returns (n,) for isotropic kinds, (n, d, d) for tensor kinds."""
    k, P = coef.kind, np.asarray(coef.params, dtype=np.float64)
    if k == COEF_CONST:
        return np.full(x.shape[0], P[0])
    if k == COEF_PER_CELL:
        return np.asarray(coef.per_cell)[cell]
    if k == COEF_SINCOS2D:
        # config 1: a(x,y) = 1 + 0.5 sin(2 pi x) cos(2 pi y)
        return P[0] + P[1] * np.sin(2 * np.pi * x[:, 0]) * np.cos(2 * np.pi * x[:, 1])
    if k == COEF_TANH_RADIAL:
        # config 5: a(x) = 1 + 0.9 tanh(20 (|x - c| - 0.25)), c = (0.5,0.5,0.5) (L22)
        a0, a1, kk, r0 = P[:4]
        c = P[4:4 + d]
        r = np.sqrt(((x - c) ** 2).sum(axis=1))
        return a0 + a1 * np.tanh(kk * (r - r0))
    if k == COEF_ANISO_FOURIER:
        # config 3: M(x) = R(x) diag(1,10,100) R(x)^T, R = Rodrigues(omega(x)) (L20)
        eig = P[0:3]
        n = int(P[3])
        kap = P[4:4 + 3 * n].reshape(n, 3)
        phi = P[4 + 3 * n:4 + 6 * n].reshape(n, 3)
        c = P[4 + 6 * n:4 + 9 * n].reshape(n, 3)
        arg = 2 * np.pi * (x @ kap.T)                         # (npts, n)
        omega = np.stack([(c[:, i][None, :] * np.cos(arg + phi[:, i][None, :])).sum(axis=1)
                          for i in range(3)], axis=1)
        R = rodrigues(omega)
        return (R * eig[None, None, :]) @ np.transpose(R, (0, 2, 1))    # R diag(eig) R^T
    if k == COEF_CONST_TENSOR:
        Mm = P[:d * d].reshape(d, d)
        return np.broadcast_to(Mm, (x.shape[0], d, d)).copy()
    raise ValueError(f"unknown coefficient kind {k}")


def as_tensor(val: np.ndarray, d: int) -> np.ndarray:
    """Isotropic m -> m I (the corollary's M = m I)."""
    if val.ndim == 1:
        return val[:, None, None] * np.eye(d)[None]
    return val
