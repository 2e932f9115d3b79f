"""Conical-product (collapsed) Gauss-Jacobi rule on the reference simplex
(oracle; test infra).

PAPER.md P:89-107 discusses simplex quadrature in general and P:694 notes that
FEniCS uses the collapsed rule of Karniadakis & Sherwin at high order; the
paper never fixes the rule used for the DoGIP weights.  Reading L10: the
contract rule, identical on both sides, is the collapsed Gauss-Jacobi rule
with n = p + 3 points per direction (exact to degree 2n - 1 = 2p + 5).

Collapsed coordinates (Duffy/Stroud), all on [0,1]:
  2D  x1 = s1,  x2 = s2 (1 - s1);                     Jacobian (1 - s1)
  3D  x1 = s1,  x2 = s2 (1 - s1),  x3 = s3 (1 - s1)(1 - s2);
                                                      Jacobian (1 - s1)^2 (1 - s2)
s_i uses Gauss-Jacobi with weight (1 - s)^(d - i), i = 1..d (the last one is
Gauss-Legendre).  Points are ordered s1 slowest, s_d fastest.
"""
from __future__ import annotations

import numpy as np
from scipy.special import roots_jacobi


def gauss_jacobi_01(n: int, a: int):
    """n-point rule for int_0^1 (1-s)^a g(s) ds: nodes/weights of
    roots_jacobi(n, a, 0) on [-1,1] mapped by s = (1+t)/2."""
    t, w = roots_jacobi(n, float(a), 0.0)
    return (1.0 + t) / 2.0, w / 2.0 ** (a + 1)


def simplex_rule(d: int, n: int):
    """Returns (points (n^d, d), weights (n^d,)), sum(weights) = 1/d!."""
    if d == 2:
        s1, w1 = gauss_jacobi_01(n, 1)
        s2, w2 = gauss_jacobi_01(n, 0)
        S1, S2 = np.meshgrid(s1, s2, indexing="ij")
        W1, W2 = np.meshgrid(w1, w2, indexing="ij")
        pts = np.stack([S1, S2 * (1.0 - S1)], axis=-1).reshape(-1, 2)
        return pts, (W1 * W2).ravel()
    if d == 3:
        s1, w1 = gauss_jacobi_01(n, 2)
        s2, w2 = gauss_jacobi_01(n, 1)
        s3, w3 = gauss_jacobi_01(n, 0)
        S1, S2, S3 = np.meshgrid(s1, s2, s3, indexing="ij")
        W1, W2, W3 = np.meshgrid(w1, w2, w3, indexing="ij")
        x1 = S1
        x2 = S2 * (1.0 - S1)
        x3 = S3 * (1.0 - S1) * (1.0 - S2)
        pts = np.stack([x1, x2, x3], axis=-1).reshape(-1, 3)
        return pts, (W1 * W2 * W3).ravel()
    raise ValueError("d must be 2 or 3")


def contract_n1d(p: int) -> int:
    """Reading L10: n = p + 3 points per direction."""
    return p + 3
