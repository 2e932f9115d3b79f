"""Reference element: Lagrange P_k on the unit right simplex (oracle; test infra).

PAPER.md P:149-157 (Lagrange nodal basis, delta property)
(reference element, affine map), P:172-175 (eq:bas_deriv chain rule),
P:283 (B-hat for WP: Bhat_jl = phi_l(xhat^W_j)), P:445 (B-hat for EL:
Bhat_rik = d phi_k / d xhat_r (xhat^W_i)).

Readings: L1 equispaced barycentric lattice nodes alpha/k (k=0:
barycentre); L2 reference simplex conv{0, e_1..e_d}, xhat_r = lambda_r,
lambda_0 = 1 - sum(xhat); L5 local order: alpha_1 fastest, alpha_d slowest.

The basis is the barycentric product formula
    phi_alpha(lambda) = prod_{i=0..d} prod_{j=0}^{alpha_i-1} (k lambda_i - j)/(j+1),
which has the delta property at the lattice nodes by inspection (a factor
vanishes whenever beta_i < alpha_i).  Tables are built in exact rational
arithmetic (fractions.Fraction) and rounded to fp64 once.
"""
from __future__ import annotations

import itertools
from fractions import Fraction
from functools import lru_cache
from math import comb

import numpy as np


def dim_P(d: int, k: int) -> int:
    """dim P_k on a d-simplex = C(k+d, d)."""
    return comb(k + d, d)


@lru_cache(maxsize=None)
def multi_indices(d: int, k: int) -> tuple:
    """Barycentric multi-indices (alpha_0, alpha_1..alpha_d), |alpha| = k,
    ordered with alpha_1 fastest and alpha_d slowest (reading L5)."""
    out = []
    for t in itertools.product(range(k + 1), repeat=d):   # t[0] slowest
        a = tuple(reversed(t))                            # (alpha_1..alpha_d)
        if sum(a) <= k:
            out.append((k - sum(a),) + a)
    return tuple(out)


def nodes_exact(d: int, k: int) -> list:
    """Reference nodes xhat = (alpha_1..alpha_d)/k as Fractions (k=0: barycentre)."""
    if k == 0:
        return [tuple(Fraction(1, d + 1) for _ in range(d))]
    return [tuple(Fraction(a, k) for a in al[1:]) for al in multi_indices(d, k)]


def nodes(d: int, k: int) -> np.ndarray:
    return np.array([[float(x) for x in n] for n in nodes_exact(d, k)])


def _bary(xhat):
    """lambda = (1 - sum xhat, xhat_1..xhat_d)  (reading L2)."""
    return (1 - sum(xhat),) + tuple(xhat)


def _f(a: int, k: int, lam):
    """prod_{j<a} (k lam - j)/(j+1) -- one factor of the product formula."""
    v = 1
    for j in range(a):
        v = v * (k * lam - j) / (j + 1)
    return v


def _df(a: int, k: int, lam):
    """d/d lam of _f (product rule)."""
    s = 0
    for m in range(a):
        t = Fraction(k, m + 1) if isinstance(lam, Fraction) else k / (m + 1)
        for j in range(a):
            if j != m:
                t = t * (k * lam - j) / (j + 1)
        s = s + t
    return s


def phi(alpha, k: int, xhat):
    """Lagrange basis function phi_alpha of P_k at reference point xhat."""
    lam = _bary(xhat)
    v = 1
    for i, a in enumerate(alpha):
        v = v * _f(a, k, lam[i])
    return v


def grad_phi(alpha, k: int, xhat):
    """Reference gradient d phi_alpha / d xhat_r, r = 1..d:
    d/d lambda_r - d/d lambda_0 (lambda_0 = 1 - sum xhat)."""
    lam = _bary(xhat)
    d = len(xhat)
    fs = [_f(a, k, lam[i]) for i, a in enumerate(alpha)]
    dfs = [_df(a, k, lam[i]) for i, a in enumerate(alpha)]

    def dlam(i):
        v = dfs[i]
        for m in range(d + 1):
            if m != i:
                v = v * fs[m]
        return v

    d0 = dlam(0)
    return tuple(dlam(r) - d0 for r in range(1, d + 1))


@lru_cache(maxsize=None)
def bhat_wp_exact(d: int, k: int) -> tuple:
    """Theorem 2: Bhat_jl = phi^l_V(xhat^j_W), V = P_k, W = P_2k.
    Returns a W_T x V_T tuple of tuples of Fractions."""
    W = nodes_exact(d, 2 * k)
    A = multi_indices(d, k)
    return tuple(tuple(phi(al, k, x) for al in A) for x in W)


@lru_cache(maxsize=None)
def bhat_el_exact(d: int, k: int) -> tuple:
    """Theorem 4 (reading L7/L9): Bhat_rik = d phi^k_V / d xhat_r at
    xhat^i_W, V = P_k, W = P_{2k-2} (discontinuous).  Shape d x W_T x V_T."""
    W = nodes_exact(d, 2 * k - 2)
    A = multi_indices(d, k)
    g = [[grad_phi(al, k, x) for al in A] for x in W]
    return tuple(tuple(tuple(g[i][l][r] for l in range(len(A)))
                       for i in range(len(W))) for r in range(d))


def bhat_wp(d: int, k: int) -> np.ndarray:
    return np.array([[float(v) for v in row] for row in bhat_wp_exact(d, k)])


def bhat_el(d: int, k: int) -> np.ndarray:
    return np.array([[[float(v) for v in row] for row in blk]
                     for blk in bhat_el_exact(d, k)])


def nnz_counts(table) -> tuple:
    """(nnz, nnz_{+-1}) of an exact table (reading: entries exactly +-1)."""
    flat = list(_flatten(table))
    nnz = sum(1 for v in flat if v != 0)
    pm1 = sum(1 for v in flat if v == 1 or v == -1)
    return nnz, pm1


def _flatten(t):
    if isinstance(t, (tuple, list)):
        for s in t:
            yield from _flatten(s)
    else:
        yield t


# ----- float evaluation at arbitrary points (quadrature points) -------------

def eval_basis(d: int, k: int, pts: np.ndarray) -> np.ndarray:
    """phi_alpha(pts) for all alpha: (npts, dim P_k), fp64 product formula."""
    pts = np.atleast_2d(pts)
    lam = np.concatenate([1.0 - pts.sum(axis=1, keepdims=True), pts], axis=1)
    out = np.empty((pts.shape[0], dim_P(d, k)))
    for c, al in enumerate(multi_indices(d, k)):
        v = np.ones(pts.shape[0])
        for i, a in enumerate(al):
            for j in range(a):
                v = v * (k * lam[:, i] - j) / (j + 1)
        out[:, c] = v
    return out


def eval_grad(d: int, k: int, pts: np.ndarray) -> np.ndarray:
    """Reference gradients (npts, dim P_k, d), fp64."""
    pts = np.atleast_2d(pts)
    lam = np.concatenate([1.0 - pts.sum(axis=1, keepdims=True), pts], axis=1)
    n = pts.shape[0]
    out = np.empty((n, dim_P(d, k), d))
    for c, al in enumerate(multi_indices(d, k)):
        fs, dfs = [], []
        for i, a in enumerate(al):
            f = np.ones(n)
            df = np.zeros(n)
            for j in range(a):
                # product rule, accumulated: (f * g)' = f' g + f g'
                g = (k * lam[:, i] - j) / (j + 1)
                df = df * g + f * (k / (j + 1))
                f = f * g
            fs.append(f)
            dfs.append(df)
        dl = []
        for i in range(d + 1):
            v = dfs[i].copy()
            for m in range(d + 1):
                if m != i:
                    v = v * fs[m]
            dl.append(v)
        for r in range(d):
            out[:, c, r] = dl[r + 1] - dl[0]
    return out
