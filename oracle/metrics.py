"""Storage / multiplication-count model of the paper (oracle; test infra).

  mem A = 2 nnz A + nrows A
  memory efficiency = nnz A_T^DoGIP * dim M / mem A          (eq:memory_eff)
  comp. efficiency  = [2 (nnz Bhat - nnz_{+-1} Bhat) + nnz A_T^DoGIP] * dim M / nnz A
                                                             (eq:comp_eff)
nnz A_T^DoGIP = W_T (WP) or d^2 W_T (EL, as the tables count it; reading L11).
``nnz_A_pattern`` counts the structural nonzeros of A (full element-coupling
pattern) exactly for small N and extends them to the paper's N through the
exact polynomial in N that they follow (degree d, Lagrange interpolation in
rational arithmetic, checked on an extra point).
"""
from __future__ import annotations

from fractions import Fraction
from math import comb

import numpy as np

from .mesh import dof_map, structured_mesh


def n_elem(d: int, N: int) -> int:
    """dim M = 2N^2 (2D) or 6N^3 (3D)."""
    return 2 * N * N if d == 2 else 6 * N ** 3


def dim_V(d: int, N: int, k: int) -> int:
    return (k * N + 1) ** d


def W_T(d: int, k: int, form: int) -> int:
    return comb(2 * k + d, d) if form == 0 else comb(2 * k - 2 + d, d)


def nnz_AT_dogip(d: int, k: int, form: int) -> int:
    return W_T(d, k, form) * (1 if form == 0 else d * d)


def nnz_A_small(d: int, N: int, k: int) -> int:
    """Structural nnz of A: pairs (i, j) of DoFs sharing an element."""
    lT = dof_map(structured_mesh(d, N), k)
    nd = dim_V(d, N, k)
    V = lT.shape[1]
    keys = (np.repeat(lT, V, axis=1) * nd + np.tile(lT, (1, V))).ravel()
    return int(np.unique(keys).size)


def nnz_A_pattern(d: int, N: int, k: int) -> int:
    """nnz of the full pattern at any N via the exact degree-d polynomial."""
    if N <= d + 4:
        return nnz_A_small(d, N, k)
    xs = list(range(2, d + 4))                   # d + 2 points for degree <= d
    ys = [nnz_A_small(d, n, k) for n in xs]

    def interp(xx, pts, vals):
        tot = Fraction(0)
        for i, xi in enumerate(pts):
            t = Fraction(vals[i])
            for j, xj in enumerate(pts):
                if j != i:
                    t *= Fraction(xx - xj, xi - xj)
            tot += t
        return tot

    # degree check: the polynomial through the first d+1 points must hit the last
    assert interp(xs[-1], xs[:-1], ys[:-1]) == ys[-1], "nnz(N) not polynomial"
    v = interp(N, xs, ys)
    assert v.denominator == 1
    return int(v)


def mem_csr(nnz: int, nrows: int) -> int:
    return 2 * nnz + nrows


def memory_efficiency(d: int, N: int, k: int, form: int, memA: int) -> float:
    return nnz_AT_dogip(d, k, form) * n_elem(d, N) / memA


def comp_efficiency(d: int, N: int, k: int, form: int, memA: int,
                    nnzB: int, nnzB_pm1: int) -> float:
    nnzA = (memA - dim_V(d, N, k)) // 2
    return (2 * (nnzB - nnzB_pm1) + nnz_AT_dogip(d, k, form)) * n_elem(d, N) / nnzA
