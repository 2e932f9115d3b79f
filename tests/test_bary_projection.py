"""The barycentric-derivative form of the EL tables used by the generated 3D EL
projection (gen_bhat.cpp `g_bary`), restated on the CPU.

D_i[j][l] = d phi_l / d lambda_i at the W nodes (2k-2 lattice), one lambda factor
differentiated; with x̂_r = lambda_r (reading L2) the reference gradient is
d/dx̂_r = d/dlambda_r - d/dlambda_0, i.e. Bhat_EL[r] = D_{r+1} - D_0.  Checked
exactly against the oracle's Bhat_EL (built from its own gradient routine), with the
nonzero counts DESIGN.md quotes, and the projection identity the kernel evaluates:
sum_r Bhat[r][j][l] h_r = sum_{i>=1} D_i[j][l] h_{i-1} - D_0[j][l] sum_r h_r.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle.reference import bhat_el_exact, multi_indices


def _factor(a, k, lam):
    v = Fraction(1)
    for m in range(a):
        v *= (k * lam - m) / Fraction(m + 1)
    return v


def _dfactor(a, k, lam):
    s = Fraction(0)
    for m in range(a):
        t = Fraction(k, m + 1)
        for j in range(a):
            if j != m:
                t *= (k * lam - j) / Fraction(j + 1)
        s += t
    return s


def _bary_tables(d, k):
    A = [tuple(a) for a in multi_indices(d, k)]
    W = [tuple(Fraction(x, 2 * k - 2) for x in w) for w in multi_indices(d, 2 * k - 2)] if k > 1 else \
        [tuple(Fraction(1, d + 1) for _ in range(d + 1))]
    D = []
    for i in range(d + 1):
        Di = []
        for w in W:
            row = []
            for a in A:
                v = _dfactor(a[i], k, w[i])
                for m in range(d + 1):
                    if m != i:
                        v *= _factor(a[m], k, w[m])
                row.append(v)
            Di.append(row)
        D.append(Di)
    return D


@pytest.mark.parametrize("d,k", [(2, 2), (2, 3), (3, 1), (3, 2), (3, 3), (3, 4)])
def test_gradient_table_is_difference_of_barycentric_derivatives(d, k):
    B = bhat_el_exact(d, k)
    D = _bary_tables(d, k)
    for r in range(d):
        for j in range(len(B[r])):
            for l in range(len(B[r][j])):
                assert B[r][j][l] == D[r + 1][j][l] - D[0][j][l]


@pytest.mark.parametrize("d,k,nnz_d,nnz_b", [(3, 2, 22, 126), (3, 3, 185, 1014), (3, 4, 893, 4590)])
def test_nonzero_counts(d, k, nnz_d, nnz_b):
    D = _bary_tables(d, k)
    B = bhat_el_exact(d, k)
    assert all(sum(v != 0 for row in Di for v in row) == nnz_d for Di in D)
    assert sum(v != 0 for Br in B for row in Br for v in row) == nnz_b


@pytest.mark.parametrize("d,k", [(3, 2), (3, 3)])
def test_projection_identity(d, k):
    B = bhat_el_exact(d, k)
    D = _bary_tables(d, k)
    rng = np.random.default_rng(7)
    for j in range(len(B[0])):
        h = [Fraction(int(x), 13) for x in rng.integers(-40, 40, d)]
        for l in range(len(B[0][0])):
            lhs = sum(B[r][j][l] * h[r] for r in range(d))
            rhs = sum(D[i][j][l] * h[i - 1] for i in range(1, d + 1)) - D[0][j][l] * sum(h)
            assert lhs == rhs
