"""The symmetry-adapted WP apply (DOGIP_STORE_SYM) restated on the CPU.

The CUDA path evaluates B̂ᵀ diag(a) B̂ u through orbit coordinates of the barycentric
involution group G = <(0 1), (2 3)> (2D: <(0 1)>).  These tests re-derive that
reformulation independently from the oracle's exact B̂ and check:

* G-equivariance  B̂[gβ, gα] = B̂[β, α]  (the product basis);
* Schur: in orbit coordinates B̂ is block diagonal by character (no entry couples
  two different characters), with the block sizes DESIGN.md quotes (3D P4: 784
  entries instead of 1729);
* for random weights a and u, the orbit-coordinate evaluation (butterflies, block
  rows, s×s weight mixing with the group Fourier coefficients of a, transposed
  blocks, inverse butterflies) equals B̂ᵀ diag(a) B̂ u exactly in rational arithmetic.
No CUDA code is used; this pins the formula the generator emits.
"""
import itertools
from fractions import Fraction

import numpy as np
import pytest

from oracle.reference import bhat_wp_exact, multi_indices


def _group(d):
    gens = [(1, 0, 2, 3), (0, 1, 3, 2)] if d == 3 else [(1, 0, 2)]
    G = []
    for e in itertools.product([0, 1], repeat=len(gens)):
        g = tuple(range(d + 1))
        for gi, ei in zip(gens, e):
            if ei:
                g = tuple(g[gi[i]] for i in range(d + 1))
        G.append((e, g))
    return G


def _act(g, a):
    return tuple(a[g[i]] for i in range(len(a)))


def _chi(c, e):
    return -1 if sum(ci * ei for ci, ei in zip(c, e)) % 2 else 1


def _orbits(pts, G):
    seen, out = set(), []
    for i, x in enumerate(pts):
        if i in seen:
            continue
        members = {}
        for e, g in G:
            members.setdefault(pts.index(_act(g, x)), e)
        seen |= set(members)
        # characters trivial on the stabiliser
        stab = [e for e, g in G if _act(g, x) == x]
        chars = [c for c in itertools.product([0, 1], repeat=len(G[0][0])) if all(_chi(c, e) == 1 for e in stab)]
        out.append((i, members, chars))      # members: index -> one group element reaching it
    return out


CASES = [(2, 2), (2, 4), (3, 2), (3, 3), (3, 4)]


@pytest.mark.parametrize("d,p", CASES)
def test_bhat_equivariant_and_block_diagonal(d, p):
    B = bhat_wp_exact(d, p)
    A = list(multi_indices(d, p))
    W = list(multi_indices(d, 2 * p))
    G = _group(d)
    for _, g in G:
        for j, b in enumerate(W):
            for l, a in enumerate(A):
                assert B[W.index(_act(g, b))][A.index(_act(g, a))] == B[j][l]
    OV, OW = _orbits(A, G), _orbits(W, G)
    nnz_blocks = 0
    for (j0, _, charsP) in OW:
        for (l0, _, charsO) in OV:
            for c in itertools.product([0, 1], repeat=len(G[0][0])):
                s = sum(_chi(c, e) * B[j0][A.index(_act(g, A[l0]))] for e, g in G)
                if c not in charsP or c not in charsO:
                    # a character not trivial on both stabilisers has no coordinate
                    continue
                nnz_blocks += s != 0
    nnz = sum(v != 0 for row in B for v in row)
    assert nnz_blocks < nnz
    if (d, p) == (3, 4):
        assert (nnz, nnz_blocks) == (1729, 784)


@pytest.mark.parametrize("d,p", CASES)
def test_orbit_evaluation_equals_algorithm_1(d, p):
    """y = B̂ᵀ diag(a) B̂ u (Algorithm 1 element body, P:504 with reading L8) through
    orbit coordinates, exactly."""
    B = bhat_wp_exact(d, p)
    A = list(multi_indices(d, p))
    W = list(multi_indices(d, 2 * p))
    G = _group(d)
    NG = len(G)
    rng = np.random.default_rng(5)
    u = [Fraction(int(x), 97) for x in rng.integers(-50, 50, len(A))]
    a = [Fraction(int(x), 89) for x in rng.integers(-50, 50, len(W))]
    ref = [sum(B[j][l] * a[j] * sum(B[j][m] * u[m] for m in range(len(A))) for j in range(len(W)))
           for l in range(len(A))]
    OV, OW = _orbits(A, G), _orbits(W, G)
    # adapted u (full-group sums)
    uh = {}
    for (l0, _, chars) in OV:
        for c in chars:
            uh[(l0, c)] = sum(_chi(c, e) * u[A.index(_act(g, A[l0]))] for e, g in G)
    z = {k: Fraction(0) for k in uh}
    for (j0, members, chars) in OW:
        # ghat_chi(P) = sum_O Bhat_chi[P,O] uhat_chi(O) / |H_O|
        gh = {}
        for c in chars:
            acc = Fraction(0)
            for (l0, mem, cO) in OV:
                if c not in cO:
                    continue
                Bc = sum(Fraction(_chi(c, e)) * B[j0][A.index(_act(g, A[l0]))] for e, g in G)
                acc += Bc * uh[(l0, c)] / (NG // len(mem))
            gh[c] = acc
        # ahat_psi(P) = (1/|G|) sum_g psi(g) a_{g j0};  hhat_chi = sum_chi' ahat_{chi chi'} ghat_chi'
        ah = {psi: sum(_chi(psi, e) * a[W.index(_act(g, W[j0]))] for e, g in G) / NG for psi in chars}
        hh = {c: sum(ah[tuple((x + y) % 2 for x, y in zip(c, c2))] * gh[c2] for c2 in chars) for c in chars}
        # zhat_chi(O) += Btilde_chi[P,O] hhat_chi(P),  Btilde = sum_{j in P} chi(k_j) B[j, l0]
        for (l0, mem, cO) in OV:
            for c in cO:
                if c not in chars:
                    continue
                Bt = sum(Fraction(_chi(c, e)) * B[j][l0] for j, e in members.items())
                z[(l0, c)] += Bt * hh[c]
    y = [Fraction(0)] * len(A)
    for (l0, members, chars) in OV:
        for l, e in members.items():
            y[l] = sum(_chi(c, e) * z[(l0, c)] for c in chars) / NG
    assert y == ref
