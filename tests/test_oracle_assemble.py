"""Oracle pins for the assembled operator A and the DoGIP weights.

(i)   WP, m = 1: 1^T A 1 = |Omega| = 1; row sums = int phi_i computed in
      EXACT arithmetic from the monomial expansion of the product basis;
      k = 1 gives the textbook P1 mass |T|/12 (1 + delta_ij) / |T|/20 (1 + delta_ij);
      DoGIP weights for m = 1, k = 1: 0 / |T|/3 (2D), -|T|/20 / |T|/5 (3D).
(ii)  EL: A 1 = 0; patch test (linear u, constant M: (Au)_i = 0 at interior
      DoFs and u^T A u = c^T M c); k = 1 textbook P1 stiffness.
(iii) Galerkin reproduction of polynomial solutions of degree <= p.
(iv)  Brute force: C^T A^DoGIP B equals the assembled A (Theorems 2/4, P:276,
      P:434) and the global Theorem 1 operator equals A.
plus: CSR route == element route == row-by-row route; symmetry and SPD.
"""
import itertools
from fractions import Fraction
from math import factorial

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import assemble as oa
from oracle import dogip as od
from oracle import reference as ref
from oracle.mesh import boundary_mask, dof_lattice
from synth.configs import (COEF_ANISO_FOURIER, COEF_CONST, COEF_CONST_TENSOR, COEF_PER_CELL,
                           COEF_SINCOS2D, COEF_TANH_RADIAL, Coefficient, aniso_fourier_params)
from synth.generators import grf_per_cell, vertex_jitter

ONE = Coefficient(COEF_CONST, np.array([1.0]))
SINCOS = Coefficient(COEF_SINCOS2D, np.array([1.0, 0.5]))
TANH = Coefficient(COEF_TANH_RADIAL, np.array([1.0, 0.9, 20.0, 0.25, 0.5, 0.5, 0.5]))
ANISO = Coefficient(COEF_ANISO_FOURIER, aniso_fourier_params(2))


def jittered(d, N, p, seed=4):
    M = N + 1
    ids = np.arange(M ** d)
    X = np.stack([(ids // M ** a) % M for a in range(d)], axis=1) / N
    return oa.build(d, N, p, X + vertex_jitter(d, N, 0.2, seed))


def exact_ref_integrals(d, k):
    """int_ref phi_alpha, exact: expand each factor of the product formula as a
    polynomial in lambda_i and integrate lambda^beta = prod beta!/(|beta|+d)!."""
    out = []
    for al in ref.multi_indices(d, k):
        polys = []
        for a in al:
            c = [Fraction(1)]                       # coefficients in lambda
            for j in range(a):                      # times (k lam - j)/(j+1)
                nc = [Fraction(0)] * (len(c) + 1)
                for e, v in enumerate(c):
                    nc[e + 1] += v * k / (j + 1)
                    nc[e] -= v * Fraction(j, j + 1)
                c = nc
            polys.append(c)
        tot = Fraction(0)
        for exps in itertools.product(*[range(len(c)) for c in polys]):
            coef = Fraction(1)
            for c, e in zip(polys, exps):
                coef *= c[e]
            tot += coef * Fraction(int(np.prod([factorial(e) for e in exps])),
                                   factorial(sum(exps) + d))
        out.append(tot)
    return out


@pytest.mark.parametrize("d,N,p", [(2, 3, 1), (2, 3, 2), (2, 2, 4), (3, 2, 1), (3, 2, 2), (3, 1, 4)])
def test_wp_unit_mass_row_sums(d, N, p):
    ed = oa.build(d, N, p)
    A = oa.assemble_csr(ed, 0, ONE)
    one = np.ones(ed.ndof)
    assert abs(one @ (A @ one) - 1.0) < 1e-13
    s = np.array([float(v) for v in exact_ref_integrals(d, p)]) * factorial(d)  # per |det|=d!|T|
    want = np.bincount(ed.lT.ravel(), weights=(np.abs(ed.det)[:, None] * s / factorial(d)).ravel(),
                       minlength=ed.ndof)
    assert np.allclose(A @ one, want, atol=1e-15)
    assert np.allclose(oa.load_vector(ed, 1.0), want, atol=1e-15)


def test_wp_C1_coefficient_total_mass():
    """int_Omega (1 + 0.5 sin 2pi x cos 2pi y) = 1 (SURVEY 8(c) check (i))."""
    ed = oa.build(2, 16, 2)
    A = oa.assemble_csr(ed, 0, SINCOS)
    one = np.ones(ed.ndof)
    assert abs(one @ (A @ one) - 1.0) < 1e-12


def test_textbook_p1_mass_and_weights():
    for d, den, wv, we in ((2, 12, 0.0, 1 / 3), (3, 20, -1 / 20, 1 / 5)):
        ed = oa.build(d, 2, 1)
        K = ed.element_matrices(0, ONE, slice(0, 1))[0]
        T = abs(ed.det[0]) / factorial(d)
        assert np.allclose(K, T / den * (np.ones((d + 1, d + 1)) + np.eye(d + 1)), atol=1e-16)
        w = od.element_weights(ed, 0, ONE)[0] / T
        lat = np.array(ref.multi_indices(d, 2))
        is_vertex = (lat == 2).any(axis=1)
        assert np.allclose(w[is_vertex], wv, atol=1e-14)
        assert np.allclose(w[~is_vertex], we, atol=1e-14)


def test_textbook_p1_stiffness_2d():
    ed = oa.build(2, 4, 1)
    K = ed.element_matrices(1, ONE, slice(0, 2))
    assert np.allclose(K[0], np.array([[1, -1, 0], [-1, 2, -1], [0, -1, 1]]) / 2, atol=1e-14)
    assert np.allclose(K[1], np.array([[1, 0, -1], [0, 1, -1], [-1, -1, 2]]) / 2, atol=1e-14)


@pytest.mark.parametrize("d,N,p,coef", [(2, 3, 2, SINCOS), (2, 2, 4, SINCOS), (3, 2, 2, ANISO),
                                        (3, 1, 3, TANH), (3, 1, 4, ANISO)])
def test_el_kills_constants(d, N, p, coef):
    ed = jittered(d, N, p)
    A = oa.assemble_csr(ed, 1, coef)
    assert np.abs(A @ np.ones(ed.ndof)).max() < 1e-11 * abs(A).max()


@pytest.mark.parametrize("d,N,p", [(2, 3, 2), (2, 2, 3), (3, 2, 2), (3, 2, 3)])
def test_el_patch_test(d, N, p):
    rng = np.random.default_rng(5)
    Q = rng.normal(size=(d, d))
    Mc = Q @ Q.T + d * np.eye(d)
    coef = Coefficient(COEF_CONST_TENSOR, Mc.ravel())
    ed = jittered(d, N, p)
    A = oa.assemble_csr(ed, 1, coef)
    c = rng.normal(size=d)
    # nodal positions of DoFs: from each element's affine map of the reference nodes
    xl = np.einsum("eij,lj->eli", ed.R, ref.nodes(d, p)) + ed.S[:, None, :]
    pos = np.zeros((ed.ndof, d))
    pos[ed.lT.ravel()] = xl.reshape(-1, d)
    u = pos @ c + 0.3
    Au = A @ u
    interior = ~boundary_mask(d, N, p)
    assert np.abs(Au[interior]).max() < 1e-12 * np.abs(A).max()
    assert abs(u @ Au - c @ Mc @ c) < 1e-12 * abs(c @ Mc @ c)


@pytest.mark.parametrize("d,N,p", [(2, 4, 2), (2, 3, 3), (3, 2, 2), (3, 2, 3)])
def test_el_polynomial_solution_reproduced(d, N, p):
    """(iii) -div(M grad u*) = f with constant M and u* in P_p: the Galerkin
    solution with Dirichlet data u* (lifting) equals u* at every DoF."""
    rng = np.random.default_rng(6)
    Q = rng.normal(size=(d, d))
    Mc = Q @ Q.T + d * np.eye(d)
    coef = Coefficient(COEF_CONST_TENSOR, Mc.ravel())
    exps = [e for e in itertools.product(range(p + 1), repeat=d) if sum(e) <= p]
    cs = rng.normal(size=len(exps))

    def ustar(x):
        return sum(c * np.prod(x ** np.array(e), axis=1) for c, e in zip(cs, exps))

    def hess(x):
        H = np.zeros((x.shape[0], d, d))
        for c, e in zip(cs, exps):
            for a in range(d):
                for b in range(d):
                    ee = np.array(e, dtype=float)
                    f = np.ones(x.shape[0]) * c
                    if a == b:
                        f = f * ee[a] * (ee[a] - 1)
                        ee[a] -= 2
                    else:
                        f = f * ee[a] * ee[b]
                        ee[a] -= 1
                        ee[b] -= 1
                    H[:, a, b] += f * np.prod(np.where(ee >= 0, x ** np.maximum(ee, 0), 0.0), axis=1)
        return H

    ed = jittered(d, N, p)
    A = oa.assemble_csr(ed, 1, coef)
    b = oa.load_vector_fn(ed, lambda x: -np.einsum("ab,nab->n", Mc, hess(x)))
    xl = np.einsum("eij,lj->eli", ed.R, ref.nodes(d, p)) + ed.S[:, None, :]
    pos = np.zeros((ed.ndof, d))
    pos[ed.lT.ravel()] = xl.reshape(-1, d)
    g = ustar(pos)
    bmask = boundary_mask(d, N, p)
    gb = np.where(bmask, g, 0.0)
    rhs = b - A @ gb
    rhs[bmask] = 0.0
    AD = oa.dirichlet_matrix(A, bmask)
    x = spla.spsolve(AD.tocsc(), rhs) + gb
    assert np.abs(x - g).max() < 1e-10 * max(1, np.abs(g).max())


@pytest.mark.parametrize("d,N,p", [(2, 3, 2), (2, 2, 4), (3, 2, 2)])
def test_wp_polynomial_projection_reproduced(d, N, p):
    """(iii) weighted projection with m = 1 of f in P_p returns f nodally."""
    rng = np.random.default_rng(7)
    exps = [e for e in itertools.product(range(p + 1), repeat=d) if sum(e) <= p]
    cs = rng.normal(size=len(exps))

    def f(x):
        return sum(c * np.prod(x ** np.array(e), axis=1) for c, e in zip(cs, exps))

    ed = jittered(d, N, p)
    A = oa.assemble_csr(ed, 0, ONE)
    b = oa.load_vector_fn(ed, f)
    x = spla.spsolve(A.tocsc(), b)
    xl = np.einsum("eij,lj->eli", ed.R, ref.nodes(d, p)) + ed.S[:, None, :]
    pos = np.zeros((ed.ndof, d))
    pos[ed.lT.ravel()] = xl.reshape(-1, d)
    assert np.abs(x - f(pos)).max() < 1e-10 * max(1, np.abs(f(pos)).max())


BRUTE = [(d, N, p, form) for d, N in ((2, 2), (3, 1)) for p in (1, 2, 3, 4) for form in (0, 1)]


@pytest.mark.parametrize("d,N,p,form", BRUTE)
def test_iv_bruteforce_dogip_equals_assembled(d, N, p, form):
    """(iv) C^T A^DoGIP B == A (dense), same rule Q, jittered mesh."""
    coef = (SINCOS if d == 2 else TANH) if form == 0 else (SINCOS if d == 2 else ANISO)
    ed = jittered(d, N, p)
    A = oa.assemble_csr(ed, form, coef).toarray()
    w = od.element_weights(ed, form, coef)
    D = od.dense_elementwise_operator(ed, form, w)
    assert np.abs(D - A).max() <= 1e-14 * np.abs(A).max() * max(1, p * p)
    u = np.random.default_rng(0).uniform(-1, 1, ed.ndof)
    y = od.algorithm1(ed, form, w, u)
    assert np.abs(y - A @ u).max() <= 1e-13 * np.abs(A @ u).max()


@pytest.mark.parametrize("d,N,p", [(2, 2, 2), (2, 2, 3), (3, 1, 2), (3, 2, 1)])
def test_iv_global_wp_theorem1(d, N, p):
    coef = SINCOS if d == 2 else TANH
    ed = jittered(d, N, p)
    A = oa.assemble_csr(ed, 0, coef).toarray()
    G = od.global_wp_operator(ed, coef)
    assert np.abs(G - A).max() <= 1e-14 * np.abs(A).max() * p


@pytest.mark.parametrize("d,N,p,form", [(2, 5, 3, 1), (3, 3, 2, 1), (3, 2, 4, 0), (2, 4, 2, 0)])
def test_routes_agree_and_spd(d, N, p, form):
    coef = (SINCOS if d == 2 else TANH) if form == 0 else (
        Coefficient(COEF_PER_CELL, np.zeros(0), grf_per_cell(d, N, 0.05, 1.0, 1)) if d == 2 else ANISO)
    ed = jittered(d, N, p)
    A = oa.assemble_csr(ed, form, coef)
    u = np.random.default_rng(0).uniform(-1, 1, ed.ndof)
    y = A @ u
    assert np.abs(oa.apply_elementwise(ed, form, coef, u) - y).max() <= 1e-14 * np.abs(y).max()
    rows = [0, ed.ndof // 3, ed.ndof - 1, ed.ndof // 2 + 1]
    assert np.allclose(oa.apply_rows(ed, form, coef, u, rows), y[rows], rtol=0, atol=1e-14 * np.abs(y).max())
    assert abs(A - A.T).max() <= 1e-14 * abs(A).max()
    Ad = A.toarray()
    if form == 1:
        Ad = oa.dirichlet_matrix(A, boundary_mask(d, N, p)).toarray()
    assert np.linalg.eigvalsh(Ad).min() > 0


def test_dirichlet_apply_matches_matrix():
    ed = oa.build(2, 4, 2)
    A = oa.assemble_csr(ed, 1, SINCOS)
    mask = boundary_mask(2, 4, 2)
    u = np.random.default_rng(0).uniform(-1, 1, ed.ndof)
    y = oa.apply_elementwise(ed, 1, SINCOS, u, dirichlet=True)
    assert np.allclose(y, oa.dirichlet_matrix(A, mask) @ u, atol=1e-14)
    assert np.array_equal(y[mask], u[mask])
    b = oa.load_vector(ed, 1.0, dirichlet=True)
    assert (b[mask] == 0).all() and (b[~mask] >= -1e-15).all()  # 2D P2 vertex integrals are 0
