"""Oracle pins for the reference element, quadrature and mesh.

Pins (none re-types the oracle's formula): the delta property P:156 checked in
exact arithmetic; partition of unity and row sums (WP rows sum to 1, EL rows
to 0); gradients against central differences of the values;
polynomial reproduction; exact monomial integrals prod(alpha!)/(|alpha|+d)!
on the simplex; mesh cardinalities P:542 and total volume 1.
"""
import itertools
from fractions import Fraction
from math import factorial

import numpy as np
import pytest

from oracle import mesh as om
from oracle import quadrature as oq
from oracle import reference as ref


@pytest.mark.parametrize("d,k", [(2, k) for k in range(0, 7)] + [(3, k) for k in range(0, 5)])
def test_delta_property_exact(d, k):
    A = ref.multi_indices(d, k)
    X = ref.nodes_exact(d, k)
    assert len(A) == ref.dim_P(d, k) == len(X)
    for i, x in enumerate(X):
        for j, a in enumerate(A):
            assert ref.phi(a, k, x) == (1 if i == j else 0)


def test_nodes_layout_examples():
    # S:145-147 examples: (2,1) vertices, (2,2) = vertices + edge midpoints, (3,4) 35 points
    assert [tuple(p) for p in ref.nodes(2, 1)] == [(0, 0), (1, 0), (0, 1)]
    n22 = {tuple(p) for p in ref.nodes(2, 2)}
    assert n22 == {(0, 0), (.5, 0), (1, 0), (0, .5), (.5, .5), (0, 1)}
    assert len(ref.nodes(3, 4)) == 35
    assert np.allclose(ref.nodes(3, 0), [[.25, .25, .25]])


@pytest.mark.parametrize("d,k", [(2, 1), (2, 2), (2, 3), (2, 4), (3, 1), (3, 2), (3, 3), (3, 4)])
def test_bhat_row_sums_exact(d, k):
    for row in ref.bhat_wp_exact(d, k):
        assert sum(row) == 1                      # interpolating 1 reproduces 1
    for blk in ref.bhat_el_exact(d, k):
        for row in blk:
            assert sum(row) == 0                  # gradient of a constant


def test_bhat_el_k1_is_hat_gradients():
    # for k=1 W_T = 1 and B-hat = constant gradients of the hat functions
    B = ref.bhat_el(2, 1)
    assert np.array_equal(B[:, 0, :], np.array([[-1, 1, 0], [-1, 0, 1]]))
    B3 = ref.bhat_el(3, 1)
    assert np.array_equal(B3[:, 0, :], np.array([[-1, 1, 0, 0], [-1, 0, 1, 0], [-1, 0, 0, 1]]))


@pytest.mark.parametrize("d,k", [(2, 2), (2, 4), (3, 2), (3, 4)])
def test_partition_of_unity_and_gradients(d, k):
    rng = np.random.default_rng(1)
    pts = rng.dirichlet(np.ones(d + 1), 50)[:, 1:]
    V = ref.eval_basis(d, k, pts)
    assert np.allclose(V.sum(axis=1), 1.0, atol=1e-13)
    G = ref.eval_grad(d, k, pts)
    h = 1e-6
    for r in range(d):
        e = np.zeros(d)
        e[r] = h
        fd = (ref.eval_basis(d, k, pts + e) - ref.eval_basis(d, k, pts - e)) / (2 * h)
        assert np.allclose(G[:, :, r], fd, atol=1e-6 * max(1, k ** 3))
    # exact gradients agree with the float ones at the W nodes
    Bel = ref.bhat_el(d, k)
    Gw = ref.eval_grad(d, k, ref.nodes(d, 2 * k - 2))
    assert np.allclose(np.transpose(Gw, (2, 0, 1)), Bel, atol=1e-12)


@pytest.mark.parametrize("d,k", [(2, 3), (3, 3)])
def test_polynomial_reproduction(d, k):
    """Interpolating a degree-k polynomial at the nodes reproduces it."""
    rng = np.random.default_rng(2)
    exps = [e for e in itertools.product(range(k + 1), repeat=d) if sum(e) <= k]
    coef = rng.normal(size=len(exps))

    def poly(x):
        return sum(c * np.prod(x ** np.array(e), axis=1) for c, e in zip(coef, exps))

    vals = poly(ref.nodes(d, k))
    pts = rng.dirichlet(np.ones(d + 1), 40)[:, 1:]
    assert np.allclose(ref.eval_basis(d, k, pts) @ vals, poly(pts), atol=1e-12)


def _simplex_monomial(alpha):
    """int_{ref simplex} x^alpha = prod(alpha_i!) / (|alpha| + d)!"""
    d = len(alpha)
    return Fraction(int(np.prod([factorial(a) for a in alpha])), factorial(sum(alpha) + d))


@pytest.mark.parametrize("d,n", [(2, 2), (2, 5), (2, 7), (3, 3), (3, 5), (3, 7)])
def test_quadrature_exactness(d, n):
    pts, w = oq.simplex_rule(d, n)
    assert pts.shape == (n ** d, d)
    assert abs(w.sum() - 1.0 / factorial(d)) < 1e-15
    assert (w > 0).all()
    bary = np.concatenate([1 - pts.sum(1, keepdims=True), pts], axis=1)
    assert (bary > 0).all()                                   # interior points
    for alpha in itertools.product(range(2 * n), repeat=d):
        if sum(alpha) <= 2 * n - 1:
            q = float(w @ np.prod(pts ** np.array(alpha), axis=1))
            ex = float(_simplex_monomial(alpha))
            assert abs(q - ex) <= 2e-15 * max(1.0, abs(ex)) + 1e-17, alpha
    # one degree higher is generally NOT exact (the rule is not trivially exact)
    alpha = (2 * n,) + (0,) * (d - 1)
    q = float(w @ pts[:, 0] ** (2 * n))
    assert abs(q - float(_simplex_monomial(alpha))) > 1e-15


@pytest.mark.parametrize("d,N", [(2, 1), (2, 5), (3, 1), (3, 2), (3, 4)])
def test_mesh_cardinalities_and_volume(d, N):
    m = om.structured_mesh(d, N)
    assert m.n_elem == (2 * N * N if d == 2 else 6 * N ** 3)
    assert m.X.shape[0] == (N + 1) ** d
    _, _, det, _ = om.affine_maps(m)
    assert np.allclose(np.abs(det), 1.0 / N ** d)
    assert abs(np.abs(det).sum() / factorial(d) - 1.0) < 1e-12
    # every interior facet is shared by exactly two elements, boundary facets by one
    facets = {}
    for e in m.elems:
        for f in itertools.combinations(sorted(e), d):
            facets[f] = facets.get(f, 0) + 1
    assert set(facets.values()) <= {1, 2}
    nb = sum(1 for v in facets.values() if v == 1)
    assert nb == 2 * d * N ** (d - 1) * (1 if d == 2 else 2)


@pytest.mark.parametrize("d,N,p", [(2, 3, 3), (3, 2, 2), (3, 2, 4)])
def test_dof_map_conforming(d, N, p):
    """Every global DoF is referenced and all elements place it at the same
    physical point (continuity of C_{N,p}), on a jittered mesh."""
    from synth.generators import vertex_jitter
    M = N + 1
    ids = np.arange(M ** d)
    X = np.stack([(ids // M ** a) % M for a in range(d)], axis=1) / N + vertex_jitter(d, N, 0.2, 4)
    m = om.structured_mesh(d, N, X)
    lT = om.dof_map(m, p)
    assert np.unique(lT).size == (p * N + 1) ** d
    R, S, _, _ = om.affine_maps(m)
    xl = np.einsum("eij,lj->eli", R, ref.nodes(d, p)) + S[:, None, :]
    pos = np.full(((p * N + 1) ** d, d), np.nan)
    for e in range(m.n_elem):
        for l, g in enumerate(lT[e]):
            if np.isnan(pos[g, 0]):
                pos[g] = xl[e, l]
            else:
                assert np.allclose(pos[g], xl[e, l], atol=1e-14)


def test_jittered_c5_mesh_positive():
    """Reading L21: the C5 jitter keeps every Kuhn tet non-degenerate."""
    from synth.configs import get_config
    c = get_config("C5")
    m = om.structured_mesh(3, c.N, c.vertices())
    _, _, det, _ = om.affine_maps(m)
    det0 = np.array([1, -1, -1, 1, 1, -1] * (c.N ** 3), dtype=float)  # lattice signs
    assert (det * det0 > 0).all()
    assert abs(np.abs(det).sum() / 6 - 1.0) < 1e-10
