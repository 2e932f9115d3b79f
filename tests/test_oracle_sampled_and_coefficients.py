"""Oracle pins for the full-size checker and the coefficient closed forms.

Every full-size GPU parity test compares sampled rows against
``oracle.assemble.apply_rows_sampled`` (which builds only the cells around a
DoF with ``oracle.mesh.cell_elements``).  These tests pin that route to the
CSR assembly of the whole mesh (the definition A = sum_T P_T^T K_T P_T,
eq:linsys_gp P:201-207, eq:linsys_se P:330-337) on small jittered meshes, for
every (d, p, form), on vertex / edge / face / interior DoFs, the boundary and
both ends of the slab axis.

The coefficient models (BASELINE.json configs; readings L20, L22) are pinned
by closed forms that do not re-type the oracle: Rodrigues rotations
(orthogonality, det 1, axis fixed, trace 1 + 2 cos|w|, the textbook z-axis
rotation, the small-angle branch), the anisotropic tensor's spectrum
{1, 10, 100} and its explicit form for a single constant mode, and point
values of the tanh inclusion and the C1 sin-cos field.
"""
import itertools

import numpy as np
import pytest

from oracle import assemble as oa
from oracle import coefficients as oc
from oracle.mesh import cell_elements, dof_lattice, structured_mesh
from synth.configs import (COEF_ANISO_FOURIER, COEF_CONST, COEF_PER_CELL, COEF_SINCOS2D,
                           COEF_TANH_RADIAL, Coefficient, aniso_fourier_params)
from synth.generators import grf_per_cell, vertex_jitter


def _jittered_vertices(d, N, seed=4):
    M = N + 1
    ids = np.arange(M ** d)
    X = np.stack([(ids // M ** a) % M for a in range(d)], axis=1) / N
    return X + vertex_jitter(d, N, 0.2, seed)


def _coef(d, N, form):
    if form == 0:
        return (Coefficient(COEF_SINCOS2D, np.array([1.0, 0.5])) if d == 2 else
                Coefficient(COEF_TANH_RADIAL, np.array([1.0, 0.9, 20.0, 0.25, 0.5, 0.5, 0.5])))
    if d == 2:
        return Coefficient(COEF_PER_CELL, np.zeros(0), grf_per_cell(d, N, 0.05, 1.0, 1))
    return Coefficient(COEF_ANISO_FOURIER, aniso_fourier_params(2))


def _rows_by_kind(d, N, p, rng):
    """DoFs of every topological kind (number of lattice coordinates on a cell
    boundary: d -> vertex, d-1 -> edge (2D: edge = facet), ..., 0 -> cell interior),
    boundary DoFs, and DoFs on the first / last plane of the slab axis."""
    lat = dof_lattice(d, N, p)
    on_grid = (lat % p == 0).sum(axis=1)
    bnd = np.any((lat == 0) | (lat == p * N), axis=1)
    rows = []
    for k in range(d + 1):
        idx = np.nonzero(on_grid == k)[0]
        for sel in (idx[bnd[idx]], idx[~bnd[idx]]):
            if sel.size:
                rows.extend(rng.choice(sel, size=min(3, sel.size), replace=False).tolist())
    for plane in (0, p * N):
        idx = np.nonzero(lat[:, d - 1] == plane)[0]
        rows.extend(rng.choice(idx, size=3, replace=False).tolist())
    return np.unique(np.array(rows, dtype=np.int64))


@pytest.mark.parametrize("d,p,form", [(d, p, f) for d in (2, 3) for p in (1, 2, 3, 4) for f in (0, 1)])
def test_apply_rows_sampled_equals_csr(d, p, form):
    N = 4 if d == 2 else (3 if p <= 2 else 2)
    verts = _jittered_vertices(d, N)
    coef = _coef(d, N, form)
    ed = oa.build(d, N, p, verts)
    u = np.random.default_rng(7).uniform(-1, 1, ed.ndof)
    y = oa.assemble_csr(ed, form, coef) @ u
    rows = _rows_by_kind(d, N, p, np.random.default_rng(d * 10 + p))
    ys = oa.apply_rows_sampled(d, N, p, verts, form, coef, u, rows)
    assert np.abs(ys - y[rows]).max() <= 1e-13 * np.abs(y).max()


@pytest.mark.parametrize("d,p", [(2, 1), (2, 3), (3, 1), (3, 2)])
def test_apply_rows_sampled_every_row_small_mesh(d, p):
    """Every row of a tiny mesh (all kinds, all boundary configurations)."""
    N = 2
    verts = _jittered_vertices(d, N, seed=9)
    coef = _coef(d, N, 1)
    ed = oa.build(d, N, p, verts)
    u = np.random.default_rng(3).uniform(-1, 1, ed.ndof)
    y = oa.assemble_csr(ed, 1, coef) @ u
    rows = np.arange(ed.ndof)
    ys = oa.apply_rows_sampled(d, N, p, verts, 1, coef, u, rows)
    assert np.abs(ys - y).max() <= 1e-13 * np.abs(y).max()


@pytest.mark.parametrize("d,N", [(2, 1), (2, 5), (3, 1), (3, 4)])
def test_cell_elements_match_structured_mesh(d, N):
    m = structured_mesh(d, N)
    ns = 2 if d == 2 else 6
    rng = np.random.default_rng(N)
    cells = np.unique(np.concatenate([[0, N ** d - 1], rng.integers(0, N ** d, 7)]))
    got = cell_elements(d, N, cells)
    want = m.elems[(ns * cells[:, None] + np.arange(ns)[None, :]).ravel()]
    assert np.array_equal(got, want)
    # and every cell at once reproduces the whole mesh
    assert np.array_equal(cell_elements(d, N, np.arange(N ** d)), m.elems)


# ------------------------------------------------------------------ coefficients
def test_rodrigues_is_a_rotation_about_omega():
    rng = np.random.default_rng(0)
    om = np.concatenate([rng.normal(0, 2.0, (64, 3)), [[0.0, 0.0, 0.0], [1e-14, 0, 0], [0, 0, np.pi],
                                                       [0, 7.0, 0]]])
    R = oc.rodrigues(om)
    I = np.eye(3)
    assert np.abs(np.einsum("nji,njk->nik", R, R) - I).max() <= 1e-14
    assert np.abs(np.linalg.det(R) - 1.0).max() <= 1e-14
    assert np.abs(np.einsum("nij,nj->ni", R, om) - om).max() <= 1e-14 * max(1.0, np.abs(om).max())
    t = np.linalg.norm(om, axis=1)
    assert np.abs(np.trace(R, axis1=1, axis2=2) - (1 + 2 * np.cos(t))).max() <= 1e-14


def test_rodrigues_textbook_axis_rotations():
    """Right-handed rotation by theta about e_z: (x, y) -> (x cos - y sin, x sin + y cos);
    about e_x: (y, z) -> (y cos - z sin, y sin + z cos).  Catches a transposed or sign-flipped K."""
    th = 0.7
    c, s = np.cos(th), np.sin(th)
    Rz = oc.rodrigues(np.array([[0.0, 0.0, th]]))[0]
    Rx = oc.rodrigues(np.array([[th, 0.0, 0.0]]))[0]
    assert np.abs(Rz - np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])).max() <= 1e-15
    assert np.abs(Rx - np.array([[1, 0, 0], [0, c, -s], [0, s, c]])).max() <= 1e-15
    # small-angle branch: first-order expansion I + [w]_x
    w = np.array([[1e-13, -2e-13, 3e-13]])
    K = np.array([[0, -3e-13, -2e-13], [3e-13, 0, -1e-13], [2e-13, 1e-13, 0]])
    assert np.abs(oc.rodrigues(w)[0] - (np.eye(3) + K)).max() <= 1e-26


def test_aniso_tensor_spectrum_and_symmetry():
    coef = Coefficient(COEF_ANISO_FOURIER, aniso_fourier_params(2))
    x = np.random.default_rng(1).uniform(0, 1, (200, 3))
    M = oc.evaluate(coef, 3, x, np.zeros(200, dtype=np.int64))
    assert np.abs(M - np.transpose(M, (0, 2, 1))).max() <= 1e-12
    ev = np.linalg.eigvalsh(M)
    assert np.abs(ev - np.array([1.0, 10.0, 100.0])).max() <= 1e-11


def test_aniso_tensor_single_constant_mode_closed_form():
    """One mode with kappa = 0, phi = 0, c = (0, 0, theta): omega = (0, 0, theta), so
    M = Rz(theta) diag(e1, e2, e3) Rz(theta)^T, written out entry by entry."""
    th, e = 0.4, (1.0, 10.0, 100.0)
    params = np.concatenate([e, [1.0], [0, 0, 0], [0, 0, 0], [0, 0, th]])
    coef = Coefficient(COEF_ANISO_FOURIER, params)
    x = np.random.default_rng(2).uniform(0, 1, (5, 3))
    M = oc.evaluate(coef, 3, x, np.zeros(5, dtype=np.int64))
    c, s = np.cos(th), np.sin(th)
    want = np.array([[e[0] * c * c + e[1] * s * s, (e[0] - e[1]) * c * s, 0],
                     [(e[0] - e[1]) * c * s, e[0] * s * s + e[1] * c * c, 0],
                     [0, 0, e[2]]])
    assert np.abs(M - want[None]).max() <= 1e-13
    # no modes: M = diag(e)
    M0 = oc.evaluate(Coefficient(COEF_ANISO_FOURIER, np.array([*e, 0.0])), 3, x, np.zeros(5, dtype=np.int64))
    assert np.abs(M0 - np.diag(e)[None]).max() == 0.0


def test_aniso_omega_varies_as_a_cosine_mode():
    """One mode kappa = (1, 0, 0), phi = (0, 0, 0), c = (0, 0, a): omega_z(x) = a cos(2 pi x_1),
    so the rotation angle at x_1 = 0, 1/4, 1/2 is a, 0, -a."""
    a = 0.3
    params = np.concatenate([[1.0, 10.0, 100.0], [1.0], [1, 0, 0], [0, 0, 0], [0, 0, a]])
    coef = Coefficient(COEF_ANISO_FOURIER, params)
    x = np.array([[0.0, 0.3, 0.6], [0.25, 0.1, 0.9], [0.5, 0.7, 0.2]])
    M = oc.evaluate(coef, 3, x, np.zeros(3, dtype=np.int64))
    for Mi, th in zip(M, (a, 0.0, -a)):
        c, s = np.cos(th), np.sin(th)
        assert abs(Mi[0, 0] - (c * c + 10 * s * s)) <= 1e-13
        assert abs(Mi[0, 1] - (1 - 10) * c * s) <= 1e-13


def test_tanh_inclusion_point_values():
    a0, a1, k, r0 = 1.0, 0.9, 20.0, 0.25
    for d in (2, 3):
        c = np.full(d, 0.5)
        coef = Coefficient(COEF_TANH_RADIAL, np.array([a0, a1, k, r0, *c]))
        e1 = np.eye(d)[0]
        diag = np.ones(d) / np.sqrt(d)
        x = np.stack([c, c + r0 * e1, c + 0.1 * e1, c + 0.4 * diag, c - 0.3 * np.eye(d)[d - 1]])
        got = oc.evaluate(coef, d, x, np.zeros(len(x), dtype=np.int64))
        want = [a0 + a1 * np.tanh(-k * r0), a0, a0 + a1 * np.tanh(k * (0.1 - r0)),
                a0 + a1 * np.tanh(k * (0.4 - r0)), a0 + a1 * np.tanh(k * (0.3 - r0))]
        assert np.abs(got - np.array(want)).max() <= 1e-15
    # C5's coefficient stays in (a0 - a1, a0 + a1) = (0.1, 1.9) (reading L22)
    x = np.random.default_rng(0).uniform(0, 1, (1000, 3))
    v = oc.evaluate(Coefficient(COEF_TANH_RADIAL, np.array([a0, a1, k, r0, .5, .5, .5])), 3, x,
                    np.zeros(1000, dtype=np.int64))
    assert v.min() > 0.1 and v.max() < 1.9


def test_sincos_and_cellwise_point_values():
    coef = Coefficient(COEF_SINCOS2D, np.array([1.0, 0.5]))
    x = np.array([[0.25, 0.0], [0.25, 0.5], [0.0, 0.3], [0.75, 0.0], [0.125, 0.125]])
    want = [1.5, 0.5, 1.0, 0.5, 1.0 + 0.5 * np.sin(np.pi / 4) * np.cos(np.pi / 4)]
    assert np.abs(oc.evaluate(coef, 2, x, np.zeros(5, dtype=np.int64)) - np.array(want)).max() <= 1e-15
    pc = np.array([3.0, 5.0, 7.0])
    v = oc.evaluate(Coefficient(COEF_PER_CELL, np.zeros(0), pc), 2, np.zeros((4, 2)), np.array([2, 0, 1, 2]))
    assert v.tolist() == [7.0, 3.0, 5.0, 7.0]
    v = oc.evaluate(Coefficient(COEF_CONST, np.array([2.5])), 3, np.zeros((3, 3)), np.zeros(3, dtype=np.int64))
    assert v.tolist() == [2.5, 2.5, 2.5]
    # isotropic -> m I (corollary)
    T = oc.as_tensor(np.array([2.0, 3.0]), 3)
    assert np.array_equal(T, np.stack([2 * np.eye(3), 3 * np.eye(3)]))


@pytest.mark.parametrize("d", [2, 3])
def test_elementwise_route_on_sampled_cells_matches_csr(d):
    """bench.py's cpu_baseline times the element route on a cell sample built with
    cell_elements; on the whole mesh that route is the CSR route."""
    from oracle.mesh import Mesh
    N, p = (4, 2) if d == 2 else (2, 2)
    cells = np.arange(N ** d)
    elems = cell_elements(d, N, cells)
    M = N + 1
    ids = np.arange(M ** d)
    vlat = np.stack([(ids // M ** a) % M for a in range(d)], axis=1)
    sub = Mesh(d, N, vlat, vlat / N, elems, np.repeat(cells, 2 if d == 2 else 6))
    ed_sub = oa.ElementData(sub, p)
    ed = oa.build(d, N, p)
    coef = _coef(d, N, 1)
    u = np.random.default_rng(0).uniform(-1, 1, ed.ndof)
    y = oa.assemble_csr(ed, 1, coef) @ u
    assert np.abs(oa.apply_elementwise(ed_sub, 1, coef, u) - y).max() <= 1e-14 * np.abs(y).max()


def test_row_kinds_cover_every_kind():
    """The row selection above really contains every topological DoF kind."""
    for d, p in itertools.product((2, 3), (2, 3)):
        N = 3
        rows = _rows_by_kind(d, N, p, np.random.default_rng(0))
        lat = dof_lattice(d, N, p)[rows]
        kinds = set(((lat % p) == 0).sum(axis=1).tolist())
        assert kinds == set(range(d + 1))


# ------------------------------------------------------------------ quadrature-point route
@pytest.mark.parametrize("d,p,form", [(d, p, f) for d in (2, 3) for p in (1, 2, 3, 4) for f in (0, 1)])
def test_qp_route_equals_csr(d, p, form):
    """The full-size residual checker (apply_qp_route, no K_T formed) is the CSR
    route's operator: plain and Dirichlet-eliminated, sequential and threaded."""
    from oracle.mesh import boundary_mask
    N = 4 if d == 2 else 2
    verts = _jittered_vertices(d, N, seed=5)
    coef = _coef(d, N, form)
    ed = oa.build(d, N, p, verts)
    u = np.random.default_rng(11).uniform(-1, 1, ed.ndof)
    A = oa.assemble_csr(ed, form, coef)
    y = A @ u
    yq = oa.apply_qp_route(ed, form, coef, u, chunk=7)
    assert np.abs(yq - y).max() <= 1e-14 * np.abs(y).max()
    assert np.array_equal(oa.apply_qp_route(ed, form, coef, u, chunk=7, workers=3), yq)
    if form == 1:
        mask = boundary_mask(d, N, p)
        yd = oa.dirichlet_matrix(A, mask) @ u
        assert np.abs(oa.apply_qp_route(ed, form, coef, u, dirichlet=True) - yd).max() <= 1e-14 * np.abs(yd).max()


@pytest.mark.parametrize("d,p", [(2, 2), (3, 4)])
def test_wp_total_is_one_A_one(d, p):
    from oracle import dogip as od
    N = 3 if d == 2 else 2
    verts = _jittered_vertices(d, N, seed=6)
    coef = _coef(d, N, 0)
    ed = oa.build(d, N, p, verts)
    A = oa.assemble_csr(ed, 0, coef)
    one = np.ones(ed.ndof)
    t = oa.wp_total(ed, coef, chunk=5)
    assert abs(t - one @ (A @ one)) <= 1e-14 * abs(t)
    assert abs(t - od.element_weights(ed, 0, coef).sum()) <= 1e-14 * abs(t)      # sum_T sum_j a_{T,j}
    assert oa.wp_total(ed, coef, chunk=5, workers=2) == pytest.approx(t, rel=1e-15)
    # closed form: m = 1 gives |Omega| = 1 on any (jittered) mesh
    assert abs(oa.wp_total(ed, Coefficient(COEF_CONST, np.array([1.0]))) - 1.0) <= 1e-14


def test_qp_route_threads_equal_sequential_on_large_chunks():
    """Threaded chunks (the full-size residual checks use workers > 1) give the sequential
    result on chunks big enough for a multithreaded BLAS GEMM -- the configuration in which
    concurrent OpenBLAS calls once corrupted the full-size C3 check."""
    from synth.configs import get_config
    c = get_config("C3").with_size(16)
    ed = oa.build(3, 16, 2)
    coef = c.coefficient()
    u = c.u()
    y1 = oa.apply_qp_route(ed, 1, coef, u, workers=1, chunk=8192)
    for _ in range(3):
        y8 = oa.apply_qp_route(ed, 1, coef, u, workers=8, chunk=8192)
        assert np.abs(y8 - y1).max() <= 1e-15 * np.abs(y1).max()
