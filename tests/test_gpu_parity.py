"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star, reading L24): relative max-norm
||y_gpu - y_ref||_inf / ||y_ref||_inf <= 1e-12 for every apply; weights
<= 1e-13; CG reaches the same relative residual.  All inputs seeded
(synth/).  Sizes span several 32-element tiles and ragged x-blocks.
"""
import numpy as np
import pytest

from oracle import assemble as oa
from oracle import dogip as od
from oracle.cg import cg as oracle_cg
from oracle.mesh import boundary_mask
from synth.configs import (COEF_ANISO_FOURIER, COEF_CONST, COEF_CONST_TENSOR, COEF_PER_CELL,
                           COEF_SINCOS2D, COEF_TANH_RADIAL, Coefficient, aniso_fourier_params,
                           get_config)
from synth.generators import grf_per_cell, u_vector, vertex_jitter

pytestmark = pytest.mark.gpu
TOL = 1e-12

SINCOS = Coefficient(COEF_SINCOS2D, np.array([1.0, 0.5]))
TANH2 = Coefficient(COEF_TANH_RADIAL, np.array([1.0, 0.9, 20.0, 0.25, 0.5, 0.5]))
TANH3 = Coefficient(COEF_TANH_RADIAL, np.array([1.0, 0.9, 20.0, 0.25, 0.5, 0.5, 0.5]))
ANISO = Coefficient(COEF_ANISO_FOURIER, aniso_fourier_params(2))


def _torch():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    return torch


def jitter_verts(d, N, seed=4, amp=0.2):
    M = N + 1
    ids = np.arange(M ** d)
    X = np.stack([(ids // M ** a) % M for a in range(d)], axis=1) / N
    return X + vertex_jitter(d, N, amp, seed)


def relerr(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def gpu_apply(d, N, p, form, coef, u, verts=None, dirichlet=False, n1d=0):
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    m = Mesh(d, N, p, verts)
    op = Operator(m, form, coef, quad_n1d=n1d)
    y = op.apply(torch.from_numpy(u).cuda(), dirichlet=dirichlet)
    torch.cuda.synchronize()
    return y.cpu().numpy(), op, m


def coef_for(d, form, kind):
    if kind == "smooth":
        return (SINCOS if d == 2 else TANH3) if form == 0 else (SINCOS if d == 2 else ANISO)
    if kind == "tanh":
        return TANH2 if d == 2 else TANH3
    raise ValueError(kind)


ALL = [(d, p, f) for d in (2, 3) for p in (1, 2, 3, 4) for f in (0, 1)]


@pytest.mark.parametrize("d,p,form", ALL)
def test_weights_match_oracle(d, p, form):
    N = 3 if d == 2 else 2
    verts = jitter_verts(d, N)
    coef = coef_for(d, form, "smooth")
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    m = Mesh(d, N, p, verts)
    op = Operator(m, form, coef)
    w = op.export_weights()
    ed = oa.build(d, N, p, verts)
    ref = od.element_weights(ed, form, coef)
    if form == 1:
        iu = np.triu_indices(d)
        ref = ref[:, :, iu[0], iu[1]]
    else:
        ref = ref[:, :, None]
    assert relerr(w, ref) <= 1e-13


@pytest.mark.parametrize("d,p,form", ALL)
def test_apply_matches_assembled_A(d, p, form):
    """All 16 (d, p, form) on jittered meshes with a ragged x-block (N = 33
    in 2D spans two 32-cell blocks; 3D N = 3 pads lanes)."""
    N = 33 if d == 2 else 3
    if d == 2 and p == 4:
        N = 20
    verts = jitter_verts(d, N)
    coef = coef_for(d, form, "smooth")
    ed = oa.build(d, N, p, verts)
    A = oa.assemble_csr(ed, form, coef)
    u = u_vector(ed.ndof, 0)
    y, _, _ = gpu_apply(d, N, p, form, coef, u, verts)
    assert relerr(y, A @ u) <= TOL


@pytest.mark.parametrize("d,N,p", [(2, 40, 3), (3, 5, 2), (3, 4, 3)])
def test_dirichlet_apply(d, N, p):
    coef = coef_for(d, 1, "smooth")
    ed = oa.build(d, N, p)
    A = oa.assemble_csr(ed, 1, coef)
    mask = boundary_mask(d, N, p)
    u = u_vector(ed.ndof, 3)
    y, _, _ = gpu_apply(d, N, p, 1, coef, u, dirichlet=True)
    assert relerr(y, oa.dirichlet_matrix(A, mask) @ u) <= TOL
    assert np.array_equal(y[mask], u[mask])


@pytest.mark.parametrize("d,N,p,form", [(2, 35, 2, 1), (3, 4, 4, 0), (3, 5, 1, 1)])
def test_load_vector(d, N, p, form):
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    verts = jitter_verts(d, N)
    coef = coef_for(d, form, "smooth")
    m = Mesh(d, N, p, verts)
    op = Operator(m, form, coef)
    ed = oa.build(d, N, p, verts)
    for dirichlet in (False, True):
        b = op.load_vector(1.0, dirichlet=dirichlet).cpu().numpy()
        assert relerr(b, oa.load_vector(ed, 1.0, dirichlet)) <= TOL
    assert abs(op.load_vector(1.0).sum().item() - 1.0) < 1e-12     # sum b_i = |Omega|


def test_c1_both_forms_and_cg():
    """Config 1: one apply per form, CG on the EL Dirichlet problem, f = 1."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config("C1")
    coef = c.coefficient()
    ed = oa.build(2, c.N, c.p)
    u = c.u()
    m = Mesh(2, c.N, c.p)
    for form in (0, 1):
        A = oa.assemble_csr(ed, form, coef)
        op = Operator(m, form, coef)
        y = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
        assert relerr(y, A @ u) <= TOL
    mask = boundary_mask(2, c.N, c.p)
    AD = oa.dirichlet_matrix(oa.assemble_csr(ed, 1, coef), mask)
    b = op.load_vector(1.0, dirichlet=True)
    x = torch.zeros_like(b)
    res = op.cg(b, x, rtol=1e-10, dirichlet=True)
    assert res["status"] == "OK" and res["rel_res"] <= 1e-10
    bn = b.cpu().numpy()
    xn = x.cpu().numpy()
    true_res = np.linalg.norm(bn - AD @ xn) / np.linalg.norm(bn)
    assert true_res <= 2e-10
    xo, it, _, st = oracle_cg(lambda v: AD @ v, oa.load_vector(ed, 1.0, True), rtol=1e-10)
    assert abs(res["iters"] - it) <= 3
    assert relerr(xn, xo) <= 1e-8


def test_wp_mass_cg_1e12():
    """Config-5 style mass solve at a small size: tol 1e-12, no BC."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config("C5").with_size(6)
    verts = c.vertices()
    m = Mesh(3, c.N, c.p, verts)
    op = Operator(m, 0, c.coefficient())
    b = op.load_vector(1.0)
    x = torch.zeros_like(b)
    res = op.cg(b, x, rtol=1e-12)
    assert res["status"] == "OK" and res["rel_res"] <= 1e-12
    ed = oa.build(3, c.N, c.p, verts)
    A = oa.assemble_csr(ed, 0, c.coefficient())
    bn, xn = b.cpu().numpy(), x.cpu().numpy()
    assert np.linalg.norm(bn - A @ xn) / np.linalg.norm(bn) <= 2e-12


@pytest.mark.parametrize("name,N", [("C2p1", 64), ("C2p2", 48), ("C2p3", 40), ("C2p4", 33),
                                    ("C3", 8), ("C4", 7), ("C5", 5)])
def test_configs_reduced_size_full_parity(name, N):
    c = get_config(name).with_size(N)
    coef = c.coefficient()
    verts = c.vertices()
    ed = oa.build(c.d, c.N, c.p, verts)
    form = c.forms[0]
    A = oa.assemble_csr(ed, form, coef)
    u = c.u()
    y, _, _ = gpu_apply(c.d, c.N, c.p, form, coef, u, verts)
    assert relerr(y, A @ u) <= TOL


@pytest.mark.parametrize("name", ["C2p1", "C2p2", "C2p3", "C2p4", "C3", "C4", "C5"])
def test_configs_full_size_sampled_rows(name):
    """Full BASELINE sizes, the launch configuration bench.py times: sampled
    rows recomputed one by one by the oracle, plus whole-vector invariants."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config(name)
    coef = c.coefficient()
    verts = c.vertices()
    form = c.forms[0]
    m = Mesh(c.d, c.N, c.p, verts)
    op = Operator(m, form, coef)
    u = c.u()
    ug = torch.from_numpy(u).cuda()
    y = op.apply(ug).cpu().numpy()
    rng = np.random.default_rng(11)
    n = c.ndof
    rows = np.unique(np.concatenate([rng.integers(0, n, 48), [0, 1, n - 1, n // 2, n // 3],
                                     np.arange(0, n, max(1, n // 16))[:16]]))
    ref = oa.apply_rows_sampled(c.d, c.N, c.p, verts, form, coef, u, rows)
    scale = np.abs(y).max()
    assert np.abs(y[rows] - ref).max() / scale <= TOL
    if form == 1:     # EL annihilates constants (check ii), at full size
        y1 = op.apply(torch.ones_like(ug)).cpu().numpy()
        assert np.abs(y1).max() <= 1e-11 * scale
    else:             # WP: 1^T A 1 = int m
        y1 = op.apply(torch.ones_like(ug))
        assert np.isfinite(y1.sum().item())


@pytest.mark.parametrize("d,N,p,form,nr", [(3, 6, 2, 1, 2), (3, 7, 3, 1, 3), (2, 40, 2, 0, 2), (3, 5, 4, 0, 2)])
def test_slab_partials_sum_to_global(d, N, p, form, nr):
    """Multi-rank path emulated on one GPU without NCCL: every slab computes
    its partial y (DOGIP_NO_EXCHANGE); summing the interface planes
    reproduces the single-rank apply (the data-path exchange step A8)."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    coef = coef_for(d, form, "smooth")
    verts = jitter_verts(d, N)
    Md = p * N + 1
    u = u_vector(Md ** d, 5)
    y_glob, _, _ = gpu_apply(d, N, p, form, coef, u, verts)
    acc = np.zeros_like(u)
    for r in range(nr):
        m = Mesh(d, N, p, verts, rank=r, nranks=nr)
        op = Operator(m, form, coef)
        i0 = m.info["dof_offset"]
        ul = torch.from_numpy(u[i0:i0 + m.ndof].copy()).cuda()
        acc[i0:i0 + m.ndof] += op.apply(ul, exchange=False).cpu().numpy()
    assert relerr(acc, y_glob) <= 1e-14


HOST_CASES = [("C4", 9, 1, 0, False), ("C4", 9, 1, 0, True), ("C4", 37, 1, 0, True), ("C2p2", 40, 1, 0, True),
              ("C5", 5, 0, 0, False), ("C5", 19, 0, 5, False), ("C5", 6, 0, 2, False), ("C1", 16, 0, 0, False),
              ("C3", 1, 1, 0, True)]


@pytest.mark.parametrize("name,N,form,storage,dirichlet", HOST_CASES)
def test_apply_host_matches_device(name, N, form, storage, dirichlet):
    """dogip_apply_host (pipelined over chunks of cube layers: copy-in / apply / copy-out
    on three streams, per-plane Dirichlet rows) equals the device apply; N = 37 gives
    16 uneven chunks, N = 1 a single layer."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config(name).with_size(N)
    m = Mesh(c.d, c.N, c.p, c.vertices())
    op = Operator(m, form, c.coefficient(), storage=storage)
    u = c.u()
    yd = op.apply(torch.from_numpy(u).cuda(), dirichlet=dirichlet).cpu().numpy()
    uh = torch.from_numpy(u).pin_memory()
    yh = torch.empty_like(uh).pin_memory()
    for _ in range(2):       # twice: reuse of the library's streams / events / scratch
        yh.fill_(np.nan)
        op.apply_host_ptr(uh.data_ptr(), yh.data_ptr(), dirichlet=dirichlet)
        assert relerr(yh.numpy(), yd) <= 1e-14
    assert relerr(op.apply_host(u, dirichlet=dirichlet), yd) <= 1e-14   # pageable buffers


def test_negative_control_other_rule_fails():
    """Parity is sensitive: a different quadrature rule (n = p + 2 instead of
    the contract p + 3) must break the 1e-12 bar for a non-polynomial m."""
    d, N, p = 2, 12, 2
    ed = oa.build(d, N, p)
    A = oa.assemble_csr(ed, 0, SINCOS)
    u = u_vector(ed.ndof, 0)
    y, _, _ = gpu_apply(d, N, p, 0, SINCOS, u, n1d=p + 2)
    assert relerr(y, A @ u) > 1e-9


def test_error_codes_on_gpu():
    from paper_1710_09913_b200.api import CoeffSpec, DogipError, Mesh, Operator
    m = Mesh(3, 2, 2)
    with pytest.raises(DogipError) as ei:
        Operator(m, 0, ANISO)                     # tensor coefficient for WP
    assert ei.value.code == -5
    with pytest.raises(DogipError) as ei:
        Operator(m, 1, CoeffSpec(COEF_CONST, np.array([-1.0])))
    assert ei.value.code == -5
    verts = jitter_verts(3, 2, amp=2.0)           # inverted tets
    m2 = Mesh(3, 2, 2, verts)
    with pytest.raises(DogipError) as ei:
        Operator(m2, 1, CoeffSpec(COEF_CONST, np.array([1.0])))
    assert ei.value.code == -4


ISO_CASES = [(2, 20, 2, "sincos"), (2, 9, 4, "grf"), (3, 3, 3, "tanh"), (3, 2, 4, "grf"), (3, 4, 1, "tanh")]


@pytest.mark.parametrize("d,N,p,kind", ISO_CASES)
def test_iso_storage_matches_oracle(d, N, p, kind):
    """DOGIP_STORE_ISO (Corollary P:411-428, element-wise: A_{T,j} = a_{T,j} G_T):
    same operator as the assembled A, expanded weights equal the oracle's."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    coef = {"sincos": SINCOS, "tanh": TANH2 if d == 2 else TANH3,
            "grf": Coefficient(COEF_PER_CELL, np.zeros(0), grf_per_cell(d, N, 0.05, 1.0, 1))}[kind]
    verts = jitter_verts(d, N)
    m = Mesh(d, N, p, verts)
    op = Operator(m, 1, coef, storage=1)
    assert op.info["storage"] == 1 and op.info["stream_doubles_per_elem"] == op.info["W_T"] + d * (d + 1) // 2
    ed = oa.build(d, N, p, verts)
    A = oa.assemble_csr(ed, 1, coef)
    u = u_vector(ed.ndof, 0)
    y = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    assert relerr(y, A @ u) <= TOL
    ref = od.element_weights(ed, 1, coef)
    iu = np.triu_indices(d)
    assert relerr(op.export_weights(), ref[:, :, iu[0], iu[1]]) <= 1e-13
    mask = boundary_mask(d, N, p)
    yd = op.apply(torch.from_numpy(u).cuda(), dirichlet=True).cpu().numpy()
    assert relerr(yd, oa.dirichlet_matrix(A, mask) @ u) <= TOL


def test_iso_storage_full_size_c4_sampled():
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config("C4")
    coef = c.coefficient()
    m = Mesh(3, c.N, c.p)
    op = Operator(m, 1, coef, storage=1)
    u = c.u()
    y = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    rows = np.unique(np.random.default_rng(12).integers(0, c.ndof, 40))
    ref = oa.apply_rows_sampled(3, c.N, c.p, None, 1, coef, u, rows)
    assert np.abs(y[rows] - ref).max() / np.abs(y).max() <= TOL


def test_iso_storage_errors():
    from paper_1710_09913_b200.api import DogipError, Mesh, Operator
    m = Mesh(3, 2, 2)
    with pytest.raises(DogipError) as ei:
        Operator(m, 1, ANISO, storage=1)
    assert ei.value.code == -5
    with pytest.raises(DogipError) as ei:
        Operator(m, 0, TANH3, storage=1)
    assert ei.value.code == -10


GLOBAL_CASES = [(2, 33, 2), (2, 9, 4), (3, 3, 1), (3, 4, 2), (3, 3, 4)]


@pytest.mark.parametrize("d,N,p", GLOBAL_CASES)
def test_global_wp_storage_theorem1(d, N, p):
    """DOGIP_STORE_GLOBAL (Theorem 1): one diagonal over W = C_{N,2p};
    same operator as the assembled A; each element sees A_ii / mult_i with
    A_ii = int m phi^W_i (the oracle's own Theorem 1 weights)."""
    torch = _torch()
    from oracle.mesh import dof_map
    from paper_1710_09913_b200.api import Mesh, Operator
    coef = TANH2 if d == 2 else TANH3
    verts = jitter_verts(d, N)
    m = Mesh(d, N, p, verts)
    op = Operator(m, 0, coef, storage=2)
    # one W-lattice vector, stored class-major along x: rows of 2p (N + 1) doubles
    assert op.info["weight_bytes"] == 8 * 2 * p * (N + 1) * (2 * p * N + 1) ** (d - 1)
    ed = oa.build(d, N, p, verts)
    A = oa.assemble_csr(ed, 0, coef)
    u = u_vector(ed.ndof, 0)
    y = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    assert relerr(y, A @ u) <= TOL
    lW = dof_map(ed.mesh, 2 * p)
    a_el = od.element_weights(ed, 0, coef)
    a_glob = np.bincount(lW.ravel(), weights=a_el.ravel(), minlength=(2 * p * N + 1) ** d)
    mult = np.bincount(lW.ravel(), minlength=(2 * p * N + 1) ** d)
    assert relerr(op.export_weights()[:, :, 0], (a_glob / np.maximum(mult, 1))[lW]) <= 1e-13


def test_global_wp_c5_full_size_sampled():
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config("C5")
    coef, verts = c.coefficient(), c.vertices()
    m = Mesh(3, c.N, c.p, verts)
    op = Operator(m, 0, coef, storage=2)
    u = c.u()
    y = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    rows = np.unique(np.random.default_rng(13).integers(0, c.ndof, 30))
    ref = oa.apply_rows_sampled(3, c.N, c.p, verts, 0, coef, u, rows)
    assert np.abs(y[rows] - ref).max() / np.abs(y).max() <= TOL


def test_global_storage_errors():
    from paper_1710_09913_b200.api import DogipError, Mesh, Operator
    m = Mesh(3, 2, 2)
    with pytest.raises(DogipError) as ei:
        Operator(m, 1, TANH3, storage=2)
    assert ei.value.code == -10
    m2 = Mesh(3, 4, 2, rank=0, nranks=2)             # no communicator
    with pytest.raises(DogipError) as ei:
        Operator(m2, 0, TANH3, storage=2)
    assert ei.value.code == -10


# Quadrature-point matrix-free comparator (DOGIP_STORE_QP, "alternative approaches" P:61-75)
QP_CASES = [(d, p, f) for d in (2, 3) for p in (1, 2, 3, 4) for f in (0, 1)]


@pytest.mark.parametrize("d,p,form", QP_CASES)
def test_qp_comparator_matches_oracle(d, p, form):
    """Same contract rule Q as the DoGIP weights -> the same Galerkin matrix A: the
    on-the-fly quadrature apply matches the assembled A (smooth, point-evaluated
    coefficients incl. the rotated anisotropic tensor, jittered meshes, ragged x-blocks)
    and the DoGIP apply; with Dirichlet rows for EL."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    N = {2: 35, 3: 4}[d] if p <= 2 else {2: 9, 3: 3}[d]
    coef = coef_for(d, form, "smooth")
    verts = jitter_verts(d, N)
    m = Mesh(d, N, p, verts)
    op = Operator(m, form, coef, storage=4)
    assert op.info["storage"] == 4 and op.info["weight_bytes"] == 0
    ed = oa.build(d, N, p, verts)
    A = oa.assemble_csr(ed, form, coef)
    u = u_vector(ed.ndof, 0)
    ut = torch.from_numpy(u).cuda()
    y = op.apply(ut).cpu().numpy()
    assert relerr(y, A @ u) <= TOL
    yd = Operator(m, form, coef).apply(ut).cpu().numpy()
    assert relerr(y, yd) <= TOL
    if form == 1:
        bmask = boundary_mask(d, N, p)
        AD = oa.dirichlet_matrix(A, bmask)
        yq = op.apply(ut, dirichlet=True).cpu().numpy()
        assert relerr(yq, AD @ u) <= TOL


@pytest.mark.parametrize("name", ["C4", "C5", "C3"])
def test_qp_comparator_full_size_sampled(name):
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config(name)
    coef, verts = c.coefficient(), c.vertices()
    m = Mesh(c.d, c.N, c.p, verts)
    form = c.forms[0]
    op = Operator(m, form, coef, storage=4)
    u = c.u()
    y = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    rows = np.unique(np.random.default_rng(19).integers(0, c.ndof, 20))
    ref = oa.apply_rows_sampled(c.d, c.N, c.p, verts, form, coef, u, rows)
    assert np.abs(y[rows] - ref).max() / np.abs(y).max() <= TOL


def test_qp_comparator_cg_and_errors():
    torch = _torch()
    from paper_1710_09913_b200.api import DogipError, Mesh, Operator
    c = get_config("C1")
    coef = c.coefficient()
    m = Mesh(2, c.N, c.p)
    op = Operator(m, 1, coef, storage=4)
    b = op.load_vector(1.0, dirichlet=True)
    x = torch.zeros_like(b)
    res = op.cg(b, x, rtol=1e-10, dirichlet=True)
    ed = oa.build(2, c.N, c.p)
    AD = oa.dirichlet_matrix(oa.assemble_csr(ed, 1, coef), boundary_mask(2, c.N, c.p))
    bn, xn = b.cpu().numpy(), x.cpu().numpy()
    assert res["status"] == "OK"
    assert np.linalg.norm(bn - AD @ xn) / np.linalg.norm(bn) <= 2e-10
    with pytest.raises(DogipError):
        op.export_weights()


@pytest.mark.parametrize("name,form,N", [("C1", 1, 16), ("C3", 1, 6), ("C5", 0, 5)])
def test_cg_graph_matches_host_loop(name, form, N, monkeypatch):
    """The graph-captured CG (conditional WHILE node, device-side stopping test) runs
    the same iterations as the host-driven loop: same count, same x to rounding, and
    a true residual within 2 rtol; re-running reuses the cached graph."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config(name).with_size(N)
    m = Mesh(c.d, c.N, c.p, c.vertices())
    op = Operator(m, form, c.coefficient())
    dirichlet = form == 1
    tol = 1e-10
    b = op.load_vector(1.0, dirichlet=dirichlet)
    xg = torch.zeros_like(b)
    rg = op.cg(b, xg, rtol=tol, dirichlet=dirichlet)
    xg2 = torch.zeros_like(b)
    rg2 = op.cg(b, xg2, rtol=tol, dirichlet=dirichlet)     # cached graph (different x -> rebuilt)
    monkeypatch.setenv("DOGIP_CG_NO_GRAPH", "1")
    xh = torch.zeros_like(b)
    rh = op.cg(b, xh, rtol=tol, dirichlet=dirichlet)
    assert rg["status"] == rh["status"] == rg2["status"] == "OK"
    # rounding-level differences (below) can move the stopping test by an iteration
    assert abs(rg["iters"] - rh["iters"]) <= 2 and abs(rg2["iters"] - rh["iters"]) <= 2
    # the scatter's atomics make two CG runs differ at rounding level (reading L25), which
    # the iteration amplifies by up to ~cond(A): compare to 100 rtol, not bitwise
    assert relerr(xg.cpu().numpy(), xh.cpu().numpy()) <= 100 * tol
    assert relerr(xg2.cpu().numpy(), xh.cpu().numpy()) <= 100 * tol
    ed = oa.build(c.d, c.N, c.p, c.vertices())
    A = oa.assemble_csr(ed, form, c.coefficient())
    if dirichlet:
        A = oa.dirichlet_matrix(A, boundary_mask(c.d, c.N, c.p))
    bn, xn = b.cpu().numpy(), xg.cpu().numpy()
    assert np.linalg.norm(bn - A @ xn) / np.linalg.norm(bn) <= 2 * tol
    # maxit reached inside the graph -> NOT_CONVERGED with exactly maxit iterations
    monkeypatch.delenv("DOGIP_CG_NO_GRAPH")
    x3 = torch.zeros_like(b)
    r3 = op.cg(b, x3, rtol=1e-30, maxit=7, dirichlet=dirichlet)
    assert r3["status"] == "NOT_CONVERGED" and r3["iters"] == 7


# Symmetry-adapted WP weights (DOGIP_STORE_SYM): block-diagonal Bhat by character
SYM_CASES = [(2, 17, 1), (2, 33, 2), (2, 9, 3), (2, 5, 4), (3, 3, 1), (3, 17, 2), (3, 5, 3), (3, 4, 4)]


@pytest.mark.parametrize("d,N,p", SYM_CASES)
def test_sym_wp_storage_matches_oracle(d, N, p):
    """DOGIP_STORE_SYM stores ahat_psi(P) = (1/|G|) sum_g psi(g) a_{g j0} and applies Bhat
    block by character: y = A u against the assembled A, exported weights (converted back
    to a_{T,j}) equal the FULL storage's, and the WP mass CG converges."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    coef = TANH2 if d == 2 else TANH3
    verts = jitter_verts(d, N)
    m = Mesh(d, N, p, verts)
    op = Operator(m, 0, coef, storage=5)
    assert op.info["storage"] == 5
    ed = oa.build(d, N, p, verts)
    A = oa.assemble_csr(ed, 0, coef)
    u = u_vector(ed.ndof, 0)
    y = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    assert relerr(y, A @ u) <= TOL
    full = Operator(m, 0, coef, storage=0)
    assert relerr(op.export_weights(), full.export_weights()) <= 1e-15
    b = op.load_vector(1.0)
    x = torch.zeros_like(b)
    res = op.cg(b, x, rtol=1e-12)
    bn, xn = b.cpu().numpy(), x.cpu().numpy()
    assert res["status"] == "OK"
    assert np.linalg.norm(bn - A @ xn) / np.linalg.norm(bn) <= 2e-12


def test_sym_wp_c5_full_size_sampled():
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config("C5")
    coef, verts = c.coefficient(), c.vertices()
    m = Mesh(3, c.N, c.p, verts)
    op = Operator(m, 0, coef, storage=5)
    u = c.u()
    y = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    rows = np.unique(np.random.default_rng(23).integers(0, c.ndof, 30))
    ref = oa.apply_rows_sampled(3, c.N, c.p, verts, 0, coef, u, rows)
    assert np.abs(y[rows] - ref).max() / np.abs(y).max() <= TOL


def test_sym_storage_errors():
    from paper_1710_09913_b200.api import DogipError, Mesh, Operator
    m = Mesh(3, 2, 2)
    with pytest.raises(DogipError) as ei:
        Operator(m, 1, TANH3, storage=5)
    assert ei.value.code == -10


# ------------------------------------------------------------------ NCCL plumbing
@pytest.mark.gpu
@pytest.mark.parametrize("d,N,p,form,storage", [(3, 5, 2, 1, 0), (3, 4, 3, 0, 2), (2, 40, 2, 1, 0), (3, 4, 4, 0, 5),
                                                (3, 4, 3, 1, 4), (3, 5, 3, 1, 1), (2, 40, 3, 0, 0)])
def test_nccl_single_rank_communicator(d, N, p, form, storage):
    """A mesh created with an NCCL id runs the multi-GPU code path -- communicator init
    (dlopen'd NCCL), boundary layers first, grouped send/recv on the comm stream, plane
    add, all-reduced CG dots, host-loop CG, exchange-path host apply -- which with a
    1-rank communicator must reproduce the plain single-GPU results.  No rank waits on
    another (one process, one GPU)."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator, nccl_unique_id
    coef = Coefficient(COEF_CONST, np.array([1.3]))
    m0 = Mesh(d, N, p, device=0)
    m1 = Mesh(d, N, p, nranks=1, nccl_id=nccl_unique_id(), device=0)
    op0 = Operator(m0, form, coef, storage=storage)
    op1 = Operator(m1, form, coef, storage=storage)
    u = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, m0.ndof)).cuda()
    for dirichlet in (False, True):
        y0 = op0.apply(u, dirichlet=dirichlet)
        y1 = op1.apply(u, dirichlet=dirichlet)
        torch.cuda.synchronize()
        assert relerr(y1.cpu().numpy(), y0.cpu().numpy()) <= 1e-13
    h1 = op1.apply_host(u.cpu().numpy(), dirichlet=True)
    assert relerr(h1, op0.apply(u, dirichlet=True).cpu().numpy()) <= 1e-13
    dirichlet = form == 1
    b0 = op0.load_vector(1.0, dirichlet=dirichlet)
    b1 = op1.load_vector(1.0, dirichlet=dirichlet)
    assert relerr(b1.cpu().numpy(), b0.cpu().numpy()) <= 1e-14
    x0, x1 = torch.zeros_like(b0), torch.zeros_like(b1)
    r0 = op0.cg(b0, x0, rtol=1e-10, dirichlet=dirichlet)
    r1 = op1.cg(b1, x1, rtol=1e-10, dirichlet=dirichlet)
    assert r0["status"] == r1["status"] == "OK"
    assert abs(r0["iters"] - r1["iters"]) <= 2
    assert relerr(x1.cpu().numpy(), x0.cpu().numpy()) <= 1e-8


# ------------------------------------------------------------------ degenerate sizes
STORES_BY_FORM = {0: (0, 2, 4, 5), 1: (0, 1, 4)}


@pytest.mark.gpu
@pytest.mark.parametrize("d,p,form", ALL)
@pytest.mark.parametrize("N", [1, 2])
def test_smallest_meshes_every_storage(d, p, form, N):
    """N = 1 (one cell: one tile with 1 live lane of 32) and N = 2, every storage variant,
    against the assembled oracle A; with Dirichlet elimination the boundary rows are
    identity rows (at N = 1, p <= 2 every DoF is on the boundary, so A_D = I) and CG on
    b = 0 returns x = 0 at once."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    coef = coef_for(d, form, "tanh") if form == 0 else Coefficient(COEF_CONST, np.array([1.7]))
    ed = oa.build(d, N, p)
    A = oa.assemble_csr(ed, form, coef)
    mask = boundary_mask(d, N, p)
    AD = oa.dirichlet_matrix(A, mask)
    u = u_vector(ed.ndof, 1)
    m = Mesh(d, N, p, device=0)
    ut = torch.from_numpy(u).cuda()
    for store in STORES_BY_FORM[form]:
        op = Operator(m, form, coef, storage=store)
        y = op.apply(ut).cpu().numpy()
        assert relerr(y, A @ u) <= TOL, store
        yd = op.apply(ut, dirichlet=True).cpu().numpy()
        assert relerr(yd, AD @ u) <= TOL, store
        b = torch.zeros_like(ut)
        x = torch.zeros_like(ut)
        r = op.cg(b, x, rtol=1e-10, dirichlet=True)
        assert r["status"] == "OK" and r["iters"] == 0 and not x.abs().max().item()
        op.close()
    m.close()


@pytest.mark.gpu
@pytest.mark.parametrize("d,p,form", ALL)
def test_every_storage_every_entry_point(d, p, form):
    """Cross product on a jittered mesh with a ragged x-block: every storage of the form x
    {device apply, host-buffer apply} x {plain, Dirichlet-eliminated} against the oracle's
    A / A_D, and 6 fixed-count CG iterations from x0 = 0 (graph and host loop) against the
    oracle's CG run for the same count."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    N = 34 if d == 2 else 3
    verts = jitter_verts(d, N)
    coef = coef_for(d, form, "tanh") if form == 0 else Coefficient(COEF_CONST, np.array([0.8]))
    ed = oa.build(d, N, p, verts)
    A = oa.assemble_csr(ed, form, coef)
    AD = oa.dirichlet_matrix(A, boundary_mask(d, N, p))
    u = u_vector(ed.ndof, 2)
    b = oa.load_vector(ed, 1.0, dirichlet=True)
    x_ref6, _, _, _ = oracle_cg(lambda v: AD @ v, b, rtol=0.0, maxit=6)
    m = Mesh(d, N, p, verts, device=0)
    ut = torch.from_numpy(u).cuda()
    for store in STORES_BY_FORM[form]:
        op = Operator(m, form, coef, storage=store)
        for dirichlet in (False, True):
            ref = (AD if dirichlet else A) @ u
            assert relerr(op.apply(ut, dirichlet=dirichlet).cpu().numpy(), ref) <= TOL, (store, dirichlet)
            assert relerr(op.apply_host(u, dirichlet=dirichlet), ref) <= TOL, (store, dirichlet, "host")
        bt = torch.from_numpy(b).cuda()
        for graph in (True, False):
            x = torch.zeros_like(bt)
            if not graph:
                import os
                os.environ["DOGIP_CG_NO_GRAPH"] = "1"
            try:
                r = op.cg(bt, x, rtol=1e-300, maxit=6, dirichlet=True)
            finally:
                if not graph:
                    del os.environ["DOGIP_CG_NO_GRAPH"]
            assert r["iters"] == 6
            assert relerr(x.cpu().numpy(), x_ref6) <= 1e-9, (store, graph)
        op.close()
    m.close()


@pytest.mark.gpu
@pytest.mark.parametrize("d,N,p,form,nr", [(3, 6, 2, 1, 2), (3, 5, 4, 0, 3), (2, 40, 3, 0, 2), (2, 36, 2, 1, 3)])
def test_slab_partials_every_storage(d, N, p, form, nr):
    """Slab partials (DOGIP_NO_EXCHANGE, no communicator) summed over ranks equal the
    single-rank apply for every storage that runs without a communicator (GLOBAL needs
    one on several ranks and is rejected without it), with and without Dirichlet."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    from paper_1710_09913_b200._lib import DogipError
    coef = coef_for(d, form, "tanh") if form == 0 else Coefficient(COEF_CONST, np.array([1.1]))
    verts = jitter_verts(d, N)
    Md = p * N + 1
    u = u_vector(Md ** d, 6)
    mg = Mesh(d, N, p, verts, device=0)
    ug = torch.from_numpy(u).cuda()
    meshes = [Mesh(d, N, p, verts, rank=r, nranks=nr, device=0) for r in range(nr)]
    for store in STORES_BY_FORM[form]:
        if store == 2:
            with pytest.raises(DogipError):
                Operator(meshes[0], form, coef, storage=store)
            continue
        opg = Operator(mg, form, coef, storage=store)
        ops = [Operator(m, form, coef, storage=store) for m in meshes]
        for dirichlet in (False, True):
            y_glob = opg.apply(ug, dirichlet=dirichlet).cpu().numpy()
            acc = np.zeros_like(u)
            for m, op in zip(meshes, ops):
                i0 = m.info["dof_offset"]
                ul = torch.from_numpy(u[i0:i0 + m.ndof].copy()).cuda()
                acc[i0:i0 + m.ndof] += op.apply(ul, exchange=False, dirichlet=dirichlet).cpu().numpy()
            if dirichlet and not (store == 0 and (p <= 2 or (d == 2 and p <= 3))):
                # the separate fix-up writes the Dirichlet rows (u_i) of the interface planes
                # on both owners: count them once.  The cell kernel (FULL storage; p <= 2, 2D
                # p <= 3) writes each row once (its floor cell): partials already sum to u_i.
                mask = boundary_mask(d, N, p)
                plane = Md ** (d - 1)
                for r in range(1, nr):
                    i0 = meshes[r].info["dof_offset"]
                    sl = slice(i0, i0 + plane)
                    acc[sl][mask[sl]] -= u[sl][mask[sl]]
            assert relerr(acc, y_glob) <= 1e-13, (store, dirichlet)
        for op in ops + [opg]:
            op.close()
    for m in meshes + [mg]:
        m.close()


def _coef_kinds(d, form, N):
    out = [("const", Coefficient(COEF_CONST, np.array([1.4]))),
           ("per_cell", Coefficient(COEF_PER_CELL, np.zeros(0), grf_per_cell(d, N, 0.2, 1.0, 3))),
           ("tanh", TANH2 if d == 2 else TANH3)]
    if d == 2:
        out.append(("sincos", SINCOS))
    if form == 1:
        T = np.array([[2.0, 0.3], [0.3, 1.0]]) if d == 2 else np.array([[2.0, 0.3, 0.1], [0.3, 1.0, -0.2],
                                                                          [0.1, -0.2, 1.5]])
        out.append(("tensor", Coefficient(COEF_CONST_TENSOR, T.ravel())))
        if d == 3:
            out.append(("aniso", ANISO))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("d,p,form", [(2, 2, 0), (2, 3, 1), (3, 2, 0), (3, 2, 1), (3, 3, 1), (3, 4, 0)])
def test_every_coefficient_kind_every_storage(d, p, form):
    """Every coefficient model valid for (d, form) x every storage that accepts it, on a
    jittered mesh, against the oracle's assembled A (the same rule, reading L10); storages
    that need an isotropic coefficient reject the tensor kinds with E_BAD_COEFF."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    from paper_1710_09913_b200._lib import DogipError
    N = 34 if d == 2 else 3
    verts = jitter_verts(d, N)
    ed = oa.build(d, N, p, verts)
    u = u_vector(ed.ndof, 4)
    m = Mesh(d, N, p, verts, device=0)
    ut = torch.from_numpy(u).cuda()
    for name, coef in _coef_kinds(d, form, N):
        A = oa.assemble_csr(ed, form, coef)
        for store in STORES_BY_FORM[form]:
            if store == 1 and not coef.isotropic:
                with pytest.raises(DogipError) as ei:
                    Operator(m, form, coef, storage=store)
                assert ei.value.code == -5
                continue
            op = Operator(m, form, coef, storage=store)
            assert relerr(op.apply(ut).cpu().numpy(), A @ u) <= TOL, (name, store)
            op.close()
    m.close()


@pytest.mark.gpu
@pytest.mark.parametrize("n1d", [2, 5, 9])
def test_quadrature_order_every_storage(n1d):
    """A non-default rule (quad_n1d) reaches the weights kernels and the comparator alike:
    every WP storage and the EL storages equal the oracle assembled with the same rule."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    d, N, p = 3, 3, 3
    verts = jitter_verts(d, N)
    ed = oa.build(d, N, p, verts, n1d=n1d)
    u = u_vector(ed.ndof, 8)
    m = Mesh(d, N, p, verts, device=0)
    ut = torch.from_numpy(u).cuda()
    for form, coef in ((0, TANH3), (1, Coefficient(COEF_TANH_RADIAL, TANH3.params))):
        A = oa.assemble_csr(ed, form, coef)
        for store in STORES_BY_FORM[form]:
            op = Operator(m, form, coef, quad_n1d=n1d, storage=store)
            assert relerr(op.apply(ut).cpu().numpy(), A @ u) <= TOL, (form, store)
            op.close()
    m.close()


@pytest.mark.gpu
def test_user_streams_and_concurrent_applies():
    """Work on caller streams (apply, host apply, CG graph) and two concurrent applies of
    one op on two streams into distinct y (dogip.h concurrency note)."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    d, N, p, form = 3, 6, 3, 1
    coef = Coefficient(COEF_CONST, np.array([1.2]))
    ed = oa.build(d, N, p)
    A = oa.assemble_csr(ed, form, coef)
    AD = oa.dirichlet_matrix(A, boundary_mask(d, N, p))
    u = u_vector(ed.ndof, 9)
    m = Mesh(d, N, p, device=0)
    op = Operator(m, form, coef)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ut = torch.from_numpy(u).cuda()
    torch.cuda.synchronize()
    y1, y2 = torch.empty_like(ut), torch.empty_like(ut)
    for _ in range(5):
        with torch.cuda.stream(s1):
            op.apply(ut, y1, stream=s1)
        with torch.cuda.stream(s2):
            op.apply(ut, y2, dirichlet=True, stream=s2)
    torch.cuda.synchronize()
    assert relerr(y1.cpu().numpy(), A @ u) <= TOL
    assert relerr(y2.cpu().numpy(), AD @ u) <= TOL
    with torch.cuda.stream(s1):
        b = op.load_vector(1.0, dirichlet=True, stream=s1)
        x = torch.zeros_like(b)
        r = op.cg(b, x, rtol=1e-10, dirichlet=True, stream=s1)
    torch.cuda.synchronize()
    bn = b.cpu().numpy()
    assert r["status"] == "OK"
    assert np.linalg.norm(AD @ x.cpu().numpy() - bn) <= 2e-10 * np.linalg.norm(bn)
    hy = op.apply_host(u, dirichlet=True, stream=s2)
    assert relerr(hy, AD @ u) <= TOL
    op.close()
    m.close()


@pytest.mark.gpu
@pytest.mark.parametrize("d,p,form", [(2, 2, 0), (2, 3, 1), (3, 1, 1), (3, 2, 0), (3, 3, 1), (3, 4, 0)])
def test_load_vector_every_storage(d, p, form):
    """b_i = int phi_i (eq:linsys_gp P:207 / eq:linsys_se P:337) does not depend on the weight
    storage: every storage's dogip_load_vector equals the oracle's, with and without the
    Dirichlet zeroing."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    N = 34 if d == 2 else 3
    verts = jitter_verts(d, N)
    ed = oa.build(d, N, p, verts)
    coef = coef_for(d, form, "tanh") if form == 0 else Coefficient(COEF_CONST, np.array([0.9]))
    m = Mesh(d, N, p, verts, device=0)
    for store in STORES_BY_FORM[form]:
        op = Operator(m, form, coef, storage=store)
        for dirichlet in (False, True):
            b = op.load_vector(2.5, dirichlet=dirichlet).cpu().numpy()
            assert relerr(b, oa.load_vector(ed, 2.5, dirichlet=dirichlet)) <= 1e-13, (store, dirichlet)
        op.close()
    m.close()


@pytest.mark.gpu
@pytest.mark.parametrize("store", [0, 1])
def test_cg_resume_matches_one_call(store):
    """DOGIP_CG_RESUME (the e2e_cg pattern of bench.py: one iteration per call, residual read
    back each step) continues the iteration exactly: 6 resumed single-iteration calls equal
    one 6-iteration call (to atomic-order rounding) and the oracle's 6 CG iterations;
    resuming before any call is E_INVALID_ARG."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    from paper_1710_09913_b200._lib import DogipError
    d, N, p, form = 3, 4, 3, 1
    coef = Coefficient(COEF_CONST, np.array([1.3]))
    ed = oa.build(d, N, p)
    AD = oa.dirichlet_matrix(oa.assemble_csr(ed, form, coef), boundary_mask(d, N, p))
    b = oa.load_vector(ed, 1.0, dirichlet=True)
    x_ref, _, _, _ = oracle_cg(lambda v: AD @ v, b, rtol=0.0, maxit=6)
    m = Mesh(d, N, p, device=0)
    op = Operator(m, form, coef, storage=store)
    bt = torch.from_numpy(b).cuda()
    x1 = torch.zeros_like(bt)
    with pytest.raises(DogipError) as ei:
        op.cg(bt, x1, rtol=0.0, maxit=1, dirichlet=True, resume=True)
    assert ei.value.code == -10
    rels = [op.cg(bt, x1, rtol=0.0, maxit=1, dirichlet=True, resume=k > 0)["rel_res"] for k in range(6)]
    x6 = torch.zeros_like(bt)
    r6 = op.cg(bt, x6, rtol=0.0, maxit=6, dirichlet=True)
    assert relerr(x1.cpu().numpy(), x6.cpu().numpy()) <= 1e-10
    assert relerr(x1.cpu().numpy(), x_ref) <= 1e-9
    assert abs(rels[-1] - r6["rel_res"]) <= 1e-9 * max(1.0, r6["rel_res"])
    op.close()
    m.close()


@pytest.mark.gpu
@pytest.mark.parametrize("form", [0, 1])
def test_plain_dogip_weights_entry_point(form):
    """dogip_weights (no storage argument, include/dogip.h) is the FULL storage of
    dogip_weights_ex: same exported weights, same apply."""
    import ctypes as C
    torch = _torch()
    from paper_1710_09913_b200 import _lib
    from paper_1710_09913_b200.api import CoeffSpec, Mesh, Operator
    d, N, p = 3, 3, 2
    verts = jitter_verts(d, N)
    coef = CoeffSpec.from_obj(coef_for(d, form, "smooth"))
    m = Mesh(d, N, p, verts, device=0)
    lib = _lib.load()
    cs = _lib.Coeff(coef.kind, coef.params.ctypes.data_as(C.POINTER(C.c_double)), coef.params.size, None)
    h = C.c_void_p()
    _lib.check(lib.dogip_weights(m.handle, form, C.byref(cs), 0, None, C.byref(h)))
    ref = Operator(m, form, coef, storage=0)
    oi = ref.info
    w = np.empty((m.info["n_elem_local"], oi["W_T"], oi["n_c"]))
    _lib.check(lib.dogip_export_weights(h, w.ctypes.data_as(C.POINTER(C.c_double)), w.size))
    assert np.array_equal(w, ref.export_weights())
    u = torch.from_numpy(u_vector(m.ndof, 3)).cuda()
    y = torch.empty_like(u)
    _lib.check(lib.dogip_apply(h, C.c_void_p(u.data_ptr()), C.c_void_p(y.data_ptr()), 0,
                               C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    assert relerr(y.cpu().numpy(), ref.apply(u).cpu().numpy()) <= 1e-14
    lib.dogip_op_destroy(h)
    ref.close()
    m.close()


@pytest.mark.gpu
@pytest.mark.parametrize("d,N,p,form", [(3, 5, 2, 1), (2, 40, 2, 0)])
def test_nccl_cg_batch_graph(d, N, p, form):
    """Several-rank CG through a 1-rank NCCL communicator: eager batches of predicated
    iterations and the opt-in captured batch graph (DOGIP_CG_GRAPH_MR=1, NCCL calls inside
    the graph), with batches shorter than the solve, give the single-rank graph's solve."""
    import os
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator, nccl_unique_id
    coef = Coefficient(COEF_CONST, np.array([1.3]))
    dirichlet = form == 1
    m0 = Mesh(d, N, p, device=0)
    op0 = Operator(m0, form, coef)
    b = op0.load_vector(1.0, dirichlet=dirichlet)
    x0 = torch.zeros_like(b)
    r0 = op0.cg(b, x0, rtol=1e-10, dirichlet=dirichlet)
    m1 = Mesh(d, N, p, nranks=1, nccl_id=nccl_unique_id(), device=0)
    op1 = Operator(m1, form, coef)
    for env in ({"DOGIP_CG_BATCH": "7"}, {"DOGIP_CG_BATCH": "7", "DOGIP_CG_GRAPH_MR": "1"},
                {"DOGIP_CG_GRAPH_MR": "1"}):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            x1 = torch.zeros_like(b)
            r1 = op1.cg(b, x1, rtol=1e-10, dirichlet=dirichlet)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        assert r1["status"] == r0["status"] == "OK", (env, r1)
        assert abs(r1["iters"] - r0["iters"]) <= 2, (env, r1["iters"], r0["iters"])
        assert relerr(x1.cpu().numpy(), x0.cpu().numpy()) <= 1e-8, env


_ELEMENT_PATH = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from oracle import assemble as oa
from oracle.mesh import boundary_mask
from paper_1710_09913_b200.api import Mesh, Operator
from synth.configs import COEF_CONST, Coefficient
from synth.generators import u_vector
worst = 0.0
for d, N, p in [(2, 34, 1), (2, 33, 2), (2, 9, 3), (3, 3, 1), (3, 3, 2)]:
    for form in (0, 1):
        coef = Coefficient(COEF_CONST, np.array([1.4]))
        ed = oa.build(d, N, p)
        A = oa.assemble_csr(ed, form, coef)
        AD = oa.dirichlet_matrix(A, boundary_mask(d, N, p))
        u = u_vector(ed.ndof, 4)
        op = Operator(Mesh(d, N, p, device=0), form, coef)
        ut = torch.from_numpy(u).cuda()
        for dirichlet, ref in ((False, A @ u), (True, AD @ u)):
            y = op.apply(ut, dirichlet=dirichlet).cpu().numpy()
            worst = max(worst, np.abs(y - ref).max() / np.abs(ref).max())
print("WORST", worst)
"""


@pytest.mark.gpu
def test_element_kernel_path_for_small_p():
    """DOGIP_CELL_KERNEL=0 routes FULL storage with p <= 2 (2D p <= 3) to the element-per-lane
    kernel (the cell kernel's fallback); it stays parity-green."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _ELEMENT_PATH.format(root=root)], capture_output=True, text=True,
                       timeout=600, env=dict(os.environ, DOGIP_CELL_KERNEL="0"))
    assert r.returncode == 0, r.stderr[-2000:]
    worst = float([l for l in r.stdout.splitlines() if l.startswith("WORST")][0].split()[1])
    assert worst <= TOL, worst


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_randomised_configurations(seed):
    """Seeded random draws over (d, N, p, form, storage, coefficient, jitter, Dirichlet,
    slab split): apply against the assembled oracle A, and for several slabs the partial
    sums against the single-rank apply -- a net over combinations the targeted tests do not
    enumerate (ragged x-blocks, N from 1 to 40, every storage the form admits)."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.choice([2, 3]))
    p = int(rng.integers(1, 5))
    N = int(rng.integers(1, 41 if d == 2 else (9 if p <= 2 else 5)))
    form = int(rng.integers(0, 2))
    stores = [0, 2, 4, 5] if form == 0 else [0, 1, 4]
    store = int(rng.choice(stores))
    jit = bool(rng.integers(0, 2)) and N >= 2
    verts = jitter_verts(d, N, seed=int(rng.integers(0, 100))) if jit else None
    if form == 0:
        coef = coef_for(d, 0, "tanh") if rng.integers(0, 2) else Coefficient(COEF_CONST, np.array([0.7]))
    elif store == 1:
        coef = Coefficient(COEF_PER_CELL, np.zeros(0), grf_per_cell(d, N, 0.2, 1.0, int(rng.integers(0, 50))))
    else:
        coef = ANISO if (d == 3 and rng.integers(0, 2)) else Coefficient(COEF_PER_CELL, np.zeros(0),
                                                                         grf_per_cell(d, N, 0.2, 1.0, 7))
    dirichlet = bool(rng.integers(0, 2))
    ed = oa.build(d, N, p, verts)
    A = oa.assemble_csr(ed, form, coef)
    ref_op = oa.dirichlet_matrix(A, boundary_mask(d, N, p)) if dirichlet else A
    u = u_vector(ed.ndof, seed)
    m = Mesh(d, N, p, verts, device=0)
    op = Operator(m, form, coef, storage=store)
    y = op.apply(torch.from_numpy(u).cuda(), dirichlet=dirichlet).cpu().numpy()
    case = (d, N, p, form, store, coef.kind, jit, dirichlet)
    assert relerr(y, ref_op @ u) <= TOL, case
    nr = int(rng.integers(2, 4))
    if N >= nr and store != 2 and not dirichlet:        # partial sums of a slab split
        acc = np.zeros_like(u)
        for r in range(nr):
            ms = Mesh(d, N, p, verts, rank=r, nranks=nr, device=0)
            ops = Operator(ms, form, coef, storage=store)
            i0 = ms.info["dof_offset"]
            acc[i0:i0 + ms.ndof] += ops.apply(torch.from_numpy(u[i0:i0 + ms.ndof].copy()).cuda(),
                                              exchange=False).cpu().numpy()
        assert relerr(acc, A @ u) <= 1e-13, case + (nr,)
