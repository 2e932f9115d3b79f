"""GPU parity at the full BASELINE sizes, in the launch configuration bench.py times.

* The Dirichlet-eliminated apply (the kernel instantiation bench.py's CG runs: C4 and
  C3 with DOGIP_DIRICHLET_ZERO, reading L14) against the oracle row by row:
  interior row i -> (A D u)_i from ``apply_rows_sampled`` on u with its boundary
  entries zeroed; boundary row i -> y_i = u_i exactly.  Rows include DoFs next to
  every face (the per-face masks) and the last x-block's lanes (ci = Nx - 1).
* The weighted projection at full size: 1^T A 1 equals the oracle's
  sum_T sum_j a_{T,j} = sum_T int_T m (Theorem 2; ``oracle.assemble.wp_total``).
* Negative control: one A_T entry perturbed through the test hook must break the
  1e-12 bar, and restoring it must restore parity.
"""
import os

import numpy as np
import pytest

from oracle import assemble as oa
from synth.configs import get_config
from synth.generators import u_vector

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _torch():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    return torch


def _boundary_zeroed(u, d, M):
    U = u.reshape((M,) * d).copy()
    for ax in range(d):
        sl = [slice(None)] * d
        sl[ax] = 0
        U[tuple(sl)] = 0.0
        sl[ax] = M - 1
        U[tuple(sl)] = 0.0
    return U.ravel()


def _rows_near_faces(d, N, p, rng, n_rand=40):
    """Random rows plus, per axis, rows at lattice coordinates 0, 1, p-1, p, pN-p, pN-1, pN
    (boundary, next to the boundary, the last cell's DoFs = lane 31 of the last x-block
    when N % 32 == 0) with the other coordinates random."""
    M = p * N + 1
    rows = list(rng.integers(0, M ** d, n_rand))
    special = sorted({0, 1, p - 1, p, p * N - p, p * N - 1, p * N, p * N - p + 1})
    for ax in range(d):
        for X in special:
            for _ in range(2):
                lat = rng.integers(0, M, d)
                lat[ax] = X
                rows.append(int(sum(int(lat[a]) * M ** a for a in range(d))))
    return np.unique(np.array(rows, dtype=np.int64))


@pytest.mark.parametrize("name", ["C3", "C4", "C2p1", "C2p2", "C2p3", "C2p4"])
def test_full_size_dirichlet_sampled_rows(name):
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config(name)
    coef, verts, form = c.coefficient(), c.vertices(), c.forms[0]
    m = Mesh(c.d, c.N, c.p, verts)
    op = Operator(m, form, coef)
    u = c.u()
    y = op.apply(torch.from_numpy(u).cuda(), dirichlet=True).cpu().numpy()
    M = c.p * c.N + 1
    rows = _rows_near_faces(c.d, c.N, c.p, np.random.default_rng(21))
    lat = np.stack([(rows // M ** a) % M for a in range(c.d)], axis=1)
    bnd = np.any((lat == 0) | (lat == M - 1), axis=1)
    assert bnd.any() and (~bnd).any()
    assert np.array_equal(y[rows[bnd]], u[rows[bnd]])           # identity rows, exactly
    ud = _boundary_zeroed(u, c.d, M)
    ref = oa.apply_rows_sampled(c.d, c.N, c.p, verts, form, coef, ud, rows[~bnd])
    scale = np.abs(y).max()
    assert np.abs(y[rows[~bnd]] - ref).max() / scale <= TOL
    # the whole boundary is identity, not just the sampled rows
    yb = y.reshape((M,) * c.d)
    ub = u.reshape((M,) * c.d)
    for ax in range(c.d):
        for X in (0, M - 1):
            sl = [slice(None)] * c.d
            sl[ax] = X
            assert np.array_equal(yb[tuple(sl)], ub[tuple(sl)])


def test_full_size_wp_total_c5():
    """1^T A 1 of the C5 weighted projection (5.3M jittered tets, tanh inclusion) against
    the oracle's sum over all elements of int_T m with the contract rule."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config("C5")
    coef, verts = c.coefficient(), c.vertices()
    m = Mesh(3, c.N, c.p, verts)
    ones = torch.ones(m.ndof, dtype=torch.float64, device="cuda")
    tot = {}
    for store in (0, 5):                  # FULL and the symmetry-adapted storage bench reports
        op = Operator(m, 0, coef, storage=store)
        tot[store] = op.apply(ones).sum().item()
        op.close()
    ed = oa.build(3, c.N, c.p, verts)
    ref = oa.wp_total(ed, coef, workers=min(32, os.cpu_count() or 1))
    for store, t in tot.items():
        assert abs(t - ref) <= TOL * abs(ref), (store, t, ref)


@pytest.mark.parametrize("d,N,p,form", [(3, 5, 3, 1), (2, 40, 2, 0), (3, 4, 4, 0)])
def test_negative_control_weight_perturbation(d, N, p, form):
    """A 1e-6 (relative) change of ONE stored weight entry must fail the parity bar; the
    bar is therefore sensitive to single-entry errors in the streamed A_T.  (3, 4, 4, 0):
    FULL WP storage with its rows in orbit order (the symmetry-adapted body), so the hook,
    the export and the kernel must agree on the row permutation."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config("C4" if form == 1 else "C5" if d == 3 else "C1").with_size(N, p)
    coef = c.coefficient()
    m = Mesh(d, N, p)
    op = Operator(m, form, coef)
    ed = oa.build(d, N, p)
    A = oa.assemble_csr(ed, form, coef)
    u = u_vector(ed.ndof, 9)
    ut = torch.from_numpy(u).cuda()
    ref = A @ u

    def err():
        y = op.apply(ut).cpu().numpy()
        return np.abs(y - ref).max() / np.abs(ref).max()

    assert err() <= TOL
    w = op.export_weights()
    e, j = m.info["n_elem_local"] // 2 + 1, w.shape[1] // 2
    delta = 1e-6 * np.abs(w).max()
    op._test_perturb_weight(e, j, 0, delta)
    assert op.export_weights()[e, j, 0] == w[e, j, 0] + delta
    assert err() > 1e3 * TOL
    op._test_perturb_weight(e, j, 0, -delta)
    assert err() <= TOL


@pytest.mark.parametrize("storage,dirichlet", [(0, True), (0, False), (1, True), (1, False)])
def test_ragged_xblocks_3d_el_element_kernel(storage, dirichlet):
    """The C4 recipe at N = 37: two x-blocks per cell row (32 + a ragged 5), the 3D P3 EL
    element kernel with its even/odd-warp pair combine of the shared Kuhn faces, FULL and
    ISO storage, with and without Dirichlet elimination; sampled rows near every face
    (incl. the last valid lane of the ragged block) against the oracle."""
    torch = _torch()
    from paper_1710_09913_b200.api import Mesh, Operator
    c = get_config("C4").with_size(37)
    coef, verts, form = c.coefficient(), c.vertices(), c.forms[0]
    m = Mesh(c.d, c.N, c.p, verts)
    op = Operator(m, form, coef, storage=storage)
    u = c.u()
    y = op.apply(torch.from_numpy(u).cuda(), dirichlet=dirichlet).cpu().numpy()
    M = c.p * c.N + 1
    rng = np.random.default_rng(37 + storage)
    rows = _rows_near_faces(c.d, c.N, c.p, rng)
    # plus the DoFs of the cells at the x-block seam (cells 31 | 32) and of the last cell
    extra = []
    for X in (3 * 31, 3 * 32, 3 * 32 + 1, 3 * 36, 3 * 37 - 1):
        for _ in range(4):
            lat = rng.integers(1, M - 1, 3)
            lat[0] = X
            extra.append(int(lat[0] + M * lat[1] + M * M * lat[2]))
    rows = np.unique(np.concatenate([rows, np.array(extra, dtype=np.int64)]))
    scale = np.abs(y).max()
    if dirichlet:
        lat = np.stack([(rows // M ** a) % M for a in range(3)], axis=1)
        bnd = np.any((lat == 0) | (lat == M - 1), axis=1)
        assert np.array_equal(y[rows[bnd]], u[rows[bnd]])
        rows = rows[~bnd]
        ref = oa.apply_rows_sampled(c.d, c.N, c.p, verts, form, coef, _boundary_zeroed(u, 3, M), rows)
    else:
        ref = oa.apply_rows_sampled(c.d, c.N, c.p, verts, form, coef, u, rows)
    assert np.abs(y[rows] - ref).max() / scale <= TOL
