"""Standard FEM assembly / application of the system matrix A (oracle; test infra).

This is the DEFINITION the DoGIP apply must reproduce:
  WP  A_ij = int m phi_j phi_i          (eq:linsys_gp)
  EL  A_ij = int M grad phi_j . grad phi_i  (eq:linsys_se)
evaluated element by element with the contract rule Q (reading L10):
  WP  K_T,ij = |det R_T| sum_q w_q m(F_T xq) phi_i(xq) phi_j(xq)
  EL  K_T,ij = |det R_T| sum_q w_q (R_T^-T grad phi_i)^T M(F_T xq) (R_T^-T grad phi_j)
(chain rule eq:bas_deriv), A = sum_T P_T^T K_T P_T.
Never uses double-grid weights.

Routes: CSR (scipy.sparse) for small meshes; element route (y = sum_T
P_T^T K_T P_T u, the "alternative approaches" form of P:66-75) for big meshes;
quadrature-point route (interpolate u_T to the rule's points, scale by the
coefficient and |det R_T| w_q, project back: the same sum without forming K_T,
P:61-75) for the full-size C3 / C5 residual checks; ``apply_rows`` /
``apply_rows_sampled`` compute selected entries of A u one by one for
full-size sampled parity.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import coefficients as coefs
from .mesh import Mesh, affine_maps, boundary_mask, dof_map, dof_lattice, structured_mesh
from .quadrature import contract_n1d, simplex_rule
from .reference import eval_basis, eval_grad

FORM_WP, FORM_EL = 0, 1


class ElementData:
    """Per-mesh precomputation shared by the routes (geometry, l_T, tables)."""

    def __init__(self, mesh: Mesh, p: int, n1d: int | None = None):
        self.mesh, self.p, self.d = mesh, p, mesh.d
        self.R, self.S, self.det, self.Rinv = affine_maps(mesh)
        self._lT = None
        self.qp, self.qw = simplex_rule(mesh.d, n1d or contract_n1d(p))
        self.Phi = eval_basis(mesh.d, p, self.qp)          # (nq, V_T)
        self.dPhi = eval_grad(mesh.d, p, self.qp)          # (nq, V_T, d)
        self.ndof = (p * mesh.N + 1) ** mesh.d

    @property
    def lT(self) -> np.ndarray:
        """l_T of every element (computed on first use; full-size routes use lT_of)."""
        if self._lT is None:
            self._lT = dof_map(self.mesh, self.p)
        return self._lT

    def lT_of(self, sl: slice) -> np.ndarray:
        return self._lT[sl] if self._lT is not None else dof_map(self.mesh, self.p, sl)

    def element_matrices(self, form: int, coef, sl: slice) -> np.ndarray:
        """K_T for elements in ``sl`` -> (nb, V_T, V_T)."""
        d = self.d
        R, S, det, Rinv = self.R[sl], self.S[sl], self.det[sl], self.Rinv[sl]
        nb, nq = R.shape[0], self.qp.shape[0]
        x = np.einsum("eij,qj->eqi", R, self.qp) + S[:, None, :]      # F_T(xq)
        cell = np.repeat(self.mesh.cell[sl], nq)
        c = coefs.evaluate(coef, d, x.reshape(-1, d), cell)
        scale = np.abs(det)[:, None] * self.qw[None, :]               # (nb, nq)
        if form == FORM_WP:
            if c.ndim != 1:
                raise ValueError("WP needs a scalar coefficient")
            wq = scale * c.reshape(nb, nq)
            return np.einsum("eq,qi,qj->eij", wq, self.Phi, self.Phi)
        Mq = coefs.as_tensor(c, d).reshape(nb, nq, d, d)
        # physical gradients: grad phi = R^-T grad_hat phi  (eq:bas_deriv)
        G = np.einsum("epr,qlp->eqlr", Rinv, self.dPhi)               # (nb,nq,V_T,d)
        MG = np.einsum("eqrs,eqls->eqlr", Mq, G)
        return np.einsum("eq,eqir,eqjr->eij", scale, G, MG)

    def chunks(self, chunk: int = 16384):
        ne = self.mesh.n_elem
        for s in range(0, ne, chunk):
            yield slice(s, min(ne, s + chunk))


def assemble_csr(ed: ElementData, form: int, coef) -> sp.csr_matrix:
    """A = sum_T P_T^T K_T P_T as a CSR matrix."""
    rows, cols, vals = [], [], []
    for sl in ed.chunks():
        K = ed.element_matrices(form, coef, sl)
        l = ed.lT[sl]
        rows.append(np.repeat(l, l.shape[1], axis=1).ravel())
        cols.append(np.tile(l, (1, l.shape[1])).ravel())
        vals.append(K.ravel())
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(ed.ndof, ed.ndof))
    return A.tocsr()


def apply_elementwise(ed: ElementData, form: int, coef, u: np.ndarray,
                      dirichlet: bool = False) -> np.ndarray:
    """y = sum_T P_T^T K_T P_T u without forming A; with
    ``dirichlet`` the symmetric-elimination operator of ``dirichlet_apply``."""
    mask = boundary_mask(ed.d, ed.mesh.N, ed.p) if dirichlet else None
    uu = np.where(mask, 0.0, u) if dirichlet else u
    y = np.zeros(ed.ndof)
    for sl in ed.chunks():
        K = ed.element_matrices(form, coef, sl)
        l = ed.lT[sl]
        yl = np.einsum("eij,ej->ei", K, uu[l])
        y += np.bincount(l.ravel(), weights=yl.ravel(), minlength=ed.ndof)
    if dirichlet:
        y[mask] = u[mask]
    return y


def elements_containing(ed: ElementData, dof: int) -> np.ndarray:
    """Elements whose closure contains global DoF ``dof`` (structured search)."""
    d, N, p = ed.d, ed.mesh.N, ed.p
    lat = dof_lattice(d, N, p)[dof]
    cand_axes = []
    for a in range(d):
        X = int(lat[a])
        cs = {X // p, (X - 1) // p} if X % p == 0 else {X // p}
        cand_axes.append([c for c in cs if 0 <= c < N])
    ns = 2 if d == 2 else 6
    out = []
    for cc in np.array(np.meshgrid(*cand_axes, indexing="ij")).reshape(d, -1).T:
        cell = int(sum(int(cc[a]) * N ** a for a in range(d)))
        for s in range(ns):
            e = ns * cell + s
            if dof in ed.lT[e]:
                out.append(e)
    return np.array(out, dtype=np.int64)


def apply_rows(ed: ElementData, form: int, coef, u: np.ndarray, rows) -> np.ndarray:
    """(A u)_i for the given rows only: sum over T containing i of (K_T u_T)_i."""
    out = np.empty(len(rows))
    for n, i in enumerate(rows):
        els = elements_containing(ed, int(i))
        acc = 0.0
        for e in els:
            K = ed.element_matrices(form, coef, slice(e, e + 1))[0]
            li = int(np.nonzero(ed.lT[e] == i)[0][0])
            acc += K[li] @ u[ed.lT[e]]
        out[n] = acc
    return out


def load_vector(ed: ElementData, f: float = 1.0, dirichlet: bool = False) -> np.ndarray:
    """b_i = int f phi_i (eq:linsys_gp P:207, eq:linsys_se P:337), f constant;
    zeroed on boundary DoFs when ``dirichlet`` (reading L14)."""
    s = ed.Phi.T @ ed.qw                                  # int_ref phi_i
    be = f * np.abs(ed.det)[:, None] * s[None, :]
    b = np.bincount(ed.lT.ravel(), weights=be.ravel(), minlength=ed.ndof)
    if dirichlet:
        b[boundary_mask(ed.d, ed.mesh.N, ed.p)] = 0.0
    return b


def load_vector_fn(ed: ElementData, f) -> np.ndarray:
    """b_i = int f phi_i for a callable f(x) (x: (n, d) physical points), by the
    contract rule (eq:linsys_gp P:207).  Used by the polynomial-reproduction pins."""
    d = ed.d
    b = np.zeros(ed.ndof)
    for sl in ed.chunks():
        R, S, det = ed.R[sl], ed.S[sl], ed.det[sl]
        x = np.einsum("eij,qj->eqi", R, ed.qp) + S[:, None, :]
        fx = f(x.reshape(-1, d)).reshape(x.shape[0], -1)
        be = np.einsum("eq,q,qi->ei", fx * np.abs(det)[:, None], ed.qw, ed.Phi)
        b += np.bincount(ed.lT[sl].ravel(), weights=be.ravel(), minlength=ed.ndof)
    return b


def dirichlet_matrix(A: sp.csr_matrix, mask: np.ndarray) -> sp.csr_matrix:
    """Symmetric elimination (reading L14): rows/cols of boundary DoFs replaced
    by the identity, A_D = D A D + (I - D), D = diag(interior)."""
    D = sp.diags((~mask).astype(np.float64))
    return (D @ A @ D + sp.diags(mask.astype(np.float64))).tocsr()


def build(d: int, N: int, p: int, vertices=None, n1d=None) -> ElementData:
    return ElementData(structured_mesh(d, N, vertices), p, n1d)


def apply_rows_sampled(d: int, N: int, p: int, vertices, form: int, coef, u: np.ndarray,
                       rows, n1d=None) -> np.ndarray:
    """(A u)_i for sampled rows of a FULL-SIZE mesh without building it: for
    each row, only the cells around its DoF are instantiated (same mesh rule,
    same element matrices as ElementData)."""
    from .mesh import Mesh, cell_elements
    Md = p * N + 1
    out = np.empty(len(rows))
    M = N + 1
    for n, i in enumerate(rows):
        i = int(i)
        lat = [(i // Md ** a) % Md for a in range(d)]
        axes = []
        for a in range(d):
            X = lat[a]
            cs = {X // p, (X - 1) // p} if X % p == 0 else {X // p}
            axes.append([c for c in cs if 0 <= c < N])
        cells = np.array([sum(int(cc[a]) * N ** a for a in range(d))
                          for cc in np.array(np.meshgrid(*axes, indexing="ij")).reshape(d, -1).T])
        elems = cell_elements(d, N, cells)
        vids = np.unique(elems)
        vlat = np.stack([(vids // M ** a) % M for a in range(d)], axis=1)
        X = vlat / N if vertices is None else np.asarray(vertices)[vids]
        remap = {int(v): k for k, v in enumerate(vids)}
        loc = np.vectorize(remap.get)(elems)
        sub = Mesh(d, N, vlat, X, loc, np.repeat(cells, 2 if d == 2 else 6))
        ed = ElementData(sub, p, n1d)
        # global DoF ids: dof_map used lattice coords of the local vertices -> still global
        ed.ndof = Md ** d
        K = ed.element_matrices(form, coef, slice(0, sub.n_elem))
        acc = 0.0
        for e in range(sub.n_elem):
            hit = np.nonzero(ed.lT[e] == i)[0]
            if hit.size:
                acc += K[e, hit[0]] @ u[ed.lT[e]]
        out[n] = acc
    return out


def _qp_chunk(ed: ElementData, form: int, coef, uu: np.ndarray, sl: slice):
    """One chunk of the quadrature-point route: (l_T, y_T) of the elements in sl."""
    d = ed.d
    R, S, det, Rinv = ed.R[sl], ed.S[sl], ed.det[sl], ed.Rinv[sl]
    nb, nq = R.shape[0], ed.qp.shape[0]
    l = ed.lT_of(sl)
    uT = uu[l]                                                     # P_T u   (nb, V_T)
    x = np.einsum("eij,qj->eqi", R, ed.qp) + S[:, None, :]         # F_T(xq)
    c = coefs.evaluate(coef, d, x.reshape(-1, d), np.repeat(ed.mesh.cell[sl], nq))
    scale = np.abs(det)[:, None] * ed.qw[None, :]                  # |det R_T| w_q
    if form == FORM_WP:
        if c.ndim != 1:
            raise ValueError("WP needs a scalar coefficient")
        uq = uT @ ed.Phi.T                                         # u_h(xq)        (nb, nq)
        yT = (scale * c.reshape(nb, nq) * uq) @ ed.Phi             # sum_q w m u phi_i
        return l, yT
    Mq = coefs.as_tensor(c, d).reshape(nb, nq, d, d)
    VT = uT.shape[1]
    gref = (uT @ ed.dPhi.transpose(1, 0, 2).reshape(VT, nq * d)).reshape(nb, nq, d)  # reference gradient
    g = np.einsum("epr,eqp->eqr", Rinv, gref)                      # R^-T grad_hat  (eq:bas_deriv)
    flux = scale[:, :, None] * np.einsum("eqrs,eqs->eqr", Mq, g)   # |det| w_q M grad u
    t = np.einsum("epr,eqr->eqp", Rinv, flux)                      # R^-1 flux
    yT = t.reshape(nb, nq * d) @ ed.dPhi.transpose(0, 2, 1).reshape(nq * d, VT)  # sum_q grad_hat phi_l . (R^-1 flux)
    return l, yT


def _blas_single_threaded():
    """Context in which BLAS runs one thread per call.  Threaded chunk evaluation
    (workers > 1) must not call a multithreaded OpenBLAS concurrently from several Python
    threads: that returns corrupted products (observed with NumPy's bundled OpenBLAS 0.3.30
    on the 8192-element chunks: 2 of 3 full-size runs wrong by up to 10 %)."""
    from threadpoolctl import threadpool_limits
    return threadpool_limits(limits=1, user_api="blas")


def apply_qp_route(ed: ElementData, form: int, coef, u: np.ndarray, dirichlet: bool = False,
                   workers: int = 1, chunk: int = 8192) -> np.ndarray:
    """y = A u by the quadrature-point route: for every element,
    u_T -> values / physical gradients at the contract rule's points -> times
    |det R_T| w_q m (WP) or |det R_T| w_q M (EL) -> tested against phi_i /
    grad phi_i, summed into y.  Algebraically sum_T P_T^T K_T P_T u with the K_T
    of element_matrices (same rule); no K_T and no global matrix are formed, so it
    runs at the full C3 / C5 sizes.  ``workers`` > 1 evaluates chunks in threads
    (NumPy releases the GIL in its kernels); the sum into y stays sequential."""
    mask = boundary_mask(ed.d, ed.mesh.N, ed.p) if dirichlet else None
    uu = np.where(mask, 0.0, u) if dirichlet else u
    y = np.zeros(ed.ndof)
    sls = list(ed.chunks(chunk))
    if workers <= 1:
        parts = (_qp_chunk(ed, form, coef, uu, sl) for sl in sls)
        for l, yT in parts:
            y += np.bincount(l.ravel(), weights=yT.ravel(), minlength=ed.ndof)
    else:
        from concurrent.futures import ThreadPoolExecutor
        with _blas_single_threaded(), ThreadPoolExecutor(workers) as ex:
            for l, yT in ex.map(lambda sl: _qp_chunk(ed, form, coef, uu, sl), sls):
                y += np.bincount(l.ravel(), weights=yT.ravel(), minlength=ed.ndof)
    if dirichlet:
        y[mask] = u[mask]
    return y


def wp_total(ed: ElementData, coef, workers: int = 1, chunk: int = 16384) -> float:
    """1^T A 1 of the weighted projection = sum_T |det R_T| sum_q w_q m(F_T xq)
    (sum_i phi_i = 1, so sum_ij K_T,ij is the rule's integral of m over T; equally
    sum_T sum_j a_{T,j} of Theorem 2's weights, since sum_j phi^W_j = 1)."""
    d, nq = ed.d, ed.qp.shape[0]

    def part(sl):
        R, S, det = ed.R[sl], ed.S[sl], ed.det[sl]
        x = np.einsum("eij,qj->eqi", R, ed.qp) + S[:, None, :]
        c = coefs.evaluate(coef, d, x.reshape(-1, d), np.repeat(ed.mesh.cell[sl], nq))
        return float((np.abs(det)[:, None] * ed.qw[None, :] * c.reshape(-1, nq)).sum())

    sls = list(ed.chunks(chunk))
    if workers <= 1:
        return sum(part(sl) for sl in sls)
    from concurrent.futures import ThreadPoolExecutor
    with _blas_single_threaded(), ThreadPoolExecutor(workers) as ex:
        return sum(ex.map(part, sls))
