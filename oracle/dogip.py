"""The paper's DoGIP decomposition, written out plainly (oracle; test infra).

Used ONLY for (a) parity of the CUDA weights kernel (the weights are an
intermediate of the hot path) and (b) check (iv): brute-force equality of
C^T A^DoGIP B with the assembled A on tiny meshes.  The apply parity itself
compares against oracle.assemble (standard FEM), never against this module.

  WP element weights  A_T,jj = int_T m phi^W_j         (Theorem 2)
  EL element weights  A_T,rs,jj = sum_pq Rinv_rp Rinv_sq int_T M_pq phi^W_j
                                                       (Theorem 4)
  WP global weights   A_ii = int_Omega m phi^W_i       (Theorem 1)
  Algorithm 1         v = 0; for T: v[l_T] += Bhat^T A_T Bhat u[l_T]
                                                       (reading L8)
The integrals use the contract rule Q (reading L10).  W = P_2p (WP) or
P_{2p-2} discontinuous (EL, reading L7).
"""
from __future__ import annotations

import numpy as np

from . import coefficients as coefs
from .assemble import FORM_EL, FORM_WP, ElementData
from .mesh import dof_map
from .reference import bhat_el, bhat_wp, eval_basis


def w_order(p: int, form: int) -> int:
    return 2 * p if form == FORM_WP else 2 * p - 2


def element_weights(ed: ElementData, form: int, coef) -> np.ndarray:
    """WP: (ne, W_T);  EL: (ne, W_T, d, d) -- P:281 / P:443."""
    d = ed.d
    PhiW = eval_basis(d, w_order(ed.p, form), ed.qp)          # (nq, W_T)
    out = []
    for sl in ed.chunks():
        R, S, det, Rinv = ed.R[sl], ed.S[sl], ed.det[sl], ed.Rinv[sl]
        nb, nq = R.shape[0], ed.qp.shape[0]
        x = np.einsum("eij,qj->eqi", R, ed.qp) + S[:, None, :]
        c = coefs.evaluate(coef, d, x.reshape(-1, d), np.repeat(ed.mesh.cell[sl], nq))
        scale = np.abs(det)[:, None] * ed.qw[None, :]
        if form == FORM_WP:
            out.append(np.einsum("eq,eq,qj->ej", scale, c.reshape(nb, nq), PhiW))
        else:
            Mq = coefs.as_tensor(c, d).reshape(nb, nq, d, d)
            Abar = np.einsum("eq,eqpr,qj->ejpr", scale, Mq, PhiW)   # int_T M phi^W_j
            out.append(np.einsum("erp,ejpq,esq->ejrs", Rinv, Abar, Rinv))
    return np.concatenate(out, axis=0)


def algorithm1(ed: ElementData, form: int, weights: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Algorithm 1 as a literal element loop: small meshes only."""
    d = ed.d
    B = bhat_wp(d, ed.p) if form == FORM_WP else bhat_el(d, ed.p)
    v = np.zeros_like(u)                                     # "allocate v"
    for T in range(ed.mesh.n_elem):
        uT = u[ed.lT[T]]
        if form == FORM_WP:
            g = B @ uT                                       # Bhat u_T
            h = weights[T] * g                               # A_T (diagonal)
            yT = B.T @ h                                     # Bhat^T (L8)
        else:
            g = np.einsum("sjl,l->js", B, uT)                # reference gradients
            h = np.einsum("jrs,js->jr", weights[T], g)       # A_T blocks
            yT = np.einsum("rjk,jr->k", B, h)
        v[ed.lT[T]] += yT
    return v


def dense_elementwise_operator(ed: ElementData, form: int, weights: np.ndarray) -> np.ndarray:
    """Check (iv): dense global B (rows = (T, j[, r])) and block-diagonal
    A^DoGIP, returning C^T A^DoGIP B with C = B."""
    d, ne = ed.d, ed.mesh.n_elem
    if form == FORM_WP:
        Bh = bhat_wp(d, ed.p)
        WT = Bh.shape[0]
        B = np.zeros((ne * WT, ed.ndof))
        for T in range(ne):
            for j in range(WT):
                np.add.at(B[T * WT + j], ed.lT[T], Bh[j])
        Ad = np.diag(weights.reshape(-1))
        return B.T @ Ad @ B
    Bh = bhat_el(d, ed.p)
    WT = Bh.shape[1]
    B = np.zeros((ne * WT * d, ed.ndof))
    Ad = np.zeros((ne * WT * d, ne * WT * d))
    for T in range(ne):
        for j in range(WT):
            base = (T * WT + j) * d
            for r in range(d):
                np.add.at(B[base + r], ed.lT[T], Bh[r, j])
            Ad[base:base + d, base:base + d] = weights[T, j]
    return B.T @ Ad @ B


def global_wp_operator(ed: ElementData, coef) -> np.ndarray:
    """Theorem 1: global diagonal over W = C_{N,2p} and global
    B_ij = phi^j_V(x^i_W); returns the dense B^T A^DoGIP B."""
    d, p = ed.d, ed.p
    a_el = element_weights(ed, FORM_WP, coef)
    lW = dof_map(ed.mesh, 2 * p)
    nW = (2 * p * ed.mesh.N + 1) ** d
    a = np.bincount(lW.ravel(), weights=a_el.ravel(), minlength=nW)   # int_Omega m phi^W_i
    Bh = bhat_wp(d, p)
    B = np.zeros((nW, ed.ndof))
    for T in range(ed.mesh.n_elem):
        for j in range(Bh.shape[0]):
            B[lW[T, j], ed.lT[T]] = Bh[j]        # same value from every element
    return B.T @ (a[:, None] * B)
