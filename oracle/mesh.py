"""Structured simplex mesh M_N, P_p DoF map l_T, affine maps (oracle; test infra).

PAPER.md P:518-526 (mesh family M_N, N elements per direction)
(2N^2 triangles / 6N^3 tetrahedra), P:167-170 (affine map F_T = R_T xhat + S_T,
local-to-global map l_T), P:139-147 (continuous space C_{N,k}).

Readings:
  L3 2D: square (i,j) -> (v00,v10,v11), (v00,v11,v01);
     3D Kuhn: for each permutation pi of (x,y,z) in lexicographic order,
     (o, o+e_pi0, o+e_pi0+e_pi1, o+1).  Element e = d!*cell + s,
     cell = i + N j (+ N^2 k).
  L4 vertices and DoFs lexicographic, x fastest: id = i + M j (+ M^2 k),
     M = N+1 (vertices) or pN+1 (DoFs).
  L6 R_T columns v_i - v_0 (signed det), |det R_T| in integrals.
DoF of local multi-index alpha (|alpha| = p) in element (v_0..v_d) sits on the
DoF lattice at sum_i alpha_i * c(v_i), c = integer vertex lattice coordinates.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .reference import multi_indices


def _simplices_of_cell(d: int):
    """Vertex offsets (in {0,1}^d) of the d! simplices of one cell (L3)."""
    if d == 2:
        return [((0, 0), (1, 0), (1, 1)), ((0, 0), (1, 1), (0, 1))]
    out = []
    for perm in itertools.permutations(range(3)):        # lexicographic order
        o = [0, 0, 0]
        verts = [tuple(o)]
        for ax in perm:
            o = list(o)
            o[ax] += 1
            verts.append(tuple(o))
        out.append(tuple(verts))
    return out


@dataclass
class Mesh:
    d: int
    N: int
    vlat: np.ndarray       # (nv, d) integer lattice coordinates of vertices
    X: np.ndarray          # (nv, d) physical coordinates
    elems: np.ndarray      # (ne, d+1) vertex ids
    cell: np.ndarray       # (ne,) cell index of each element

    @property
    def n_elem(self) -> int:
        return self.elems.shape[0]


def structured_mesh(d: int, N: int, vertices: Optional[np.ndarray] = None) -> Mesh:
    """The mesh M_N of the unit square/cube (readings L3, L4).
    ``vertices`` overrides the lattice coordinates (config 5 jitter)."""
    if d not in (2, 3):
        raise ValueError("invalid-dimension")
    if N < 1:
        raise ValueError("invalid-size")
    M = N + 1
    ids = np.arange(M ** d)
    vlat = np.stack([(ids // M ** a) % M for a in range(d)], axis=1)
    X = vlat / N if vertices is None else np.asarray(vertices, dtype=np.float64)
    cells = np.arange(N ** d)
    clat = np.stack([(cells // N ** a) % N for a in range(d)], axis=1)
    simp = _simplices_of_cell(d)
    ns = len(simp)
    elems = np.empty((N ** d * ns, d + 1), dtype=np.int64)
    for s, verts in enumerate(simp):
        for v, off in enumerate(verts):
            c = clat + np.array(off)
            elems[s::ns, v] = sum(c[:, a] * M ** a for a in range(d))
    cell = np.repeat(cells, ns)
    return Mesh(d, N, vlat, X, elems, cell)


def dof_map(mesh: Mesh, p: int, sl: slice = slice(None)) -> np.ndarray:
    """l_T: (ne, V_T) global DoF ids of C_{N,p}; local order of
    reference.multi_indices (L5).  ``sl`` restricts to a range of elements."""
    d, N = mesh.d, mesh.N
    Md = p * N + 1
    A = np.array(multi_indices(d, p))                    # (V_T, d+1)
    cv = mesh.vlat[mesh.elems[sl]]                       # (ne, d+1, d)
    lat = np.einsum("la,eac->elc", A, cv)                # (ne, V_T, d)
    return sum(lat[:, :, a] * Md ** a for a in range(d)).astype(np.int64)


def dof_lattice(d: int, N: int, p: int) -> np.ndarray:
    """Integer lattice coordinates (ndof, d) of every global DoF (L4)."""
    Md = p * N + 1
    ids = np.arange(Md ** d)
    return np.stack([(ids // Md ** a) % Md for a in range(d)], axis=1)


def boundary_mask(d: int, N: int, p: int) -> np.ndarray:
    """DoFs on the boundary of the unit square/cube (reading L14)."""
    lat = dof_lattice(d, N, p)
    return np.any((lat == 0) | (lat == p * N), axis=1)


def affine_maps(mesh: Mesh):
    """R_T (columns x_{v_i} - x_{v_0}), S_T = x_{v_0}, signed det R_T, R_T^{-1}
    (reading L6)."""
    Xe = mesh.X[mesh.elems]                              # (ne, d+1, d)
    S = Xe[:, 0, :]
    R = np.transpose(Xe[:, 1:, :] - S[:, None, :], (0, 2, 1))   # columns
    det = np.linalg.det(R)
    Rinv = np.linalg.inv(R)
    return R, S, det, Rinv


def cell_elements(d: int, N: int, cells: np.ndarray) -> np.ndarray:
    """Vertex ids (n, d+1) of the d! simplices of the given cells, in canonical
    order e = d!*cell + s (same rule as structured_mesh, for sampled rows)."""
    M = N + 1
    cells = np.asarray(cells, dtype=np.int64)
    clat = np.stack([(cells // N ** a) % N for a in range(d)], axis=1)
    simp = _simplices_of_cell(d)
    ns = len(simp)
    elems = np.empty((cells.size * ns, d + 1), dtype=np.int64)
    for s, verts in enumerate(simp):
        for v, off in enumerate(verts):
            c = clat + np.array(off)
            elems[s::ns, v] = sum(c[:, a] * M ** a for a in range(d))
    return elems
