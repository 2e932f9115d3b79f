"""Seeded random inputs (readings L19-L23).

Every function here only draws random numbers with ``numpy.random.default_rng``
and reshapes them; none evaluates basis functions, integrals or operators.
The vertex / cell numbering convention (x fastest, z slowest; L4) is
an input-layout convention shared by both sides.
"""
from __future__ import annotations

import numpy as np


def u_vector(ndof: int, seed: int = 0) -> np.ndarray:
    """Input nodal vector u ~ U[-1, 1]^ndof (BASELINE.json config 1 "i.i.d.
    uniform[-1,1] nodal values, seed 0"; reading L23 uses it for every config)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, int(ndof))


def grf_per_cell(d: int, N: int, ell: float = 0.05, sigma: float = 1.0,
                 seed: int = 1) -> np.ndarray:
    """Log-normal per-cell coefficient exp(g), g a stationary Gaussian random
    field with covariance sigma^2 exp(-|r|^2 / (2 ell^2)) (BASELINE.json
    configs 2 and 4), sampled by circulant embedding on the periodic (2N)^d
    grid of cell centres (reading L19).

    Returns an array of N^d values indexed cell = i + N*j (+ N^2*k).
    """
    M = 2 * N
    h = 1.0 / N
    idx = np.arange(M)
    dist1 = np.minimum(idx, M - idx) * h           # periodic distance per axis
    grids = np.meshgrid(*([dist1] * d), indexing="ij")
    r2 = sum(g * g for g in grids)
    c = sigma * sigma * np.exp(-r2 / (2.0 * ell * ell))
    lam = np.maximum(np.real(np.fft.fftn(c)), 0.0)
    rng = np.random.default_rng(seed)
    z1 = rng.standard_normal((M,) * d)
    z2 = rng.standard_normal((M,) * d)
    xi = z1 + 1j * z2
    g = np.real(np.fft.fftn(np.sqrt(lam / M ** d) * xi))
    g = g[(slice(0, N),) * d]                      # axes (x, y[, z])
    return np.exp(g).reshape(-1, order="F").copy()  # cell = i + N j + N^2 k


def rotation_field_params(seed: int = 2, n_modes: int = 8) -> dict:
    """Parameters of the smooth rotation field of config 3 (reading L20):
    axis-angle omega(x)_i = sum_m c[m,i] cos(2 pi kappa[m].x + phi[m,i]).

    Draw order: kappa (integers in [-2,2], zero rows redrawn), phi, c."""
    rng = np.random.default_rng(seed)
    kappa = rng.integers(-2, 3, (n_modes, 3))
    while True:
        zero = np.all(kappa == 0, axis=1)
        if not zero.any():
            break
        kappa[zero] = rng.integers(-2, 3, (int(zero.sum()), 3))
    phi = rng.uniform(0.0, 2.0 * np.pi, (n_modes, 3))
    c = rng.normal(0.0, 1.0, (n_modes, 3)) * (np.pi / 2.0) / np.sqrt(n_modes)
    return {"kappa": kappa.astype(np.float64), "phi": phi, "c": c,
            "eig": np.array([1.0, 10.0, 100.0])}


def vertex_jitter(d: int, N: int, amp: float = 0.2, seed: int = 4) -> np.ndarray:
    """Vertex displacement of config 5 (reading L21): uniform in
    [-amp*h, amp*h]^d per vertex, zero on boundary vertices.

    Returns ((N+1)^d, d) in vertex order id = i + (N+1) j (+ (N+1)^2 k)."""
    h = 1.0 / N
    M = N + 1
    J = np.random.default_rng(seed).uniform(-amp * h, amp * h, (M ** d, d))
    ids = np.arange(M ** d)
    on_bnd = np.zeros(M ** d, dtype=bool)
    for a in range(d):
        ia = (ids // M ** a) % M
        on_bnd |= (ia == 0) | (ia == N)
    J[on_bnd] = 0.0
    return J
