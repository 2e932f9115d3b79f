"""The five benchmark configurations of BASELINE.json ``configs`` (C1-C5).

A config names the mesh (d, N, jitter), the order p, the form(s) and the
coefficient model with its parameters.  Coefficient *evaluation* lives on each
side separately (oracle/coefficients.py and the CUDA weights kernel); only the
parameter values are shared here.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

from . import generators as gen

# coefficient kinds (same integer codes as include/dogip.h DOGIP_COEF_*)
COEF_CONST = 0          # m = params[0] (EL: M = m I)
COEF_PER_CELL = 1       # m = per_cell[cell]         (isotropic, cell-constant)
COEF_SINCOS2D = 2       # m = a0 + a1 sin(2 pi x) cos(2 pi y)
COEF_TANH_RADIAL = 3    # m = a0 + a1 tanh(k (|x - c| - r0))
COEF_ANISO_FOURIER = 4  # M = R(x) diag(eig) R(x)^T, R = Rodrigues(omega(x))
COEF_CONST_TENSOR = 5   # M = constant symmetric d x d matrix (row-major params)

FORM_WP = 0  # weighted projection  (PAPER.md eq:bilf_gp)
FORM_EL = 1  # scalar elliptic      (PAPER.md eq:bilf_se)


@dataclass
class Coefficient:
    kind: int
    params: np.ndarray = field(default_factory=lambda: np.zeros(0))
    per_cell: Optional[np.ndarray] = None

    @property
    def isotropic(self) -> bool:
        return self.kind in (COEF_CONST, COEF_PER_CELL, COEF_SINCOS2D,
                             COEF_TANH_RADIAL)


def aniso_fourier_params(seed: int = 2) -> np.ndarray:
    """Flat parameter vector [eig(3), n_modes, kappa(n*3), phi(n*3), c(n*3)]."""
    r = gen.rotation_field_params(seed)
    n = r["kappa"].shape[0]
    return np.concatenate([r["eig"], [float(n)], r["kappa"].ravel(),
                           r["phi"].ravel(), r["c"].ravel()])


@dataclass
class Config:
    name: str
    d: int
    N: int
    p: int
    forms: Tuple[int, ...]
    coef_name: str
    jitter_seed: Optional[int] = None
    u_seed: int = 0
    description: str = ""

    @property
    def n_elem(self) -> int:
        return (2 if self.d == 2 else 6) * self.N ** self.d

    @property
    def ndof(self) -> int:
        return (self.p * self.N + 1) ** self.d

    def vertices(self) -> Optional[np.ndarray]:
        """Vertex coordinates ((N+1)^d, d), or None for the plain lattice."""
        if self.jitter_seed is None:
            return None
        M = self.N + 1
        ids = np.arange(M ** self.d)
        X = np.stack([(ids // M ** a) % M for a in range(self.d)], axis=1)
        return X / self.N + gen.vertex_jitter(self.d, self.N, 0.2, self.jitter_seed)

    def coefficient(self) -> Coefficient:
        c = self.coef_name
        if c == "sincos2d":
            return Coefficient(COEF_SINCOS2D, np.array([1.0, 0.5]))
        if c.startswith("grf"):
            seed = int(c[3:])
            return Coefficient(COEF_PER_CELL, np.zeros(0),
                               gen.grf_per_cell(self.d, self.N, 0.05, 1.0, seed))
        if c == "aniso2":
            return Coefficient(COEF_ANISO_FOURIER, aniso_fourier_params(2))
        if c == "tanh":
            return Coefficient(COEF_TANH_RADIAL,
                               np.array([1.0, 0.9, 20.0, 0.25, 0.5, 0.5, 0.5]))
        if c == "one":
            return Coefficient(COEF_CONST, np.array([1.0]))
        raise ValueError(c)

    def u(self) -> np.ndarray:
        return gen.u_vector(self.ndof, self.u_seed)

    def with_size(self, N: int, p: Optional[int] = None) -> "Config":
        """Same recipe on a smaller mesh (parity tests at oracle-friendly sizes)."""
        return Config(self.name + f"@N{N}", self.d, N, self.p if p is None else p,
                      self.forms, self.coef_name, self.jitter_seed, self.u_seed,
                      self.description)


CONFIGS = {
    "C1": Config("C1", 2, 16, 2, (FORM_WP, FORM_EL), "sincos2d",
                 description="2D 16x16x2 P2, WP a=1+0.5sin(2pi x)cos(2pi y) and EL a*I"),
    "C2p1": Config("C2p1", 2, 1024, 1, (FORM_EL,), "grf1", description="2D 1024^2x2 P1 EL, exp(GRF)"),
    "C2p2": Config("C2p2", 2, 1024, 2, (FORM_EL,), "grf1", description="2D 1024^2x2 P2 EL, exp(GRF)"),
    "C2p3": Config("C2p3", 2, 1024, 3, (FORM_EL,), "grf1", description="2D 1024^2x2 P3 EL, exp(GRF)"),
    "C2p4": Config("C2p4", 2, 1024, 4, (FORM_EL,), "grf1", description="2D 1024^2x2 P4 EL, exp(GRF)"),
    "C3": Config("C3", 3, 64, 2, (FORM_EL,), "aniso2",
                 description="3D 64^3x6 P2 EL, R(x)diag(1,10,100)R(x)^T"),
    "C4": Config("C4", 3, 128, 3, (FORM_EL,), "grf3",
                 description="3D 128^3x6 P3 EL, isotropic exp(GRF) per cell"),
    "C5": Config("C5", 3, 96, 4, (FORM_WP,), "tanh", jitter_seed=4,
                 description="3D 96^3x6 jittered P4 WP, 1+0.9tanh(20(|x-c|-0.25))"),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]
