"""Oracle CG pins (reading L15; SPEC S:478-480 examples)."""
import numpy as np

from oracle.cg import CG_BREAKDOWN, CG_CONVERGED, CG_NOT_CONVERGED, cg


def test_identity_one_iteration():
    b = np.array([1.0, -2.0, 3.0])
    x, it, res, st = cg(lambda v: v, b)
    assert st == CG_CONVERGED and it == 1 and np.allclose(x, b)


def test_diag_example():
    D = np.array([2.0, 4.0])
    x, it, res, st = cg(lambda v: D * v, np.array([2.0, 4.0]), rtol=1e-14)
    assert st == CG_CONVERGED and it <= 2
    assert np.allclose(x, [1.0, 1.0], atol=1e-14)


def test_spd_solve_and_maxit():
    rng = np.random.default_rng(0)
    Q = rng.normal(size=(30, 30))
    A = Q @ Q.T + 30 * np.eye(30)
    b = rng.normal(size=30)
    x, it, res, st = cg(lambda v: A @ v, b, rtol=1e-12)
    assert st == CG_CONVERGED and res <= 1e-12
    assert np.linalg.norm(A @ x - b) <= 2e-12 * np.linalg.norm(b)
    _, it2, _, st2 = cg(lambda v: A @ v, b, rtol=1e-12, maxit=2)
    assert st2 == CG_NOT_CONVERGED and it2 == 2


def test_breakdown_on_indefinite():
    A = np.diag([1.0, -1.0])
    _, _, _, st = cg(lambda v: A @ v, np.array([0.0, 1.0]))
    assert st == CG_BREAKDOWN


def test_zero_rhs():
    x, it, res, st = cg(lambda v: 2 * v, np.zeros(4))
    assert it == 0 and st == CG_CONVERGED and not x.any()
