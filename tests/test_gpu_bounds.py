"""Out-of-bounds guard bands around every device buffer the library reads or writes
(the stand-in for compute-sanitizer memcheck, which this pool does not allow; SURVEY §4
T2).  For every (d, p, form, storage, coefficient path) on meshes with several tiles and
a ragged last tile:

* u, b sit inside NaN guard bands: a read past either end would turn y / x non-finite;
* y, x sit inside sentinel guard bands: a write past either end changes the sentinel;
* the same for the host-buffer apply (numpy arrays with guards).

Exercises weights (quadrature + DMMA GEMM + finalize, and the cell-constant direct path),
apply (plain, Dirichlet, host pipelined), load vector and CG (CUDA graph, host loop,
fixed count).  Values are checked by tests/test_gpu_parity.py; this checks only bounds.
"""
import os

import numpy as np
import pytest

from synth.configs import COEF_CONST, get_config

G = 4096          # guard elements on each side (32 KB)
SENT = 12345.0

STORES = {0: (0, 2, 4, 5), 1: (0, 1, 4)}      # DOGIP_STORE_* per form (WP, EL)


def _cases():
    out = []
    for p in (1, 2, 3, 4):
        out.append(("C1", 2, 34, p))             # 2D, sincos coefficient (quadrature path)
        out.append(("C4", 3, 3, p))              # 3D, per-cell coefficient (direct path)
    out.append(("C5", 3, 3, 4))                  # jittered, tanh coefficient
    out.append(("C3", 3, 3, 2))                  # anisotropic EL coefficient
    return out


def _guarded(torch, n, fill, inner=None):
    big = torch.full((n + 2 * G,), fill, dtype=torch.float64, device="cuda")
    if inner is not None:
        big[G:G + n] = inner
    return big, big[G:G + n]


@pytest.mark.gpu
@pytest.mark.parametrize("base,d,N,p", _cases())
def test_guard_bands(base, d, N, p):
    import torch

    from paper_1710_09913_b200.api import CoeffSpec, Mesh, Operator

    c = get_config(base).with_size(N, p)
    mesh = Mesh(d, N, p, vertices=c.vertices(), device=0)
    n = mesh.ndof
    u_np = c.u()
    u_big, u = _guarded(torch, n, float("nan"), torch.from_numpy(u_np).cuda())
    forms = (0, 1) if base == "C1" else c.forms
    ran = 0
    for form in forms:
        for coef in (c.coefficient(), CoeffSpec(COEF_CONST, np.array([1.5]))):
            for store in STORES[form]:
                try:
                    op = Operator(mesh, form, coef, storage=store)
                except RuntimeError as e:              # storage not defined for (d, p, form, coefficient)
                    assert any(k in str(e) for k in ("UNSUPPORTED", "INVALID", "BAD_COEFF")), e
                    continue
                tag = f"form={form} store={store} coef={coef.kind}"
                dir_ok = True
                y_big, y = _guarded(torch, n, SENT)
                for dirichlet in (False, True) if dir_ok else (False,):
                    op.apply(u, y, dirichlet=dirichlet)
                    torch.cuda.synchronize()
                    assert torch.isfinite(y).all(), tag
                    assert (y_big[:G] == SENT).all() and (y_big[-G:] == SENT).all(), tag
                if store != 4:
                    hu = np.full(n + 2 * G, np.nan)
                    hu[G:G + n] = u_np
                    hy = np.full(n + 2 * G, SENT)
                    op.apply_host(hu[G:G + n], hy[G:G + n], dirichlet=dir_ok)
                    assert np.isfinite(hy[G:G + n]).all(), tag
                    assert (hy[:G] == SENT).all() and (hy[-G:] == SENT).all(), tag
                b_big, b = _guarded(torch, n, float("nan"))
                op.load_vector(1.0, dirichlet=dir_ok, out=b)
                x_big, x = _guarded(torch, n, SENT, 0.0)
                op.cg(b, x, rtol=1e-8, maxit=5, dirichlet=dir_ok)        # CUDA-graph CG
                os.environ["DOGIP_CG_NO_GRAPH"] = "1"
                try:
                    op.cg(b, x, rtol=1e-8, maxit=5, dirichlet=dir_ok)    # host loop
                finally:
                    del os.environ["DOGIP_CG_NO_GRAPH"]
                op.cg(b, x, rtol=1e-8, maxit=-3, dirichlet=dir_ok)       # fixed count
                torch.cuda.synchronize()
                assert torch.isfinite(b).all() and torch.isfinite(x).all(), tag
                assert (b_big[:G].isnan()).all() and (b_big[-G:].isnan()).all(), tag
                assert (x_big[:G] == SENT).all() and (x_big[-G:] == SENT).all(), tag
                op.close()
                ran += 1
    mesh.close()
    assert ran > 0
