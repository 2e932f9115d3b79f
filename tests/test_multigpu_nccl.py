"""The multi-GPU path over NCCL (one process per GPU), against the CPU oracle.

Skipped when fewer than 2 GPUs are visible (the development pool has one; the 1-GPU
coverage of the same code is tests/test_multirank_loopback.py and the 1-rank NCCL
communicator test).  Two ranks, z-slabs, every collective call made by both:
apply (with and without Dirichlet elimination), load vector, CG to 1e-10 and a
fixed 6-iteration CG, compared with the oracle to 1e-12 / 1e-8, and the interface
planes bitwise equal on both owners.
"""
import os
import tempfile

import numpy as np
import pytest

from oracle import assemble as oa
from oracle.cg import cg as oracle_cg
from oracle.mesh import boundary_mask
from synth.configs import COEF_PER_CELL, Coefficient
from synth.generators import grf_per_cell, u_vector

pytestmark = pytest.mark.gpu
NR = 2
CASES = [(3, 8, 3, 1), (3, 6, 4, 0), (2, 64, 2, 1)]


def _n_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _coef(d, N):
    return Coefficient(COEF_PER_CELL, np.zeros(0), grf_per_cell(d, N, 0.2, 1.0, 3))


def _rank_main(rank, nccl_id, d, N, p, form, outdir):
    import torch
    from paper_1710_09913_b200.api import Mesh, Operator
    torch.cuda.set_device(rank)
    m = Mesh(d, N, p, rank=rank, nranks=NR, nccl_id=nccl_id, device=rank)
    op = Operator(m, form, _coef(d, N))
    i0 = m.info["dof_offset"]
    u = u_vector((p * N + 1) ** d, 8)
    ul = torch.from_numpy(u[i0:i0 + m.ndof].copy()).cuda()
    dirichlet = form == 1
    y = op.apply(ul)
    yd = op.apply(ul, dirichlet=True)
    b = op.load_vector(1.0, dirichlet=dirichlet)
    x = torch.zeros_like(b)
    res = op.cg(b, x, rtol=1e-10, maxit=5000, dirichlet=dirichlet)
    x6 = torch.zeros_like(b)
    op.cg(b, x6, maxit=-6, dirichlet=dirichlet)
    torch.cuda.synchronize()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), i0=i0, y=y.cpu().numpy(), yd=yd.cpu().numpy(),
             b=b.cpu().numpy(), x=x.cpu().numpy(), x6=x6.cpu().numpy(), iters=res["iters"],
             ok=res["status"] == "OK")
    op.close()
    m.close()


@pytest.mark.skipif(_n_gpus() < NR, reason="needs >= 2 GPUs (one NCCL rank per GPU)")
@pytest.mark.parametrize("d,N,p,form", CASES)
def test_two_gpu_nccl_matches_oracle(d, N, p, form):
    import torch.multiprocessing as mp
    from paper_1710_09913_b200.api import nccl_unique_id
    nid = nccl_unique_id()
    with tempfile.TemporaryDirectory() as td:
        mp.start_processes(_rank_main, args=(nid, d, N, p, form, td), nprocs=NR, join=True, start_method="spawn")
        out = [dict(np.load(os.path.join(td, f"r{r}.npz"))) for r in range(NR)]
    ed = oa.build(d, N, p)
    coef = _coef(d, N)
    A = oa.assemble_csr(ed, form, coef)
    AD = oa.dirichlet_matrix(A, boundary_mask(d, N, p))
    u = u_vector(ed.ndof, 8)
    b_ref = oa.load_vector(ed, 1.0, dirichlet=form == 1)
    Acg = AD if form == 1 else A
    x_ref, it_ref, _, _ = oracle_cg(lambda v: Acg @ v, b_ref, rtol=1e-10, maxit=5000)
    x6_ref, _, _, _ = oracle_cg(lambda v: Acg @ v, b_ref, rtol=0.0, maxit=6)
    y_ref, yd_ref = A @ u, AD @ u
    for o in out:
        sl = slice(int(o["i0"]), int(o["i0"]) + o["y"].size)
        assert np.abs(o["y"] - y_ref[sl]).max() <= 1e-12 * np.abs(y_ref).max()
        assert np.abs(o["yd"] - yd_ref[sl]).max() <= 1e-12 * np.abs(yd_ref).max()
        assert np.abs(o["b"] - b_ref[sl]).max() <= 1e-14 * np.abs(b_ref).max()
        assert bool(o["ok"]) and abs(int(o["iters"]) - it_ref) <= max(3, it_ref // 100)
        assert np.abs(o["x"] - x_ref[sl]).max() <= 1e-8 * np.abs(x_ref).max()
        assert np.abs(o["x6"] - x6_ref[sl]).max() <= 1e-9 * np.abs(x6_ref).max()
    plane = (p * N + 1) ** (d - 1)
    for key in ("y", "yd", "b", "x", "x6"):
        assert np.array_equal(out[0][key][-plane:], out[1][key][:plane]), key
