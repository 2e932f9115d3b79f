"""Multi-rank slab decomposition on CPU: world size 2 (and 3) with gloo.

Each rank takes the library's own host-side plan (dogip_mesh_setup with
device = -1: slab range, DoF offset, owned range, local l_T), computes its
partial y on its slab's elements (oracle element matrices), exchanges the two
interface planes with its neighbours exactly as dogip_apply does (send my
first plane to rank-1 and my last plane to rank+1, add what is received), and
runs CG with dots over owned DoFs all-reduced.  The result must equal the
global oracle apply / solve.  This covers the N > 1 host logic without GPUs
(the NCCL calls are the same plan on device buffers).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, d, N, p, form, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import assemble as oa
        from oracle.cg import cg as ocg
        from oracle.mesh import boundary_mask
        from paper_1710_09913_b200.api import Mesh
        from synth.configs import (COEF_ANISO_FOURIER, COEF_SINCOS2D, COEF_TANH_RADIAL, Coefficient,
                                   aniso_fourier_params)
        from synth.generators import u_vector
        coef = (Coefficient(COEF_SINCOS2D, np.array([1.0, 0.5])) if d == 2 else
                (Coefficient(COEF_ANISO_FOURIER, aniso_fourier_params(2)) if form == 1 else
                 Coefficient(COEF_TANH_RADIAL, np.array([1.0, 0.9, 20.0, 0.25, 0.5, 0.5, 0.5]))))
        ed = oa.build(d, N, p)
        m = Mesh(d, N, p, rank=rank, nranks=world, device=-1)
        info = m.info
        off, n, plane = info["dof_offset"], info["ndof_local"], info["plane_size"]
        ns = 2 if d == 2 else 6
        e0 = ns * N ** (d - 1) * info["z0"]
        e1 = ns * N ** (d - 1) * info["z1"]
        lT = m.dofmap()                                   # LOCAL ids from the library
        assert np.array_equal(lT + off, ed.lT[e0:e1])
        K = ed.element_matrices(form, coef, slice(e0, e1))
        dirichlet = form == 1
        bmask_g = boundary_mask(d, N, p)
        bmask = bmask_g[off:off + n]

        def local_apply(v):
            vv = np.where(bmask, 0.0, v) if dirichlet else v
            yl = np.einsum("eij,ej->ei", K, vv[lT])
            y = np.bincount(lT.ravel(), weights=yl.ravel(), minlength=n)
            # interface exchange (A8), same plan as dogip_apply
            reqs, lo, hi = [], None, None
            if rank > 0:
                lo = torch.empty(plane, dtype=torch.float64)
                reqs.append(dist.isend(torch.from_numpy(y[:plane].copy()), rank - 1))
                reqs.append(dist.irecv(lo, rank - 1))
            if rank < world - 1:
                hi = torch.empty(plane, dtype=torch.float64)
                reqs.append(dist.isend(torch.from_numpy(y[n - plane:].copy()), rank + 1))
                reqs.append(dist.irecv(hi, rank + 1))
            for r in reqs:
                r.wait()
            if lo is not None:
                y[:plane] += lo.numpy()
            if hi is not None:
                y[n - plane:] += hi.numpy()
            if dirichlet:
                y[bmask] = v[bmask]
            return y

        ob, oe = info["owned_begin"], info["owned_end"]

        def gdot(a, b):
            t = torch.tensor([float(a[ob:oe] @ b[ob:oe])], dtype=torch.float64)
            dist.all_reduce(t)
            return t.item()

        u = u_vector(ed.ndof, 2)
        A = oa.assemble_csr(ed, form, coef)
        AD = oa.dirichlet_matrix(A, bmask_g) if dirichlet else A
        y_ref = (AD @ u)[off:off + n]
        y = local_apply(u[off:off + n])
        err_apply = np.abs(y - y_ref).max() / np.abs(AD @ u).max()
        # owned ranges tile the global vector exactly once
        cnt = torch.tensor([float(oe - ob)], dtype=torch.float64)
        dist.all_reduce(cnt)
        # distributed CG (same recurrences as dogip_cg)
        b = oa.load_vector(ed, 1.0, dirichlet)[off:off + n]
        x = np.zeros(n)
        r = b.copy()
        pv = r.copy()
        rr = gdot(r, r)
        bn = np.sqrt(gdot(b, b))
        it = 0
        while np.sqrt(rr) > 1e-10 * bn and it < 5000:
            qv = local_apply(pv)
            alpha = rr / gdot(pv, qv)
            x += alpha * pv
            r -= alpha * qv
            rr_new = gdot(r, r)
            pv = r + (rr_new / rr) * pv
            rr = rr_new
            it += 1
        xg, itg, _, _ = ocg(lambda v: AD @ v, oa.load_vector(ed, 1.0, dirichlet), rtol=1e-10)
        err_x = np.abs(x - xg[off:off + n]).max() / np.abs(xg).max()
        q.put((rank, err_apply, cnt.item(), ed.ndof, it, itg, err_x))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d,N,p,form,world", [(3, 4, 2, 1, 2), (2, 9, 3, 1, 3), (3, 5, 2, 0, 2)])
def test_slab_exchange_and_distributed_cg(d, N, p, form, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, N, p, form, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, err_apply, cnt, ndof, it, itg, err_x in res:
        assert err_apply <= 1e-13, (rank, err_apply)
        assert cnt == ndof
        assert abs(it - itg) <= 3
        assert err_x <= 1e-8
