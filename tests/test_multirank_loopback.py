"""The multi-rank data path on ONE GPU with real neighbour partial sums.

Every rank of a z-slab (2D: y-slab) partition is a mesh with the in-process loopback
communicator (include/dogip.h DOGIP_COMM_LOOPBACK), driven from its own host thread
with its own CUDA stream: boundary cube layers first, the interface-plane exchange
(A8: the neighbours' partial sums moved with cudaMemcpyAsync), the plane add, the
all-reduced CG dots and the batched predicated CG loop -- the same code the NCCL
backend runs, minus NCCL.  No kernel waits on another rank's kernel (host threads
rendezvous per collective; streams are ordered by events).

Checked against the CPU oracle (BASELINE north_star: apply 1e-12, CG to the same
residual) and for the invariant of SURVEY 8(e): interface planes bitwise equal on
both owners (IEEE a + b = b + a).
"""
import threading

import numpy as np
import pytest

from oracle import assemble as oa
from oracle.cg import cg as oracle_cg
from oracle.mesh import boundary_mask
from synth.configs import (COEF_ANISO_FOURIER, COEF_PER_CELL, COEF_TANH_RADIAL, Coefficient,
                           aniso_fourier_params)
from synth.generators import grf_per_cell, u_vector, vertex_jitter

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _jitter(d, N, seed=4):
    M = N + 1
    ids = np.arange(M ** d)
    X = np.stack([(ids // M ** a) % M for a in range(d)], axis=1) / N
    return X + vertex_jitter(d, N, 0.2, seed)


def _coef(kind, d, N):
    if kind == "aniso":
        return Coefficient(COEF_ANISO_FOURIER, aniso_fourier_params(2))
    if kind == "grf":
        return Coefficient(COEF_PER_CELL, np.zeros(0), grf_per_cell(d, N, 0.2, 1.0, 3))
    return Coefficient(COEF_TANH_RADIAL, np.array([1.0, 0.9, 20.0, 0.25] + [0.5] * d))


def _run_ranks(fn, nr):
    """fn(rank) in nr threads; re-raise the first failure."""
    errs, out = [None] * nr, [None] * nr

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:   # noqa: BLE001 -- reported below
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(nr)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a rank hung"
    for e in errs:
        if e is not None:
            raise e
    return out


CASES = [  # d, N, p, form, nranks, storage, coefficient
    (3, 6, 2, 1, 2, 0, "aniso"),
    (3, 7, 3, 1, 3, 1, "grf"),
    (3, 5, 4, 0, 2, 5, "tanh"),
    (2, 40, 2, 0, 3, 2, "tanh"),        # GLOBAL (Theorem 1): the weights setup itself exchanges
    (2, 36, 3, 1, 4, 0, "grf"),
    (3, 4, 2, 0, 4, 4, "tanh"),         # the quadrature-point comparator
    (3, 8, 1, 1, 8, 0, "grf"),          # one cube layer per rank
]


@pytest.mark.parametrize("d,N,p,form,nr,storage,ckind", CASES)
def test_loopback_ranks_match_oracle(d, N, p, form, nr, storage, ckind):
    import torch
    from paper_1710_09913_b200.api import LoopbackGroup, Mesh, Operator
    verts = _jitter(d, N)
    coef = _coef(ckind, d, N)
    ed = oa.build(d, N, p, verts)
    A = oa.assemble_csr(ed, form, coef)
    mask = boundary_mask(d, N, p)
    AD = oa.dirichlet_matrix(A, mask)
    dirichlet_cg = form == 1
    u = u_vector(ed.ndof, 8)
    b_ref = oa.load_vector(ed, 1.0, dirichlet=dirichlet_cg)
    Acg = AD if dirichlet_cg else A
    x_ref, it_ref, _, st_ref = oracle_cg(lambda v: Acg @ v, b_ref, rtol=1e-10, maxit=5000)
    x6_ref, _, _, _ = oracle_cg(lambda v: Acg @ v, b_ref, rtol=0.0, maxit=6)
    assert st_ref == 0

    group = LoopbackGroup(nr, device=0)
    meshes = [Mesh(d, N, p, verts, rank=r, nranks=nr, device=0, loopback=group) for r in range(nr)]
    streams = [torch.cuda.Stream() for _ in range(nr)]
    ops = [None] * nr

    def setup(r):
        ops[r] = Operator(meshes[r], form, coef, storage=storage, stream=streams[r])

    _run_ranks(setup, nr)                       # collective for GLOBAL storage

    def work(r):
        m, op, st = meshes[r], ops[r], streams[r]
        i0 = m.info["dof_offset"]
        with torch.cuda.stream(st):
            ul = torch.from_numpy(u[i0:i0 + m.ndof].copy()).cuda()
            st.synchronize()
            y = op.apply(ul, stream=st)
            yd = op.apply(ul, dirichlet=True, stream=st)
            b = op.load_vector(1.0, dirichlet=dirichlet_cg, stream=st)
            x = torch.zeros_like(b)
            res = op.cg(b, x, rtol=1e-10, maxit=5000, dirichlet=dirichlet_cg, stream=st)
            x6 = torch.zeros_like(b)
            res6 = op.cg(b, x6, maxit=-6, dirichlet=dirichlet_cg, stream=st)
            st.synchronize()
        return {"i0": i0, "n": m.ndof, "y": y.cpu().numpy(), "yd": yd.cpu().numpy(), "b": b.cpu().numpy(),
                "x": x.cpu().numpy(), "x6": x6.cpu().numpy(), "res": res, "res6": res6}

    out = _run_ranks(work, nr)
    torch.cuda.synchronize()
    y_ref, yd_ref = A @ u, AD @ u
    scale = np.abs(y_ref).max()
    for r, o in enumerate(out):
        sl = slice(o["i0"], o["i0"] + o["n"])
        assert np.abs(o["y"] - y_ref[sl]).max() <= TOL * scale, r
        assert np.abs(o["yd"] - yd_ref[sl]).max() <= TOL * np.abs(yd_ref).max(), r
        assert np.abs(o["b"] - b_ref[sl]).max() <= 1e-14 * np.abs(b_ref).max(), r
        assert o["res"]["status"] == "OK", o["res"]
        assert abs(o["res"]["iters"] - it_ref) <= max(3, it_ref // 100), (o["res"]["iters"], it_ref)
        assert np.abs(o["x"] - x_ref[sl]).max() <= 1e-8 * np.abs(x_ref).max(), r
        assert o["res6"]["iters"] == 6
        assert np.abs(o["x6"] - x6_ref[sl]).max() <= 1e-9 * np.abs(x6_ref).max(), r
    # every rank ran the same iteration count (one device-side stopping test per rank on
    # all-reduced scalars), and the interface planes agree bitwise on both owners
    assert len({o["res"]["iters"] for o in out}) == 1
    plane = (p * N + 1) ** (d - 1)
    for a, b in zip(out, out[1:]):
        for key in ("y", "yd", "b", "x", "x6"):
            assert np.array_equal(a[key][-plane:], b[key][:plane]), key
    for op in ops:
        op.close()
    for m in meshes:
        m.close()
    group.close()


def test_loopback_partials_without_exchange_and_group_lifetime():
    """DOGIP_NO_EXCHANGE on a loopback mesh returns this rank's partial sums (no
    collective, so one thread suffices); the group refuses to die while meshes use it."""
    import torch
    from paper_1710_09913_b200.api import DogipError, LoopbackGroup, Mesh, Operator
    d, N, p, nr = 3, 5, 2, 2
    coef = _coef("grf", d, N)
    group = LoopbackGroup(nr, device=0)
    meshes = [Mesh(d, N, p, rank=r, nranks=nr, device=0, loopback=group) for r in range(nr)]
    ed = oa.build(d, N, p)
    u = u_vector(ed.ndof, 2)
    acc = np.zeros_like(u)
    for m in meshes:
        op = Operator(m, 1, coef)
        i0 = m.info["dof_offset"]
        acc[i0:i0 + m.ndof] += op.apply(torch.from_numpy(u[i0:i0 + m.ndof].copy()).cuda(),
                                        exchange=False).cpu().numpy()
        op.close()
    y = oa.assemble_csr(ed, 1, coef) @ u
    assert np.abs(acc - y).max() <= 1e-13 * np.abs(y).max()
    with pytest.raises(DogipError):
        group.close()
    with pytest.raises(DogipError):                  # one mesh per rank and group
        Mesh(d, N, p, rank=1, nranks=nr, device=0, loopback=group)
    for m in meshes:
        m.close()
    group.close()


_DEAD_PEER = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_1710_09913_b200.api import DogipError, LoopbackGroup, Mesh, Operator
from synth.configs import COEF_CONST, Coefficient
g = LoopbackGroup(2, device=0)
ms = [Mesh(3, 4, 2, rank=r, nranks=2, device=0, loopback=g) for r in range(2)]
ops = [Operator(m, 1, Coefficient(COEF_CONST, np.array([1.0]))) for m in ms]
u = torch.zeros(ms[0].ndof, dtype=torch.float64, device="cuda")
try:                                   # rank 1 never calls: rank 0 must not hang
    ops[0].apply(u)
    print("NO_ERROR")
except DogipError as e:
    print("RANK0", e.code, str(e))
try:                                   # the group is dead: rank 1 fails at once
    ops[1].apply(torch.zeros(ms[1].ndof, dtype=torch.float64, device="cuda"))
    print("NO_ERROR")
except DogipError as e:
    print("RANK1", e.code, str(e))
"""


def test_dead_peer_times_out_instead_of_hanging():
    """A rank whose neighbour never joins the collective gets E_NCCL after
    DOGIP_COMM_TIMEOUT_S instead of hanging, and the communicator is then dead for every
    rank (include/dogip.h dogip_apply / dogip_cg error behaviour)."""
    import os
    import subprocess
    import sys
    import time
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DOGIP_COMM_TIMEOUT_S="2")
    t0 = time.time()
    r = subprocess.run([sys.executable, "-c", _DEAD_PEER.format(root=root)], capture_output=True, text=True,
                       timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = {l.split()[0]: l for l in r.stdout.splitlines() if l.startswith("RANK")}
    assert "NO_ERROR" not in r.stdout
    assert lines["RANK0"].split()[1] == "-8" and "timeout" in lines["RANK0"]
    assert lines["RANK1"].split()[1] == "-8" and "dead" in lines["RANK1"]
    assert time.time() - t0 < 200
