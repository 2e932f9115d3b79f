#!/usr/bin/env python
"""Full-size CG parity: the GPU solves C3 and C5 through the C ABI, the CPU oracle
recomputes the TRUE residual of the GPU solution (reading L15: ||b - A x|| / ||b|| must
be <= 2 tol).

  C3  3D 64^3 x 6 P2 EL, rotated anisotropic tensor, f = 1, zero Dirichlet, tol 1e-10
  C5  3D 96^3 x 6 jittered P4 WP, tanh inclusion, f = 1, no BC,          tol 1e-12
  C4  3D 128^3 x 6 P3 EL, log-normal per cell, f = 1, zero Dirichlet,    tol 1e-8 (optional)

The oracle side builds b by its own load vector (eq:linsys_gp P:207 / eq:linsys_se P:337)
and applies A by the quadrature-point route (oracle.assemble.apply_qp_route, pinned equal
to the CSR assembly in tests/test_oracle_sampled_and_coefficients.py); nothing on that side
comes from the CUDA path except the solution x under test.

    python tests/oracle_residual.py [--out gpurun_out/r02_oracle_residual.json] [C3 C5]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TOLS = {"C3": 1e-10, "C5": 1e-12, "C4": 1e-8}   # C4: BJ times CG per iteration; solved to 1e-8 here


def gpu_solve(name, storage):
    import torch
    from paper_1710_09913_b200.api import Mesh, Operator
    from synth.configs import get_config
    c = get_config(name)
    form = c.forms[0]
    dirichlet = form == 1
    m = Mesh(c.d, c.N, c.p, c.vertices())
    op = Operator(m, form, c.coefficient(), storage=storage)
    b = op.load_vector(1.0, dirichlet=dirichlet)
    x = torch.zeros_like(b)
    res = op.cg(b, x, rtol=TOLS[name], maxit=40000, dirichlet=dirichlet)
    torch.cuda.synchronize()
    out = (b.cpu().numpy(), x.cpu().numpy(), res, op.info["weights_ms"])
    op.close()
    m.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C3", "C5"])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "r02_oracle_residual.json"))
    ap.add_argument("--workers", type=int, default=min(32, os.cpu_count() or 1))
    a = ap.parse_args()
    from oracle import assemble as oa
    from synth.configs import get_config
    rows = []
    for name in a.configs:
        c = get_config(name)
        form = c.forms[0]
        dirichlet = form == 1
        storages = [0] if form == 1 else [0, 5]          # C5: FULL and the symmetry-adapted storage
        t0 = time.perf_counter()
        ed = oa.build(c.d, c.N, c.p, c.vertices())
        coef = c.coefficient()
        b_ref = oa.load_vector(ed, 1.0, dirichlet=dirichlet)
        t_build = time.perf_counter() - t0
        for storage in storages:
            b, x, res, wms = gpu_solve(name, storage)
            t1 = time.perf_counter()
            Ax = oa.apply_qp_route(ed, form, coef, x, dirichlet=dirichlet, workers=a.workers)
            t_apply = time.perf_counter() - t1
            true_res = float(np.linalg.norm(b_ref - Ax) / np.linalg.norm(b_ref))
            b_err = float(np.abs(b - b_ref).max() / np.abs(b_ref).max())
            row = {"config": name, "storage": {0: "full", 5: "sym"}[storage], "tol": TOLS[name],
                   "gpu_iters": res["iters"], "gpu_status": res["status"], "gpu_rel_res_recursive": res["rel_res"],
                   "gpu_solve_s": res["seconds"], "weights_ms": wms,
                   "oracle_true_rel_res": true_res, "pass": bool(true_res <= 2 * TOLS[name] and b_err <= 1e-12),
                   "load_vector_rel_err": b_err, "ndof": int(b.size),
                   "oracle_route": "apply_qp_route (quadrature-point route, %d threads)" % a.workers,
                   "oracle_build_s": t_build, "oracle_apply_s": t_apply}
            print(json.dumps(row), flush=True)
            rows.append(row)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"rows": rows, "cpu_cores": os.cpu_count()}, f, indent=1)
    if not all(r["pass"] for r in rows):
        sys.exit(1)


if __name__ == "__main__":
    main()
