"""C4 solved to convergence (rtol 1e-8, Dirichlet, graph CG) with FULL and ISO storage;
prints iterations, recursive and true relative residual, wall time.  python scripts/c4_solve.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1710_09913_b200.api import Mesh, Operator  # noqa: E402
from synth.configs import get_config  # noqa: E402
for store in (0, 1):
    c = get_config("C4")
    m = Mesh(c.d, c.N, c.p, c.vertices(), device=0)
    op = Operator(m, 1, c.coefficient(), storage=store)
    b = op.load_vector(1.0, dirichlet=True)
    x = torch.zeros_like(b)
    torch.cuda.synchronize(); t0 = time.time()
    r = op.cg(b, x, rtol=1e-8, maxit=20000, dirichlet=True)
    torch.cuda.synchronize(); t1 = time.time()
    y = op.apply(x, dirichlet=True)
    true = (torch.linalg.norm(y - b) / torch.linalg.norm(b)).item()
    print(json.dumps({"config": "C4", "storage": ["full", "iso"][store], "rtol": 1e-8, "iters": r["iters"], "status": r["status"],
                      "rel_res": r["rel_res"], "true_rel_res": true, "solve_s": t1 - t0,
                      "ms_per_iter": 1e3 * (t1 - t0) / max(1, r["iters"])}))
    op.close(); m.close(); torch.cuda.empty_cache()
