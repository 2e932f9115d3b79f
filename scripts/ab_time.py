#!/usr/bin/env python
"""Apply timing for A/B builds (DOGIP_LIB=<variant .so>): median of K applies, each after
an L2 flush, per (config, storage).   python scripts/ab_time.py C5:sym C5:full C4:full"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1710_09913_b200.api import Mesh, Operator  # noqa: E402
from synth.configs import get_config  # noqa: E402
from bench import graph_timed_apply  # noqa: E402

CODE = {"full": 0, "iso": 1, "global": 2, "qp": 4, "sym": 5}
K = int(os.environ.get("AB_K", "15"))
flush = torch.empty(32 * 2 ** 20, dtype=torch.float64, device="cuda")
for spec in sys.argv[1:]:
    name, st = spec.split(":")
    c = get_config(name)
    form = c.forms[-1]
    m = Mesh(c.d, c.N, c.p, c.vertices())
    op = Operator(m, form, c.coefficient(), storage=CODE[st])
    u = torch.from_numpy(c.u()).cuda()
    y = torch.empty_like(u)
    for _ in range(3):
        op.apply(u, y, dirichlet=form == 1)
    t, ts = graph_timed_apply(torch, op, u, y, form == 1, flush, K)
    print(f"{os.path.basename(os.environ.get('DOGIP_LIB', 'base'))} {spec:12s} apply {t * 1e3:.4f} ms "
          f"(min {min(ts) * 1e3:.4f}; CUDA-graph replay, L2 flushed)", flush=True)
    op.close()
    m.close()
