#!/usr/bin/env python
"""One config, one storage variant, a few applies -- the target of an ncu capture.

    python scripts/prof_apply.py C5 --storage 3 --reps 3
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1710_09913_b200.api import Mesh, Operator  # noqa: E402
from synth.configs import get_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--storage", type=int, default=0)
ap.add_argument("--form", type=int, default=-1)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
c = get_config(a.config)
form = a.form if a.form >= 0 else c.forms[0]
m = Mesh(c.d, c.N, c.p, c.vertices())
op = Operator(m, form, c.coefficient(), storage=a.storage)
u = torch.from_numpy(c.u()).cuda()
y = torch.empty_like(u)
for _ in range(a.reps):
    op.apply(u, y, dirichlet=form == 1)
torch.cuda.synchronize()
print("ok", a.config, form, a.storage)
