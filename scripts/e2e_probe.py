#!/usr/bin/env python
"""Host-buffer apply (C4) vs raw pinned-copy bandwidth: is the pipelined e2e copy-bound?

    python scripts/e2e_probe.py            # DOGIP_HOST_CHUNKS sweep via env
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1710_09913_b200.api import Mesh, Operator  # noqa: E402
from synth.configs import get_config  # noqa: E402

c = get_config(os.environ.get("CFG", "C4"))
n = c.ndof
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


out = {"bytes": 8 * n,
       "h2d_ms": timed(lambda: d1.copy_(h1, non_blocking=True)),
       "d2h_ms": timed(lambda: h2.copy_(d2, non_blocking=True)),
       "both_ms": timed(both)}
m = Mesh(c.d, c.N, c.p, c.vertices())
op = Operator(m, c.forms[0], c.coefficient())
u = torch.from_numpy(c.u()).pin_memory()
y = torch.empty_like(u).pin_memory()
for k in (8, 16, 24, 32):
    os.environ["DOGIP_HOST_CHUNKS"] = str(k)
    out[f"apply_host_ms_K{k}"] = timed(lambda: op.apply_host_ptr(u.data_ptr(), y.data_ptr(), dirichlet=c.forms[0] == 1))
os.environ.pop("DOGIP_HOST_CHUNKS")
out["apply_device_ms"] = timed(lambda: op.apply(d1, d2, dirichlet=c.forms[0] == 1))
print(json.dumps(out))
