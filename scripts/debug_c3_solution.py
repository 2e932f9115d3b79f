"""Save the GPU C3 solve (x) and the GPU's A_D x for an offline oracle check."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1710_09913_b200.api import Mesh, Operator
from synth.configs import get_config
c = get_config("C3")
m = Mesh(3, c.N, c.p)
op = Operator(m, 1, c.coefficient())
b = op.load_vector(1.0, dirichlet=True)
x = torch.zeros_like(b)
res = op.cg(b, x, rtol=1e-10, maxit=20000, dirichlet=True)
y = op.apply(x, dirichlet=True)
print(res, (torch.linalg.vector_norm(b - y) / torch.linalg.vector_norm(b)).item())
os.makedirs(os.path.join(ROOT, "gpurun_out", "dbg"), exist_ok=True)
np.save(os.path.join(ROOT, "gpurun_out", "dbg", "c3_x.npy"), x.cpu().numpy())
np.save(os.path.join(ROOT, "gpurun_out", "dbg", "c3_y.npy"), y.cpu().numpy())
